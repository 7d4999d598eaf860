#!/bin/bash
# GPU box: the final round-2 evidence set under gpurun_out/r02w/ -- GPU suite,
# bench lines for every config (config 2 at every cut-off of BASELINE's
# sweep), ncu FP64-pipe / DRAM counters (configs 3, 4, 5), the config-3 launch
# list, and ncu --set full captures of the config-3 and config-4 hot kernels
# (each ncu run only after its own command exited 0 without ncu).
cd "$(dirname "$0")/.."
P=gpurun_out/r02w; mkdir -p $P
python -m pytest tests -m gpu -q 2>&1 | tail -4 > $P/pytest_gpu.log
python bench.py > $P/bench_config3.json 2> $P/bench_config3.err
for c in 4 5 1 2; do python bench.py --config $c --no-cpu > $P/bench_config$c.json 2> $P/bench_config$c.err; done
for m in 2 4 6 10; do python bench.py --config 2 --m $m --no-cpu > $P/bench_config2_m$m.json 2> /dev/null; done
OUT=$P/pipes tools/ncu_pipes.sh > $P/pipes.log 2>&1
cmd="python bench.py --config 3 --no-cpu --steps 2 --warmup 3"
$cmd > $P/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $P/launches_config3.csv $cmd > $P/ncu_launch.log 2>&1
$cmd > $P/plain2.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_spread|_r1|k_gather2" -s 0 -c 5 -o $P/c3 $cmd > $P/ncu_c3.log 2>&1
cmd4="python bench.py --config 4 --no-cpu --steps 1 --warmup 3"
$cmd4 > $P/plain4.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_spread_bw|k_gather_b|_rb" -s 5 -c 5 -o $P/c4 $cmd4 > $P/ncu_c4.log 2>&1
for c in 3 4; do
  python tools/ncu_digest.py $P/c$c.ncu-rep > $P/ncu_summary_config$c.txt 2>&1
  python tools/ncu_traffic.py $c $P/c$c.ncu-rep > $P/traffic_config$c.log 2>&1
done
cp profiles/ncu_traffic.json $P/ncu_traffic.json
python - <<PY > $P/fp64_pipes.txt 2>&1
import sys, subprocess
sys.path.insert(0, "tools")
for c in (3, 4, 5):
    print(f"== config {c}")
    print(subprocess.run([sys.executable, "tools/pipes_digest.py", "$P/pipes/pipes_config%d.csv" % c],
                         capture_output=True, text=True).stdout)
sys.argv = ["pipes_digest.py", "$P/pipes/pipes_config3.csv"]
import io, contextlib
with contextlib.redirect_stdout(io.StringIO()):
    import pipes_digest
print(pipes_digest.fp64_json([(c, "$P/pipes/pipes_config%d.csv" % c) for c in (3, 4, 5)], "$P/ncu_fp64.json"))
PY
ls -la $P
