#!/bin/bash
# GPU box: the round-2 evidence set under gpurun_out/prof2/ -- GPU suite, bench
# lines for every config, ncu FP64-pipe / DRAM counters (configs 3, 4, 5), the
# config-3 launch list, and one ncu --set full capture of the config-3 hot
# kernels (each ncu run only after its own command exited 0 without ncu).
cd "$(dirname "$0")/.."
P=gpurun_out/prof2; mkdir -p $P
python -m pytest tests -m gpu -q 2>&1 | tail -4 > $P/pytest_gpu.log
python bench.py > $P/bench_config3.json 2> $P/bench_config3.err
for c in 4 5 1 2; do python bench.py --config $c --no-cpu > $P/bench_config$c.json 2> $P/bench_config$c.err; done
OUT=$P/pipes tools/ncu_pipes.sh > $P/pipes.log 2>&1
cmd="python bench.py --config 3 --no-cpu --steps 2 --warmup 3"
$cmd > $P/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $P/launches_config3.csv $cmd > $P/ncu_launch.log 2>&1
$cmd > $P/plain2.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_spread|_r1|k_gather2" -s 0 -c 5 -o $P/c3 $cmd > $P/ncu_c3.log 2>&1
ls -la $P
