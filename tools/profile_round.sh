#!/bin/bash
# GPU box: the round's evidence set under gpurun_out/prof/ -- bench lines for
# every config, the config-3 launch list (gpu__time_duration, the profiling
# recipe's pass) and one ncu --set full capture of the hot kernels of
# configs 3 and 4 (each only after its own command exited 0 without ncu).
cd "$(dirname "$0")/.."
P=gpurun_out/prof
mkdir -p $P
python bench.py --config 3 > $P/bench_config3.json 2> $P/bench_config3.err || exit 1
for c in 4 5 1 2; do
  python bench.py --config $c --no-cpu > $P/bench_config$c.json 2> $P/bench_config$c.err || exit 1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $P/launches_config3.csv python bench.py --config 3 --no-cpu --steps 2 --warmup 3 \
    > $P/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_spread|_r1|k_gather2" \
    --launch-count 5 -o $P/c3 python bench.py --config 3 --no-cpu --steps 1 --warmup 3 \
    > $P/ncu_c3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_spread_b|_rb|k_gather_b" \
    --launch-count 5 -o $P/c4 python bench.py --config 4 --no-cpu --steps 1 --warmup 3 \
    > $P/ncu_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_spread_dense|k_spread_small|k_gather2|_d?step" \
    --launch-count 8 -o $P/c5 python bench.py --config 5 --no-cpu --steps 1 --warmup 3 \
    > $P/ncu_c5.log 2>&1
ls -la $P
