#!/bin/bash
# GPU box: one ncu --set full capture of the kernels matching $1 in config $2
# (default 3) after a plain run of the same command; report -> $OUT/$3.ncu-rep
cd "$(dirname "$0")/.."
OUT=${OUT:-gpurun_out/ncu}; mkdir -p $OUT
cmd="python bench.py --config ${2:-3} --no-cpu --steps 1 --warmup 3"
$cmd > $OUT/plain.log 2>&1 || { echo "plain run failed"; tail $OUT/plain.log; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:"$1" -s ${SKIP:-2} -c ${COUNT:-1} \
    -o $OUT/${3:-prof} $cmd > $OUT/ncu.log 2>&1
tail -3 $OUT/ncu.log
