#!/bin/bash
# GPU box: per-kernel FP64-pipe and DRAM counters for the hot kernels of
# configs 3, 4 and 5 (one ncu metrics pass each, after a plain run of the
# same command exited 0).  Output: $OUT/pipes_config{3,4,5}.csv
cd "$(dirname "$0")/.."
OUT=${OUT:-gpurun_out/pipes}
mkdir -p $OUT
MET=gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_fp64_pred_on.sum,sm__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg,sm__warps_active.avg.pct_of_peak_sustained_active
for c in ${CONFIGS:-3 4 5}; do
  cmd="python bench.py --config $c --no-cpu --steps 2 --warmup 3"
  $cmd > $OUT/plain_config$c.log 2>&1 || { echo "plain run config $c failed"; exit 1; }
  ncu --metrics $MET --clock-control none -k regex:"${KREGEX:-k_}" -s ${SKIP:-0} -c ${COUNT:-160} --csv \
      --log-file $OUT/pipes_config$c.csv $cmd > $OUT/ncu_config$c.log 2>&1
done
ls -la $OUT
