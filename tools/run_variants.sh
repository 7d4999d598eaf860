#!/bin/bash
# dev helper (GPU box): in-stream kernel times of config $CFG (default 3) for
# the default library and every lib/var_*.so, each checked against the first.
cd "$(dirname "$0")/.."
OUT=${OUT:-gpurun_out/var}; mkdir -p $OUT; rm -f /tmp/var_base.npy
for lib in paper_2107_02671_b200/lib/libsincfft_b200.so paper_2107_02671_b200/lib/var_*.so; do
  n=$(basename $lib .so)
  for rep in ${REPS:-1}; do
    VAR_REF=/tmp/var_base.npy SINCFFT_B200_LIB=$PWD/$lib timeout 300 python tools/kernel_times.py ${CFG:-3} > $OUT/$n.txt 2>&1
  done
  echo "== $n"; grep -E "k_|total|max\|" $OUT/$n.txt | head -${TOP:-12}
done
