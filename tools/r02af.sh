P=gpurun_out/r02af; mkdir -p $P
for m in 2 4 6 8 10; do python bench.py --config 2 --m $m --no-cpu > $P/bench_config2_m$m.json 2>$P/err_m$m.txt; done
python tools/kernel_times.py 5 > $P/kt5.txt 2>&1
python tools/kernel_times.py 2 > $P/kt2.txt 2>&1
