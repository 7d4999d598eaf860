P=gpurun_out/r02ag; mkdir -p $P
for m in 2 4 6 8 10; do python bench.py --config 2 --m $m --no-cpu > $P/new_m$m.json 2>/dev/null; SFB_DIRECT_PARMIN=0 python bench.py --config 2 --m $m --no-cpu > $P/old_m$m.json 2>/dev/null; done
python bench.py --config 5 --no-cpu > $P/c5.json 2>/dev/null; python bench.py --config 1 --no-cpu > $P/c1.json 2>/dev/null
python -m pytest tests -q -m gpu -x -k "not slow" 2>&1 | tail -2
