P=gpurun_out/r02u; mkdir -p $P
python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > $P/pytest_gpu.log
python bench.py > $P/bench_config3.json 2> $P/bench_config3.err
for c in 4 5 1 2; do python bench.py --config $c --no-cpu > $P/bench_config$c.json 2> $P/bench_config$c.err; done
python bench.py --config 3 --no-cpu --steps 2 --warmup 3 > $P/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $P/launches_config3.csv \
    python bench.py --config 3 --no-cpu --steps 2 --warmup 3 > $P/ncu_launch.log 2>&1
ls -la $P
