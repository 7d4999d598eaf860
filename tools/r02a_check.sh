set -x
mkdir -p gpurun_out/r02a
python -m pytest tests -m gpu -q -x -s 2>&1 | tail -40 > gpurun_out/r02a/pytest_gpu.log
python bench.py --gpus 2 --dist-backend gloo --same-device --check-shards --steps 5 --no-cpu > gpurun_out/r02a/bench_2rank_gloo.json 2> gpurun_out/r02a/bench_2rank_gloo.err; echo rc=$? >> gpurun_out/r02a/bench_2rank_gloo.err
python tools/sanitize_cases.py > gpurun_out/r02a/sanitize_plain.log 2>&1; echo rc=$? >> gpurun_out/r02a/sanitize_plain.log
python bench.py > gpurun_out/r02a/bench_config3.json 2> gpurun_out/r02a/bench_config3.err
