mkdir -p gpurun_out/r02b
python -m pytest tests/test_windows.py -q -m gpu 2>&1 | tail -3 > gpurun_out/r02b/pytest_windows.log
python tools/diag_small_m.py > gpurun_out/r02b/diag_small_m.log 2>&1
python tools/sanitize_cases.py > gpurun_out/r02b/sanitize_plain.log 2>&1; echo rc=$? >> gpurun_out/r02b/sanitize_plain.log
OUT=gpurun_out/r02b/var tools/run_variants.sh > gpurun_out/r02b/variants.log 2>&1
