mkdir -p gpurun_out/r02p
python -m pytest tests -m gpu -q -x -s -k "fullsize or windows" 2>&1 | grep -E "config|window parity|passed|failed|Error" > gpurun_out/r02p/pytest_fullsize.log
python tools/sanitize_cases.py > gpurun_out/r02p/sanitize_plain.log 2>&1 && \
compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_cases.py > gpurun_out/r02p/memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/r02p/memcheck.log
