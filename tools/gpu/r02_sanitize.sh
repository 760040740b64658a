set -x
mkdir -p gpurun_out/r02/sanitize
timeout 600 python tests/sanitize_case.py > gpurun_out/r02/sanitize/plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check no python tests/sanitize_case.py > gpurun_out/r02/sanitize/memcheck.log 2>&1
timeout 1500 compute-sanitizer --tool synccheck python tests/sanitize_case.py > gpurun_out/r02/sanitize/synccheck.log 2>&1
tail -n 5 gpurun_out/r02/sanitize/*.log
