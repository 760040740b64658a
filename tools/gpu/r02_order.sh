# Tile-order independence (bitwise) on one GPU, then compute-sanitizer memcheck of the
# default step (K1 / K4 in dynamic tile order: the shared-memory tile ring across the pair).
set -x
mkdir -p gpurun_out/r02/order
timeout 1200 python -m pytest tests/test_gpu_tile_order.py -q -s -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/r02/order/tile_order_test.log
cat gpurun_out/r02/order/tile_order_test.log
timeout 600 python tests/sanitize_case.py > gpurun_out/r02/order/plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check no python tests/sanitize_case.py > gpurun_out/r02/order/memcheck.log 2>&1
tail -n 5 gpurun_out/r02/order/*.log
