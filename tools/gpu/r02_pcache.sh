# K4 from K1's probability cache (RL_P_CACHE, default 1) vs the recompute GEMM (RL_P_CACHE=0):
# parity first (the whole single-GPU parity set with the cache on), then 3 alternating bench rounds.
set -x
mkdir -p gpurun_out/r02/pcache
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_bwd.py tests/test_gpu_kl_temperature.py tests/test_gpu_degenerate.py -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r02/pcache/parity.log
tail -3 gpurun_out/r02/pcache/parity.log
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
for i in 1 2 3; do
  RL_P_CACHE=0 $B > gpurun_out/r02/pcache/off_$i.jsonl 2>gpurun_out/r02/pcache/off_$i.err
  RL_P_CACHE=1 $B > gpurun_out/r02/pcache/on_$i.jsonl 2>gpurun_out/r02/pcache/on_$i.err
done
python tools/bench_summary.py gpurun_out/r02/pcache/*.jsonl
tail -3 gpurun_out/r02/pcache/on_1.err
