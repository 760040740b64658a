# Split-K dH for chunks with fewer output tiles than CTA pairs: the whole -m gpu suite (the mid-size
# parity cases split), then small-T bench A/B vs the previous build (ab_libs/librl_prev.so).
set -x
mkdir -p gpurun_out/r02/dhsplit2
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_bwd.py tests/test_gpu_kl_temperature.py -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/r02/dhsplit2/gpu1_suite.log
for t in 1024 1536 2048; do
  for v in prev cur; do
    lib=""; [ $v = prev ] && lib=ab_libs/librl_prev.so
    RL_LIBRARY=$lib timeout 600 python bench.py --tokens $t --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/dhsplit2/t${t}_$v.jsonl 2>/dev/null
  done
done
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/dhsplit2/t16384_cur.jsonl 2>/dev/null
cat gpurun_out/r02/dhsplit2/gpu1_suite.log
python tools/bench_summary.py gpurun_out/r02/dhsplit2/*.jsonl
