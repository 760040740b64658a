# Probability cache with chunked dU (the cache holds the whole batch; K4 fills each chunk from it):
# parity subset (chunked cases included), then the chunked configs (small, glm64k) with the cache on / off.
set -x
D=gpurun_out/r02/pchunk
mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_workspace_poison.py tests/test_gpu_parity.py tests/test_gpu_sparse_bwd.py tests/test_gpu_kl_temperature.py tests/test_gpu_kernel_variants.py -q -p no:cacheprovider 2>&1 | tail -3 > $D/parity.log
cat $D/parity.log
for c in small glm64k; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $D/${c}_on.jsonl 2>/dev/null
  RL_P_CACHE=0 timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $D/${c}_off.jsonl 2>/dev/null
done
python tools/bench_summary.py $D/*.jsonl
