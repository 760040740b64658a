# NVLS reductions on dedicated communication warps (rl_nvls_reduce.lag = 0, default) vs the round-1
# schedule (epilogue warps, lag 2): parity first, then alternating A/B at N = 2 (DP glm16k, DP stress,
# vocab-parallel glm64k).
set -x
mkdir -p gpurun_out/r02/comm
timeout 1200 python -m pytest tests -m gpu -q -s -p no:cacheprovider -k "multi or nvls" > gpurun_out/r02/comm/gpu2_suite.log 2>&1
tail -3 gpurun_out/r02/comm/gpu2_suite.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29513 --nproc-per-node 2"
for i in 1 2; do
  for lag in 0 2; do
    RL_NVLS_LAG=$lag timeout 900 $T bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02/comm/dp_lag${lag}_$i.jsonl 2>/dev/null
    RL_NVLS_LAG=$lag timeout 900 $T bench.py --gpus 2 --config stress --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/comm/stress_lag${lag}_$i.jsonl 2>/dev/null
    RL_NVLS_LAG=$lag timeout 900 $T bench.py --gpus 2 --config glm64k --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/comm/vp_lag${lag}_$i.jsonl 2>/dev/null
  done
done
python tools/bench_summary.py gpurun_out/r02/comm/*.jsonl
