# the sparse backward keeps its gain with the fused NVLS collectives on.
# N = 2, NVLS on: vocab-parallel glm64k with the stress config's mismatch (delta sigma 1.0,
# ~43% of rows masked; NVLS dH reduction in K5) and DP stress (NVLS dW reduction in K6),
# sparse (default) vs --dense-backward, alternating.
set -x
mkdir -p gpurun_out/r02/sparse_nvls
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29512 --nproc-per-node 2"
for i in 1 2; do
  timeout 900 $T bench.py --gpus 2 --config glm64k --delta-sigma 1.0 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02/sparse_nvls/vp_sparse_$i.jsonl 2>/dev/null
  timeout 900 $T bench.py --gpus 2 --config glm64k --delta-sigma 1.0 --steps 10 --warmup 3 --no-cpu-baseline --dense-backward > gpurun_out/r02/sparse_nvls/vp_dense_$i.jsonl 2>/dev/null
  timeout 900 $T bench.py --gpus 2 --config stress --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02/sparse_nvls/dp_stress_sparse_$i.jsonl 2>/dev/null
  timeout 900 $T bench.py --gpus 2 --config stress --steps 20 --warmup 3 --no-cpu-baseline --dense-backward > gpurun_out/r02/sparse_nvls/dp_stress_dense_$i.jsonl 2>/dev/null
done
python tools/bench_summary.py gpurun_out/r02/sparse_nvls/*.jsonl
