# NVLS reduce-scatter (FSDP-consistent) vs all-reduce of dW with the communication warps, N = 2, alternating.
set -x
mkdir -p gpurun_out/r02/rs
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29514 --nproc-per-node 2"
for i in 1 2; do
  timeout 900 $T bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/rs/ar_$i.jsonl 2>/dev/null
  timeout 900 $T bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --dw-reduce-scatter > gpurun_out/r02/rs/rs_$i.jsonl 2>/dev/null
done
python tools/bench_summary.py gpurun_out/r02/rs/*.jsonl
