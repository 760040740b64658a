# N = 4 DP glm16k: current build vs b9773dc (before the K6 8-warp / K1 early-release changes), alternating
set -x
mkdir -p gpurun_out/r02/n4ab
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29516 --nproc-per-node 4"
for i in 1 2; do
  RL_LIBRARY=ab_libs/librl_prev.so timeout 900 $T bench.py --gpus 4 --steps 20 --warmup 3 --no-e2e > gpurun_out/r02/n4ab/prev_$i.jsonl 2>/dev/null
  timeout 900 $T bench.py --gpus 4 --steps 20 --warmup 3 --no-e2e > gpurun_out/r02/n4ab/cur_$i.jsonl 2>/dev/null
done
python tools/bench_summary.py gpurun_out/r02/n4ab/*.jsonl
