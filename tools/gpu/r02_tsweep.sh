# Micro-batch size sweep at the GLM shape on one GPU (tokens per step 1k..64k), default kernels
set -x
mkdir -p gpurun_out/r02/tsweep
for t in 1024 2048 4096 8192 16384 32768 65536; do
  timeout 600 python bench.py --tokens $t --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02/tsweep/t$t.jsonl 2>/dev/null
done
python tools/bench_summary.py gpurun_out/r02/tsweep/*.jsonl
