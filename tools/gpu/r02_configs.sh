# Round-2 numbers for every BASELINE config on one GPU (default kernels), plus the reference arm.
set -x
mkdir -p gpurun_out/r02/configs
for c in glm16k small glm64k stress; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02/configs/n1_$c.jsonl 2> gpurun_out/r02/configs/n1_$c.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02/configs/reference.jsonl 2> gpurun_out/r02/configs/reference.err
python tools/bench_summary.py gpurun_out/r02/configs/n1_*.jsonl
cat gpurun_out/r02/configs/reference.jsonl
