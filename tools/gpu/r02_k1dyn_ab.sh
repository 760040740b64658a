# K1 knobs re-measured in the dynamic tile order: 16 epilogue warps, MMA skew 2 (default 8 warps, skew 3).
set -x
mkdir -p gpurun_out/r02/k1dyn_ab
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
for i in 1 2 3; do
  $B > gpurun_out/r02/k1dyn_ab/default_$i.jsonl 2>/dev/null
  RL_EPI_WARPS_FWD=16 $B > gpurun_out/r02/k1dyn_ab/epi16_$i.jsonl 2>/dev/null
  RL_SKEW=2 $B > gpurun_out/r02/k1dyn_ab/skew2_$i.jsonl 2>/dev/null
done
python tools/bench_summary.py gpurun_out/r02/k1dyn_ab/*.jsonl
