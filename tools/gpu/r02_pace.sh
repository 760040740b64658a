# K4 store pacing (RL_EPI_PACE_DZ ns after each chunk's store), alternating A/B, 2 rounds (2nd reversed)
set -x
mkdir -p gpurun_out/r02/pace
for p in 0 500 1000 2000; do RL_EPI_PACE_DZ=$p timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/pace/p${p}_1.jsonl 2>/dev/null; done
for p in 2000 1000 500 0; do RL_EPI_PACE_DZ=$p timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/pace/p${p}_2.jsonl 2>/dev/null; done
python tools/bench_summary.py gpurun_out/r02/pace/*.jsonl
