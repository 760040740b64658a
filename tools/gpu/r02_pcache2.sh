# Probability cache after the padding-row fix: the whole -m gpu suite on one GPU, then 3 alternating
# bench rounds cache on (default) / off.
set -x
mkdir -p gpurun_out/r02/pcache2
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/r02/pcache2/gpu1_suite.log
tail -3 gpurun_out/r02/pcache2/gpu1_suite.log
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
for i in 1 2 3; do
  $B > gpurun_out/r02/pcache2/on_$i.jsonl 2>gpurun_out/r02/pcache2/on_$i.err
  RL_P_CACHE=0 $B > gpurun_out/r02/pcache2/off_$i.jsonl 2>gpurun_out/r02/pcache2/off_$i.err
done
python tools/bench_summary.py gpurun_out/r02/pcache2/*.jsonl
