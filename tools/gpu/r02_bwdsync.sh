# K5 / K6 soft k-barrier re-tuned now that K1 / K4 run in the dynamic order: window (RL_SYNC_EVERY_DH/DW)
# and lead (RL_SYNC_SLACK_DH/DW), 3 alternating rounds of the default step.
set -x
mkdir -p gpurun_out/r02/bwdsync
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
for i in 1 2 3; do
  $B > gpurun_out/r02/bwdsync/default_$i.jsonl 2>/dev/null
  RL_SYNC_SLACK_DH=4 RL_SYNC_SLACK_DW=4 $B > gpurun_out/r02/bwdsync/slack4_$i.jsonl 2>/dev/null
  RL_SYNC_SLACK_DH=1 RL_SYNC_SLACK_DW=1 $B > gpurun_out/r02/bwdsync/slack1_$i.jsonl 2>/dev/null
  RL_SYNC_EVERY_DH=8 RL_SYNC_EVERY_DW=8 $B > gpurun_out/r02/bwdsync/every8_$i.jsonl 2>/dev/null
  RL_SYNC_EVERY_DH=32 RL_SYNC_EVERY_DW=32 $B > gpurun_out/r02/bwdsync/every32_$i.jsonl 2>/dev/null
done
python tools/bench_summary.py gpurun_out/r02/bwdsync/*.jsonl
