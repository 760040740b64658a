# K4's soft k-barrier: the cycle counters show K4 at the MMA floor without it (32.8k cycles per tile vs
# 39.2k with it) while the barrier keeps its DRAM reads (and the power-capped clock) in check.
# Sweep the lead it allows (RL_SYNC_SLACK_DZ) and its interval (RL_SYNC_EVERY_DZ), 2 rounds.
set -x
mkdir -p gpurun_out/r02/k4sync
for i in 1 2; do
  for cfg in "2 32" "4 32" "8 32" "16 32" "4 64" "8 64" "0 0"; do
    set -- $cfg
    RL_SYNC_SLACK_DZ=$1 RL_SYNC_EVERY_DZ=$2 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/r02/k4sync/s$1_e$2_$i.jsonl 2>/dev/null
  done
done
for cfg in "2 32" "8 32" "8 64" "0 0"; do
  set -- $cfg
  RL_SYNC_SLACK_DZ=$1 RL_SYNC_EVERY_DZ=$2 timeout 300 python tools/gemm_traffic.py > /dev/null 2>&1 && \
  RL_SYNC_SLACK_DZ=$1 RL_SYNC_EVERY_DZ=$2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:gemm_kernel -s 4 -c 4 --csv --log-file gpurun_out/r02/k4sync/ncu_s$1_e$2.csv python tools/gemm_traffic.py > /dev/null 2>&1
done
python tools/bench_summary.py gpurun_out/r02/k4sync/*.jsonl
