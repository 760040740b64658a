# K1's probability-cache stores with an L2 evict-first policy (RL_P_EVICT=1, default) vs plain stores:
# parity subset, 3 alternating bench rounds, ncu DRAM per kernel of the fused step for both, and one
# ncu --set full capture of the fused step's K1 / K4 / K6 / K5 (tools/step_traffic.py).
set -x
D=gpurun_out/r02/pevict
mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_workspace_poison.py tests/test_gpu_parity.py tests/test_gpu_sparse_bwd.py -q -p no:cacheprovider 2>&1 | tail -3 > $D/parity.log
cat $D/parity.log
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
for i in 1 2 3; do
  $B > $D/evict_$i.jsonl 2>/dev/null
  RL_P_EVICT=0 $B > $D/plain_$i.jsonl 2>/dev/null
done
python tools/bench_summary.py $D/*.jsonl
timeout 300 python tools/step_traffic.py > $D/step_traffic_plain.log 2>&1 && \
for v in 1 0; do
  RL_P_EVICT=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.max \
    --clock-control none -k regex:"gemm_kernel|dz_from_cache" -s 5 -c 4 --csv --log-file $D/ncu_evict$v.csv python tools/step_traffic.py > $D/ncu_evict$v.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|dz_from_cache" -s 5 -c 4 \
  -o $D/step_full python tools/step_traffic.py > $D/ncu_full.log 2>&1
cat $D/step_traffic_plain.log
