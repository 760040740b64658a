# K1's cache stores through shared memory + TMA (RL_P_TMA=1, default) vs direct global stores:
# parity subset + poison test + the hostio equality, 3 alternating bench rounds, ncu cycles.
set -x
D=gpurun_out/r02/ptma
mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_workspace_poison.py tests/test_gpu_parity.py tests/test_gpu_sparse_bwd.py tests/test_gpu_kl_temperature.py tests/test_gpu_fullsize.py -q -p no:cacheprovider 2>&1 | tail -3 > $D/parity.log
cat $D/parity.log
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
for i in 1 2 3; do
  $B > $D/tma_$i.jsonl 2>/dev/null
  RL_P_TMA=0 $B > $D/direct_$i.jsonl 2>/dev/null
done
python tools/bench_summary.py $D/*.jsonl
timeout 300 python tools/step_traffic.py > $D/step_traffic_plain.log 2>&1 && \
for v in 1 0; do
  RL_P_TMA=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.max \
    --clock-control none -k regex:"gemm_kernel|dz_from_cache" -s 5 -c 4 --csv --log-file $D/ncu_tma$v.csv python tools/step_traffic.py > $D/ncu_tma$v.log 2>&1
done
