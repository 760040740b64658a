# K6 (dW) with 8 epilogue warps that release each TMEM half before storing (RL_EPI_WARPS_DW=8) vs 4: parity, ncu, bench A/B.
set -x
mkdir -p gpurun_out/r02/k6w8e
RL_EPI_WARPS_DW=8 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_bwd.py -q -p no:cacheprovider > gpurun_out/r02/k6w8e/parity.log 2>&1
for w in 4 8; do
  RL_EPI_WARPS_DW=$w timeout 300 python tools/gemm_traffic.py > /dev/null 2>&1 && \
  RL_EPI_WARPS_DW=$w ncu --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.max \
    --clock-control none -k regex:gemm_kernel -s 6 -c 1 --csv --log-file gpurun_out/r02/k6w8e/ncu_w$w.csv python tools/gemm_traffic.py > /dev/null 2>&1
done
run() { RL_EPI_WARPS_DW=$2 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/k6w8e/$1.jsonl 2>/dev/null; }
run w4_1 4; run w8_1 8; run w8_2 8; run w4_2 4
tail -n 1 gpurun_out/r02/k6w8e/parity.log
for w in 4 8; do grep -h "sm__\|Kernel" gpurun_out/r02/k6w8e/ncu_w$w.csv | awk -F'","' '{print "w'$w'", substr($5,1,40), $(NF-2), $NF}'; done
python tools/bench_summary.py gpurun_out/r02/k6w8e/*.jsonl
