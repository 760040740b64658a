# K1: half 1 loaded between the two halves of half 0 arithmetic (product now) vs the previous product.
# arithmetic under the next MMAs (product now) vs the previous product (ab_libs/librl_prev.so).
set -x
mkdir -p gpurun_out/r02/k1inter
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl_temperature.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "not variants and not hostio" > gpurun_out/r02/k1inter/parity.log 2>&1
RL_EPI_WARPS_FWD=16 timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/r02/k1inter/parity16.log 2>&1
for v in prev prod; do
  lib=""; [ $v != prod ] && lib=ab_libs/librl_$v.so
  RL_LIBRARY=$lib timeout 300 python tools/gemm_traffic.py > /dev/null 2>&1 && \
  RL_LIBRARY=$lib ncu --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.max \
    --clock-control none -k regex:gemm_kernel -s 4 -c 1 --csv --log-file gpurun_out/r02/k1inter/ncu_$v.csv python tools/gemm_traffic.py > /dev/null 2>&1
done
RL_LIBRARY=ab_libs/librl_stats.so timeout 300 python tools/gemm_stats.py > gpurun_out/r02/k1inter/stats_prod.log 2>&1
run() { RL_LIBRARY=$2 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/k1inter/$1.jsonl 2>/dev/null; }
run prev_1 ab_libs/librl_prev.so; run prod_1 ""; run prod_2 ""; run prev_2 ab_libs/librl_prev.so
tail -n 1 gpurun_out/r02/k1inter/parity*.log
for v in prev prod; do grep -h "sm__" gpurun_out/r02/k1inter/ncu_$v.csv | awk -F'","' '{print "'$v'", $(NF-2), $NF}'; done
grep -h "^K1" gpurun_out/r02/k1inter/stats_prod.log
python tools/bench_summary.py gpurun_out/r02/k1inter/*.jsonl
