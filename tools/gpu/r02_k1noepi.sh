# Is K1's ~9% loss in the MMA loop or in the drain? K1 with an epilogue that releases TMEM without
# reading it (A/B build -DRL_AB_K1_NOEPI), ncu cycles + cycle counters, vs the product.
set -x
mkdir -p gpurun_out/r02/k1noepi
for v in prod k1noepi k1nomath; do
  lib=""; [ $v != prod ] && lib=ab_libs/librl_$v.so
  RL_LIBRARY=$lib timeout 300 python tools/gemm_traffic.py > /dev/null 2>&1 && \
  RL_LIBRARY=$lib ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.max,dram__bytes_read.sum \
    --clock-control none -k regex:gemm_kernel -s 4 -c 1 --csv --log-file gpurun_out/r02/k1noepi/ncu_$v.csv python tools/gemm_traffic.py > /dev/null 2>&1
done
RL_LIBRARY=ab_libs/librl_stats.so timeout 300 python tools/gemm_stats.py > gpurun_out/r02/k1noepi/stats_prod.log 2>&1
RL_LIBRARY=ab_libs/librl_stats_k1noepi.so timeout 300 python tools/gemm_stats.py > gpurun_out/r02/k1noepi/stats_k1noepi.log 2>&1
RL_LIBRARY=ab_libs/librl_stats_k1nomath.so timeout 300 python tools/gemm_stats.py > gpurun_out/r02/k1noepi/stats_k1nomath.log 2>&1
for v in prod k1noepi k1nomath; do grep -h "sm__\|gpu__\|dram" gpurun_out/r02/k1noepi/ncu_$v.csv | awk -F'","' '{print "'$v'", $(NF-2), $NF}'; done
grep -h "^K1" gpurun_out/r02/k1noepi/stats_*.log
