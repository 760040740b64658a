# K1 drain: scale folded into one FFMA (product now) and every k-th exponential on the FMA pipe
# (A/B builds fastp{3,4,8}): parity, ncu cycles, cycle counters, bench A/B (2 rounds, 2nd reversed).
set -x
mkdir -p gpurun_out/r02/k1fast
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl_temperature.py -q -p no:cacheprovider > gpurun_out/r02/k1fast/parity_prod.log 2>&1
RL_LIBRARY=ab_libs/librl_fastp4.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl_temperature.py -q -p no:cacheprovider > gpurun_out/r02/k1fast/parity_fastp4.log 2>&1
for v in prod fastp3 fastp4 fastp8; do
  lib=""; [ $v != prod ] && lib=ab_libs/librl_$v.so
  RL_LIBRARY=$lib timeout 300 python tools/gemm_traffic.py > /dev/null 2>&1 && \
  RL_LIBRARY=$lib ncu --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.max \
    --clock-control none -k regex:gemm_kernel -s 4 -c 1 --csv --log-file gpurun_out/r02/k1fast/ncu_$v.csv python tools/gemm_traffic.py > /dev/null 2>&1
done
RL_LIBRARY=ab_libs/librl_stats.so timeout 300 python tools/gemm_stats.py > gpurun_out/r02/k1fast/stats_prod.log 2>&1
RL_LIBRARY=ab_libs/librl_stats_fastp4.so timeout 300 python tools/gemm_stats.py > gpurun_out/r02/k1fast/stats_fastp4.log 2>&1
run() { RL_LIBRARY=$2 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/k1fast/$1.jsonl 2>/dev/null; }
for v in prod fastp4 fastp8; do lib=""; [ $v != prod ] && lib=ab_libs/librl_$v.so; run ${v}_1 "$lib"; done
for v in fastp8 fastp4 prod; do lib=""; [ $v != prod ] && lib=ab_libs/librl_$v.so; run ${v}_2 "$lib"; done
tail -n 1 gpurun_out/r02/k1fast/parity_*.log
for v in prod fastp3 fastp4 fastp8; do grep -h "sm__" gpurun_out/r02/k1fast/ncu_$v.csv | awk -F'","' '{print "'$v'", $(NF-2), $NF}'; done
grep -h "^K1" gpurun_out/r02/k1fast/stats_*.log
python tools/bench_summary.py gpurun_out/r02/k1fast/*.jsonl
