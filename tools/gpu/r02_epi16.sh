# K1 with 16 epilogue warps (four per TMEM lane quarter, 64 columns of a half each) vs 8, alternating,
# plus parity of the 16-warp build and its ncu tensor activity.
set -x
mkdir -p gpurun_out/r02/epi16
for i in 1 2; do
  for w in 8 16; do RL_EPI_WARPS_FWD=$w timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/epi16/w${w}_$i.jsonl 2>/dev/null; done
done
RL_EPI_WARPS_FWD=16 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kl_temperature.py -q -p no:cacheprovider > gpurun_out/r02/epi16/parity16.log 2>&1
for w in 8 16; do
  RL_EPI_WARPS_FWD=$w timeout 300 python tools/gemm_traffic.py > /dev/null 2>&1 && \
  RL_EPI_WARPS_FWD=$w ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.max \
    --clock-control none -k regex:gemm_kernel -s 4 -c 1 --csv --log-file gpurun_out/r02/epi16/ncu_w$w.csv python tools/gemm_traffic.py > /dev/null 2>&1
done
python tools/bench_summary.py gpurun_out/r02/epi16/*.jsonl
tail -n 2 gpurun_out/r02/epi16/parity16.log
grep -h "sm__" gpurun_out/r02/epi16/ncu_w*.csv | cut -c1-40,150-
