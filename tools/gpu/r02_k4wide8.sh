# K4 on wide 256x512 tiles with 8 epilogue warps (RL_WIDE_DZ=1 RL_EPI_WARPS_DZ=8) vs the product's 256x256
# double-buffered K4: parity of the variant, ncu, alternating bench A/B (2 rounds, 2nd reversed).
set -x
mkdir -p gpurun_out/r02/k4wide8
RL_WIDE_DZ=1 RL_EPI_WARPS_DZ=8 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_bwd.py tests/test_gpu_kl_temperature.py -q -p no:cacheprovider > gpurun_out/r02/k4wide8/parity.log 2>&1
for v in base wide4 wide8; do
  case $v in base) e="X=0";; wide4) e="RL_WIDE_DZ=1";; wide8) e="RL_WIDE_DZ=1 RL_EPI_WARPS_DZ=8";; esac
  env $e timeout 300 python tools/gemm_traffic.py > /dev/null 2>&1 && \
  env $e ncu --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.max,dram__bytes_read.sum \
    --clock-control none -k regex:gemm_kernel -s 5 -c 1 --csv --log-file gpurun_out/r02/k4wide8/ncu_$v.csv python tools/gemm_traffic.py > /dev/null 2>&1
done
run() { env $2 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/k4wide8/$1.jsonl 2>/dev/null; }
run base_1 "X=0"; run wide8_1 "RL_WIDE_DZ=1 RL_EPI_WARPS_DZ=8"; run wide8_2 "RL_WIDE_DZ=1 RL_EPI_WARPS_DZ=8"; run base_2 "X=0"
tail -n 1 gpurun_out/r02/k4wide8/parity.log
for v in base wide4 wide8; do grep -h "sm__\|dram" gpurun_out/r02/k4wide8/ncu_$v.csv | awk -F'","' '{print "'$v'", $(NF-2), $NF}'; done
python tools/bench_summary.py gpurun_out/r02/k4wide8/*.jsonl
