# K4 on wide 256x512 tiles with 8 epilogue warps, now in dynamic tile order (the default order
# for K4), vs the default 256x256 K4: parity of the variant, 3 alternating bench rounds, ncu.
set -x
mkdir -p gpurun_out/r02/k4wide8_dyn
W="RL_WIDE_DZ=1 RL_EPI_WARPS_DZ=8"
env $W timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_bwd.py -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/r02/k4wide8_dyn/parity.log
run() { env $2 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/k4wide8_dyn/$1.jsonl 2>/dev/null; }
for i in 1 2 3; do run base_$i "X=0"; run wide8_$i "$W"; done
for v in base wide8; do
  e="X=0"; [ $v = wide8 ] && e="$W"
  env $e ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.max \
    --clock-control none -k regex:gemm_kernel -s 4 -c 4 --csv --log-file gpurun_out/r02/k4wide8_dyn/ncu_$v.csv python tools/gemm_traffic.py > /dev/null 2>&1
done
cat gpurun_out/r02/k4wide8_dyn/parity.log
python tools/bench_summary.py gpurun_out/r02/k4wide8_dyn/*.jsonl
