# Probability cache with the row-group K4 kernel: parity subset + poison tests, 3 bench rounds, ncu of K4'.
set -x
mkdir -p gpurun_out/r02/pcache4
timeout 1500 python -m pytest tests/test_gpu_workspace_poison.py tests/test_gpu_parity.py tests/test_gpu_sparse_bwd.py tests/test_gpu_kl_temperature.py -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/r02/pcache4/parity.log
cat gpurun_out/r02/pcache4/parity.log
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
for i in 1 2 3; do
  $B > gpurun_out/r02/pcache4/on_$i.jsonl 2>gpurun_out/r02/pcache4/on_$i.err
done
python tools/bench_summary.py gpurun_out/r02/pcache4/*.jsonl
timeout 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
  --clock-control none -k regex:"gemm_kernel|dz_from_cache" -c 12 --csv --log-file gpurun_out/r02/pcache4/ncu.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/pcache4/ncu.log 2>&1
