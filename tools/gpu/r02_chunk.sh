# dU chunk rows at glm16k (K6's hidden rows per pass: 16k = 134 MB does not fit L2 beside the
# dU stream, 8k = 67 MB might): step A/B over 3 alternating rounds, DRAM bytes per GEMM launch.
set -x
mkdir -p gpurun_out/r02/chunk
for i in 1 2 3; do
  for c in 0 8192 4096; do
    timeout 300 python bench.py --dz-chunk $c --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/chunk/c${c}_$i.jsonl 2>/dev/null
  done
done
for c in 0 8192; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:gemm_kernel -c 40 --csv --log-file gpurun_out/r02/chunk/ncu_c$c.csv \
    python bench.py --dz-chunk $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/chunk/ncu_c$c.log 2>&1
done
python tools/bench_summary.py gpurun_out/r02/chunk/*.jsonl
