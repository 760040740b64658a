# Dynamic tile order (RL_DYN_TILES[_<K>]): parity with it on for every store GEMM, then the
# step A/B (default = static round robin + soft k-barrier) over 3 alternating rounds, and
# the DRAM bytes / tensor activity per GEMM launch.
set -x
mkdir -p gpurun_out/r02/dyn
RL_DYN_TILES=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_bwd.py tests/test_gpu_muon.py -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r02/dyn/parity_dyn.log
tail -3 gpurun_out/r02/dyn/parity_dyn.log
for i in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/dyn/base_$i.jsonl 2>/dev/null
  RL_DYN_TILES_DZ=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/dyn/dz_$i.jsonl 2>/dev/null
  RL_DYN_TILES=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/dyn/all_$i.jsonl 2>/dev/null
done
python tools/bench_summary.py gpurun_out/r02/dyn/*.jsonl
for v in base all; do
  e=0; [ $v = all ] && e=1
  RL_DYN_TILES=$e ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:gemm_kernel -c 16 --csv --log-file gpurun_out/r02/dyn/ncu_$v.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/dyn/ncu_$v.log 2>&1
done
