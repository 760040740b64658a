# Dynamic tile order, round 2: K4 dynamic by default; K1 dynamic too (RL_DYN_TILES_FWD=1), and
# larger raster groups for K1 / K4 now that the pairs cannot drift apart. Parity with every
# GEMM dynamic (K1 included), the step A/B over 3 alternating rounds, ncu per GEMM.
set -x
mkdir -p gpurun_out/r02/dyn2
RL_DYN_TILES=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_bwd.py tests/test_gpu_kl_temperature.py -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r02/dyn2/parity_dyn_all.log
tail -3 gpurun_out/r02/dyn2/parity_dyn_all.log
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
for i in 1 2 3; do
  $B > gpurun_out/r02/dyn2/dz_$i.jsonl 2>/dev/null
  RL_DYN_TILES_DZ=0 $B > gpurun_out/r02/dyn2/static_$i.jsonl 2>/dev/null
  RL_DYN_TILES_FWD=1 $B > gpurun_out/r02/dyn2/fwd_dz_$i.jsonl 2>/dev/null
  RL_GROUP_M_DZ=32 $B > gpurun_out/r02/dyn2/dz_g32_$i.jsonl 2>/dev/null
  RL_DYN_TILES_FWD=1 RL_GROUP_M_FWD=32 RL_GROUP_M_DZ=32 $B > gpurun_out/r02/dyn2/fwd_dz_g32_$i.jsonl 2>/dev/null
done
python tools/bench_summary.py gpurun_out/r02/dyn2/*.jsonl
for v in dz fwd_dz; do
  f=0; [ $v = fwd_dz ] && f=1
  RL_DYN_TILES_FWD=$f ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:gemm_kernel -c 16 --csv --log-file gpurun_out/r02/dyn2/ncu_$v.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/dyn2/ncu_$v.log 2>&1
done
RL_GROUP_M_DZ=32 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:gemm_kernel -c 16 --csv --log-file gpurun_out/r02/dyn2/ncu_dz_g32.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/dyn2/ncu_dz_g32.log 2>&1
