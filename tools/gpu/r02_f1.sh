# SURVEY §8(f)1 measured: how much could removing the backward's dU HBM round trip gain?
# Upper-bound variants (A/B libraries, garbage outputs, timing only):
#   k4nostore: K4 computes dU but never writes it
#   dufree:    K4 never writes dU AND K5/K6 read dU from a 256-row window resident in L2
# alternated with the product library, 3 rounds; then per-GEMM DRAM bytes of each.
set -x
mkdir -p gpurun_out/r02/f1
timeout 900 python -m pytest tests/test_gpu_artifact.py -q -s -p no:cacheprovider > gpurun_out/r02/f1/artifact_test.log 2>&1
for i in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/f1/prod_$i.jsonl 2>/dev/null
  RL_LIBRARY=ab_libs/librl_dufree.so timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/f1/dufree_$i.jsonl 2>/dev/null
  RL_LIBRARY=ab_libs/librl_k4nostore.so timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/f1/k4nostore_$i.jsonl 2>/dev/null
done
for v in prod dufree k4nostore; do
  lib=""; [ $v != prod ] && lib=ab_libs/librl_$v.so
  RL_LIBRARY=$lib timeout 300 python tools/gemm_traffic.py > gpurun_out/r02/f1/plain_$v.log 2>&1 && \
  RL_LIBRARY=$lib ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:gemm_kernel -s 4 -c 4 --csv --log-file gpurun_out/r02/f1/ncu_$v.csv python tools/gemm_traffic.py > gpurun_out/r02/f1/ncu_$v.log 2>&1
done
python tools/bench_summary.py gpurun_out/r02/f1/*.jsonl 2>&1 | tail -20
