# Serpentine K order for K6 / NS (RL_SERPENTINE): A/B against RL_SERPENTINE=0 (3 alternating
# pairs), DRAM bytes per GEMM of both, then the 1-GPU -m gpu suite with the new default.
set -x
mkdir -p gpurun_out/r02/serp
for i in 1 2 3; do
  RL_SERPENTINE=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/serp/off_$i.jsonl 2>/dev/null
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/serp/on_$i.jsonl 2>/dev/null
done
RL_SERPENTINE=1 RL_SERPENTINE_DH=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/serp/on_dh_1.jsonl 2>/dev/null
for v in off on; do
  s=1; [ $v = off ] && s=0
  RL_SERPENTINE=$s timeout 300 python tools/gemm_traffic.py > gpurun_out/r02/serp/plain_$v.log 2>&1 && \
  RL_SERPENTINE=$s ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:gemm_kernel -s 4 -c 4 --csv --log-file gpurun_out/r02/serp/ncu_$v.csv python tools/gemm_traffic.py > gpurun_out/r02/serp/ncu_$v.log 2>&1
done
timeout 300 python tools/bench_muon.py > gpurun_out/r02/serp/muon_on.log 2>&1
RL_SERPENTINE=0 timeout 300 python tools/bench_muon.py > gpurun_out/r02/serp/muon_off.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/r02/serp/gpu1_suite.log
python tools/bench_summary.py gpurun_out/r02/serp/*.jsonl
tail -3 gpurun_out/r02/serp/gpu1_suite.log
