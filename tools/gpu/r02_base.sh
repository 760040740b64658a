# Round-2 baseline on one B200: full -m gpu suite + smoke, default bench, K1 epilogue-warps A/B
# (RL_EPI_WARPS=4 vs the default 8, alternating), launch list, one full ncu capture of the four GEMMs.
set -x
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -s -p no:cacheprovider 2>&1 | tail -80 > gpurun_out/r02/gpu1_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02/bench_n1.jsonl 2> gpurun_out/r02/bench_n1.err
for i in 1 2; do
  RL_EPI_WARPS=4 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/ab_epi4_$i.jsonl 2>/dev/null
  RL_EPI_WARPS=8 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/ab_epi8_$i.jsonl 2>/dev/null
done
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/plain_for_ncu.jsonl 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/ncu_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/ncu_launches.log 2>&1
timeout 300 python tools/gemm_traffic.py > gpurun_out/r02/gemm_traffic_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 4 -c 4 \
  -o gpurun_out/r02/gemms_full python tools/gemm_traffic.py > gpurun_out/r02/ncu_full.log 2>&1
tail -3 gpurun_out/r02/gpu1_suite.log gpurun_out/r02/smoke.log; head -c 400 gpurun_out/r02/bench_n1.jsonl
