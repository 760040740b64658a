# Final round-2 validation on one B200: the whole -m gpu suite + smoke, the default bench line, the
# launch list of the same bench command, and one ncu --set full capture of the four step GEMMs.
set -x
mkdir -p gpurun_out/r02/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/r02/final/gpu1_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/final/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02/final/bench_n1.jsonl 2> gpurun_out/r02/final/bench_n1.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/final/plain_for_ncu.jsonl 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/final/ncu_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/final/ncu_launches.log 2>&1
timeout 300 python tools/gemm_traffic.py > gpurun_out/r02/final/gemm_traffic_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 4 -c 4 \
  -o gpurun_out/r02/final/gemms_full python tools/gemm_traffic.py > gpurun_out/r02/final/ncu_full.log 2>&1
tail -3 gpurun_out/r02/final/gpu1_suite.log gpurun_out/r02/final/smoke.log
python tools/bench_summary.py gpurun_out/r02/final/bench_n1.jsonl
