# Final round-2 validation with the probability cache and the TMA-staged cache stores: the whole -m gpu
# suite + smoke, the default bench line, every BASELINE config and the reference arm, the launch
# list of the bench command and one ncu --set full capture of the four step GEMMs.
set -x
D=gpurun_out/r02/final4
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -40 > $D/gpu1_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > $D/bench_n1.jsonl 2> $D/bench_n1.err
for c in small glm64k stress; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $D/n1_$c.jsonl 2> $D/n1_$c.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $D/reference.jsonl 2> $D/reference.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $D/plain_for_ncu.jsonl 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/ncu_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $D/ncu_launches.log 2>&1
timeout 300 python tools/step_traffic.py > $D/step_traffic_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|dz_from_cache" -s 5 -c 4 \
  -o $D/gemms_full python tools/step_traffic.py > $D/ncu_full.log 2>&1
tail -3 $D/gpu1_suite.log $D/smoke.log
python tools/bench_summary.py $D/*.jsonl
