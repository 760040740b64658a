# K1's LSE epilogue with part of its exponentials on the FMA pipe (RL_LSE_POLY_EVERY = k: every k-th),
# alternating A/B (round 1 in order, round 2 reversed), cycle counters, parity of the poly4 build,
# and the new H = 8192 / C-ABI tests on the product build.
set -x
mkdir -p gpurun_out/r02/poly
run() { RL_LIBRARY=$2 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/poly/$1.jsonl 2>/dev/null; }
for v in base poly8 poly4 poly3; do lib=""; [ $v != base ] && lib=ab_libs/librl_$v.so; run ${v}_1 "$lib"; done
for v in poly3 poly4 poly8 base; do lib=""; [ $v != base ] && lib=ab_libs/librl_$v.so; run ${v}_2 "$lib"; done
RL_LIBRARY=ab_libs/librl_stats.so timeout 300 python tools/gemm_stats.py > gpurun_out/r02/poly/stats_base.log 2>&1
RL_LIBRARY=ab_libs/librl_stats_poly4.so timeout 300 python tools/gemm_stats.py > gpurun_out/r02/poly/stats_poly4.log 2>&1
RL_LIBRARY=ab_libs/librl_poly4.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -p no:cacheprovider -k "sampled or ragged or tiny" > gpurun_out/r02/poly/parity_poly4.log 2>&1
timeout 900 python -m pytest tests/test_c_abi_example.py tests/test_gpu_parity.py -q -s -p no:cacheprovider -k "example or 8192" > gpurun_out/r02/poly/new_tests.log 2>&1
python tools/bench_summary.py gpurun_out/r02/poly/*.jsonl
grep "^K1" gpurun_out/r02/poly/stats_*.log
tail -2 gpurun_out/r02/poly/parity_poly4.log gpurun_out/r02/poly/new_tests.log
