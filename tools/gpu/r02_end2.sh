# End-of-round check on one GPU with the final build: the whole -m gpu suite, smoke, the default bench line.
set -x
D=gpurun_out/r02/end2
mkdir -p $D
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -20 > $D/gpu1_suite.log
tail -2 $D/gpu1_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
tail -1 $D/smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > $D/bench_n1.jsonl 2> $D/bench_n1.err
python tools/bench_summary.py $D/bench_n1.jsonl
