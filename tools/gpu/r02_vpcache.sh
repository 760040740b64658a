# The whole -m gpu suite on 4 GPUs (single- and multi-GPU modules), smoke, the default bench line, then
# vocab-parallel split phases with the probability cache (rl_fwd_partials_ex(RL_FWD_CACHE) +
# rl_bwd_ex(RL_BWD_FROM_CACHE)): the multi-GPU tests on 4 GPUs, the single-GPU split-phase test, and
# glm64k vocab-parallel at N = 4 / 2 with the cache on / off.
set -x
D=gpurun_out/r02/vpcache
mkdir -p $D
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > $D/gpu4_all_suite.log
tail -2 $D/gpu4_all_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > $D/bench_n1.jsonl 2> $D/bench_n1.err
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29511"
for n in 4 2; do
  timeout 900 $T --nproc-per-node $n bench.py --gpus $n --config glm64k --steps 10 --warmup 3 > $D/vp_n${n}_on.jsonl 2> $D/vp_n${n}_on.err
  RL_P_CACHE=0 timeout 900 $T --nproc-per-node $n bench.py --gpus $n --config glm64k --steps 10 --warmup 3 > $D/vp_n${n}_off.jsonl 2> $D/vp_n${n}_off.err
done
python tools/bench_summary.py $D/*.jsonl
