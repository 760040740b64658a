# Vocab-parallel split phases with the probability cache, after the workspace-size fix: the vocab-parallel
# and split tests on 4 GPUs, then glm64k vocab-parallel at N = 4 / 2 with the cache on / off.
set -x
D=gpurun_out/r02/vpcache2
mkdir -p $D
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "multi or nvls or split or vocab_parallel" 2>&1 | tail -5 > $D/gpu4_multi_suite.log
tail -2 $D/gpu4_multi_suite.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29511"
for n in 4 2; do
  timeout 900 $T --nproc-per-node $n bench.py --gpus $n --config glm64k --steps 10 --warmup 3 > $D/vp_n${n}_on.jsonl 2> $D/vp_n${n}_on.err
  RL_P_CACHE=0 timeout 900 $T --nproc-per-node $n bench.py --gpus $n --config glm64k --steps 10 --warmup 3 > $D/vp_n${n}_off.jsonl 2> $D/vp_n${n}_off.err
done
python tools/bench_summary.py $D/*.jsonl
