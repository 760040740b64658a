# Last validation of the round on 4 GPUs of one box: the whole -m gpu suite (single-GPU modules plus the
# multi-GPU ones at world size 4 and 2), smoke, the default bench line with e2e and cpu_baseline, the
# scaling runs N = 1 / 2 / 4 back to back, every config at N = 1 and the multi-GPU configs at N = 4.
set -x
D=gpurun_out/r02/last4
mkdir -p $D
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > $D/gpu4_all_suite.log
tail -3 $D/gpu4_all_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29511"
timeout 600 python bench.py --steps 20 --warmup 3 > $D/scale_n1.jsonl 2> $D/scale_n1.err
for n in 2 4; do
  timeout 900 $T --nproc-per-node $n bench.py --gpus $n --steps 20 --warmup 3 > $D/scale_n$n.jsonl 2> $D/scale_n$n.err
done
for c in small glm64k stress; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $D/n1_$c.jsonl 2> $D/n1_$c.err
done
timeout 900 $T --nproc-per-node 4 bench.py --gpus 4 --config glm64k --steps 10 --warmup 3 > $D/vp_glm64k_n4.jsonl 2> $D/vp_glm64k_n4.err
timeout 900 $T --nproc-per-node 4 bench.py --gpus 4 --config stress --steps 20 --warmup 3 > $D/stress_n4.jsonl 2> $D/stress_n4.err
python tools/bench_summary.py $D/*.jsonl
