# (round 2, with the probability cache: K4 elementwise from K1s numerators)
# 4 GPUs of one box: the whole -m gpu suite (multi-GPU modules run at world size 4 and 2),
# then the scaling runs the driver does (N = 1, 2, 4 back to back, default config) and the
# vocab-parallel / stress configs at N = 4.
set -x
mkdir -p gpurun_out/r02/multi4_pc
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv
nvidia-smi topo -m > gpurun_out/r02/multi4_pc/topo.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider -k "multi or nvls or muon_dist or split" \
  > gpurun_out/r02/multi4_pc/gpu4_multi_suite.log 2>&1
tail -3 gpurun_out/r02/multi4_pc/gpu4_multi_suite.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29511"
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r02/multi4_pc/scale_n1.jsonl 2> gpurun_out/r02/multi4_pc/scale_n1.err
for n in 2 4; do
  timeout 900 $T --nproc-per-node $n bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/r02/multi4_pc/scale_n$n.jsonl 2> gpurun_out/r02/multi4_pc/scale_n$n.err
done
timeout 900 $T --nproc-per-node 4 bench.py --gpus 4 --config glm64k --steps 10 --warmup 3 > gpurun_out/r02/multi4_pc/vp_glm64k_n4.jsonl 2> gpurun_out/r02/multi4_pc/vp_glm64k_n4.err
timeout 900 $T --nproc-per-node 2 bench.py --gpus 2 --config glm64k --steps 10 --warmup 3 > gpurun_out/r02/multi4_pc/vp_glm64k_n2.jsonl 2> gpurun_out/r02/multi4_pc/vp_glm64k_n2.err
timeout 900 $T --nproc-per-node 4 bench.py --gpus 4 --config stress --steps 20 --warmup 3 > gpurun_out/r02/multi4_pc/stress_n4.jsonl 2> gpurun_out/r02/multi4_pc/stress_n4.err
python tools/bench_summary.py gpurun_out/r02/multi4_pc/*.jsonl
