set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r02_gpu1.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r02_gpu1.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench1.json 2> gpurun_out/r02_bench1.err
tail -3 gpurun_out/r02_gpu1.log; cat gpurun_out/r02_bench1.json | head -c 600
