# Newton-Schulz raster group (RL_GROUP_M_NS, now wired to every NS GEMM launch), 2 rounds
set -x
mkdir -p gpurun_out/r02/nsgroup
for i in 1 2; do for g in 2 4 8 16; do
  RL_GROUP_M_NS=$g timeout 300 python tools/bench_muon.py > gpurun_out/r02/nsgroup/g${g}_$i.log 2>&1
done; done
grep -h librl_ms gpurun_out/r02/nsgroup/*.log | cut -c1-120
