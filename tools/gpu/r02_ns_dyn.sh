# Newton-Schulz (Muon, f3) GEMMs in dynamic tile order (RL_DYN_TILES_NS=1) vs the static
# order + k-barrier, 3 alternating rounds of tools/bench_muon.py, then the Muon parity tests.
set -x
mkdir -p gpurun_out/r02/ns_dyn
for i in 1 2 3; do
  RL_DYN_TILES_NS=0 timeout 300 python tools/bench_muon.py > gpurun_out/r02/ns_dyn/static_$i.log 2>&1
  RL_DYN_TILES_NS=1 timeout 300 python tools/bench_muon.py > gpurun_out/r02/ns_dyn/dyn_$i.log 2>&1
done
RL_DYN_TILES_NS=1 timeout 900 python -m pytest tests/test_gpu_muon.py -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/r02/ns_dyn/muon_parity_dyn.log
grep -h librl_ms gpurun_out/r02/ns_dyn/*.log
