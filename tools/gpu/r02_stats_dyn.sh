# Per-role cycle counters of the four step GEMMs with K1 / K4 in dynamic tile order (default)
# and with every GEMM static (RL_DYN_TILES=0), RL_AB_STATS build.
set -x
mkdir -p gpurun_out/r02/stats_dyn
RL_LIBRARY=ab_libs/librl_stats.so timeout 300 python tools/gemm_stats.py > gpurun_out/r02/stats_dyn/gemm_stats_default.log 2>&1
RL_LIBRARY=ab_libs/librl_stats.so RL_DYN_TILES=0 timeout 300 python tools/gemm_stats.py > gpurun_out/r02/stats_dyn/gemm_stats_static.log 2>&1
tail -n 5 gpurun_out/r02/stats_dyn/*.log
