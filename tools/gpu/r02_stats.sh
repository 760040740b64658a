set -x
mkdir -p gpurun_out/r02/stats
RL_LIBRARY=ab_libs/librl_stats.so timeout 300 python tools/gemm_stats.py > gpurun_out/r02/stats/gemm_stats.log 2>&1
RL_LIBRARY=ab_libs/librl_stats.so RL_SYNC_EVERY=0 timeout 300 python tools/gemm_stats.py > gpurun_out/r02/stats/gemm_stats_nosync.log 2>&1
RL_LIBRARY=ab_libs/librl_stats.so RL_WIDE_DZ=1 timeout 300 python tools/gemm_stats.py > gpurun_out/r02/stats/gemm_stats_widedz.log 2>&1
RL_LIBRARY=ab_libs/librl_stats.so RL_EPI_WARPS=4 timeout 300 python tools/gemm_stats.py > gpurun_out/r02/stats/gemm_stats_epi4.log 2>&1
tail -n 4 gpurun_out/r02/stats/*.log
