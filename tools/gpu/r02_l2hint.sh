# K1 / K4 with L2 eviction hints (hidden rows evict_last, W evict_first) and larger raster groups:
# DRAM per launch (ncu) and bench A/B (round 2 in reverse order).
set -x
mkdir -p gpurun_out/r02/l2hint
CFGS="base:X=0 h16:RL_L2HINT_FWD=1,RL_L2HINT_DZ=1 h32:RL_L2HINT_FWD=1,RL_L2HINT_DZ=1,RL_GROUP_M_FWD=32,RL_GROUP_M_DZ=32 h24:RL_L2HINT_FWD=1,RL_L2HINT_DZ=1,RL_GROUP_M_FWD=24,RL_GROUP_M_DZ=24"
for c in $CFGS; do n=${c%%:*}; e=${c#*:}; e=${e//,/ }
  env $e timeout 300 python tools/gemm_traffic.py > /dev/null 2>&1 && \
  env $e ncu --metrics dram__bytes_read.sum,sm__cycles_elapsed.max --clock-control none -k regex:gemm_kernel -s 4 -c 2 --csv \
    --log-file gpurun_out/r02/l2hint/ncu_$n.csv python tools/gemm_traffic.py > /dev/null 2>&1
done
run() { env $2 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/l2hint/$1.jsonl 2>/dev/null; }
for c in $CFGS; do n=${c%%:*}; e=${c#*:}; run ${n}_1 "${e//,/ }"; done
for c in $(echo $CFGS | tr ' ' '\n' | tac); do n=${c%%:*}; e=${c#*:}; run ${n}_2 "${e//,/ }"; done
for n in base h16 h32 h24; do grep -h "dram\|sm__" gpurun_out/r02/l2hint/ncu_$n.csv | awk -F'","' '{print "'$n'", substr($5,1,28), $(NF-2), $NF}'; done
python tools/bench_summary.py gpurun_out/r02/l2hint/*.jsonl
