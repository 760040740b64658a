# Rotated K start per CTA pair (RL_KROT_<K> phases): K4 loses 11% of its cycles in the soft k-barrier's
# lockstep (99.9% tensor-active without it, at twice the DRAM reads); the guess is L2 hot spots when every
# pair reads the same k-slice of a shared block. Round 1 in order, round 2 reversed.
set -x
mkdir -p gpurun_out/r02/krot
run() { env $2 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/krot/$1.jsonl 2>/dev/null; }
CFGS="base:X=0 dz4:RL_KROT_DZ=4 dz8:RL_KROT_DZ=8 fwd8dz8:RL_KROT_DZ=8,RL_KROT_FWD=8 all8:RL_KROT=8"
for c in $CFGS; do n=${c%%:*}; e=${c#*:}; run ${n}_1 "${e//,/ }"; done
for c in $(echo $CFGS | tr ' ' '\n' | tac); do n=${c%%:*}; e=${c#*:}; run ${n}_2 "${e//,/ }"; done
for c in base:X=0 fwd8dz8:RL_KROT_DZ=8,RL_KROT_FWD=8; do n=${c%%:*}; e=${c#*:}
  env ${e//,/ } timeout 300 python tools/gemm_traffic.py > /dev/null 2>&1 && \
  env ${e//,/ } ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:gemm_kernel -s 4 -c 4 --csv --log-file gpurun_out/r02/krot/ncu_$n.csv python tools/gemm_traffic.py > /dev/null 2>&1
done
python tools/bench_summary.py gpurun_out/r02/krot/*.jsonl
