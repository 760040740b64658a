# K4 (and K1) with the k order rotated inside each soft-barrier window (RL_KWROT_<K> phases):
# ncu cycles / DRAM and bench A/B (round 2 reversed).
set -x
mkdir -p gpurun_out/r02/kwrot
CFGS="base:X=0 dz2:RL_KWROT_DZ=2 dz4:RL_KWROT_DZ=4 both4:RL_KWROT_DZ=4,RL_KWROT_FWD=4"
for c in $CFGS; do n=${c%%:*}; e=${c#*:}; e=${e//,/ }
  env $e timeout 300 python tools/gemm_traffic.py > /dev/null 2>&1 && \
  env $e ncu --metrics dram__bytes_read.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel -s 4 -c 2 --csv \
    --log-file gpurun_out/r02/kwrot/ncu_$n.csv python tools/gemm_traffic.py > /dev/null 2>&1
done
run() { env $2 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02/kwrot/$1.jsonl 2>/dev/null; }
for c in $CFGS; do n=${c%%:*}; e=${c#*:}; run ${n}_1 "${e//,/ }"; done
for c in $(echo $CFGS | tr ' ' '\n' | tac); do n=${c%%:*}; e=${c#*:}; run ${n}_2 "${e//,/ }"; done
for n in base dz2 dz4 both4; do grep -h "dram\|sm__" gpurun_out/r02/kwrot/ncu_$n.csv | awk -F'","' '{print "'$n'", substr($5,1,28), $(NF-2), $NF}'; done
python tools/bench_summary.py gpurun_out/r02/kwrot/*.jsonl
