# Grid of the cache-fed K4 (RL_DZC_BLOCKS_PER_SM 4 / 8 default / 16), 2 alternating rounds.
set -x
D=gpurun_out/r02/dzc
mkdir -p $D
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
for i in 1 2; do
  for b in 8 4 16; do RL_DZC_BLOCKS_PER_SM=$b $B > $D/b${b}_$i.jsonl 2>/dev/null; done
done
for f in $D/*.jsonl; do python -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);k=d['kernels']['K4_dz_from_cache'];print('$f', round(d['ms_per_step'],2), round(k['avg_ms'],3), round(k['gbs']))"; done
