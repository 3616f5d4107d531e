for rep in 1 2; do
for E in "S2_PDL=1" "S2_PDL=0"; do
env $E timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-hybrid --no-decode --no-configs 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$E bench ms', round(d['ms_per_step'],3), {k: round(v['avg_ms'],3) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
done
