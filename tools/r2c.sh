for rep in 1 2; do
for G in "S2_DKV_GROUP=0" "S2_X=1"; do
 echo "== $G cfg3"; env $G timeout 120 python tools/perf_bwd.py --uniform 2>&1 | tail -1
 echo "== $G cfg2"; env $G timeout 120 python tools/perf_bwd.py --uniform --b 4 --n 8192 2>&1 | tail -1
 echo "== $G cfg5"; env $G timeout 300 python tools/perf_bwd.py --uniform --n 131072 --iters 3 2>&1 | tail -1
done
done
