for r in 1 2; do
timeout 200 python tools/perf_dense.py
S2_DQ_V2=1 timeout 200 python tools/perf_dense.py
done
S2_DQ_V2=1 N=8192 timeout 200 python tools/perf_dense.py
N=8192 timeout 200 python tools/perf_dense.py
