mkdir -p gpurun_out
timeout 120 python tools/trace_fwd2.py 2>&1 | tail -20
timeout 600 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_edges.py tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for E in "S2_FWD_2CTA=0" "S2_FWD_2CTA=1"; do echo "== $E"; env $E timeout 120 python tools/perf_fwd.py 2>&1 | tail -1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pair2 -c 1 -o gpurun_out/p2_full -f python tools/perf_fwd.py --iters 1 > gpurun_out/p2_ncu.log 2>&1; echo "ncu rc=$?"
