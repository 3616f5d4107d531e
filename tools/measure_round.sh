#!/bin/bash
# One measurement session on the GPU box (profiles/rXX_*):
#   gpurun -- 'bash tools/measure_round.sh r1h'
# GPU test suite, bench line, cold launch list, selftest grid, and one ncu --set full
# capture of the four training-step kernels plus the decode kernel.
TAG=${1:-rX}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1
echo "gpu tests rc=$?"; tail -3 gpurun_out/gpu_tests_$TAG.log
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; tail -c 600 gpurun_out/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e \
  --no-cpu-baseline --no-hybrid --no-decode --no-configs > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launches rc=$?"
timeout 600 python tests/selftest.py --csv gpurun_out/selftest_$TAG.csv > gpurun_out/selftest_$TAG.log 2>&1
echo "selftest rc=$?"; tail -2 gpurun_out/selftest_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'s2_(fwd_sm100|bwd)' -c 4 \
  -o gpurun_out/bwd_full_$TAG -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-configs \
  --no-hybrid --no-decode > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:'s2_decode_split' -c 1 \
  -o gpurun_out/dec_full_$TAG -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-configs \
  --no-hybrid > gpurun_out/ncu_dec_$TAG.log 2>&1
echo "ncu dec rc=$?"
