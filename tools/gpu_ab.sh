#!/bin/bash
# A/B session on the GPU box: backward/forward parity tests + timing of the
# variants selected by env (e.g. S2_DQ_V1=1).  Usage:
#   gpurun -- 'bash tools/gpu_ab.sh TAG "ENV_A" "ENV_B" [pytest-k-expr]'
TAG=${1:-ab}; A=${2:-}; B=${3:-S2_DQ_V1=1}; K=${4:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv,noheader > gpurun_out/smi_$TAG.txt
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$K" > gpurun_out/tests_$TAG.log 2>&1
  echo "tests rc=$?"; tail -3 gpurun_out/tests_$TAG.log
fi
for rep in 1 2; do
  for E in "$A" "$B"; do
    echo "== [$E] rep $rep"
    env $E timeout 300 python tools/perf_bwd.py --uniform --iters 20 2>&1 | tail -2
  done
done
