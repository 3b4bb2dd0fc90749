#!/bin/bash
# One measurement cycle on the GPU box: parity tests, bench, warm launch list.
# usage: tools/gpu_cycle.sh TAG [pytest-k-expr]
TAG=${1:-run}
K=${2:-}
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$K" > gpurun_out/tests_$TAG.log 2>&1
else
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1
fi
echo "tests_rc=$?"; tail -4 gpurun_out/tests_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1
echo "bench_rc=$?"; tail -c 600 gpurun_out/bench_$TAG.log | head -c 600; echo
export IRK_NO_COND_GRAPH=1
timeout 300 python tools/profile_step.py > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none \
  --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py \
  > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu_rc=$?"; cat gpurun_out/plain_$TAG.log | head -1
