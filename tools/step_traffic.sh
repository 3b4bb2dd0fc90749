#!/bin/bash
# Measured DRAM traffic of one whole IRK step (SURVEY §8d cross-check):
# every launch of one step (host-driven graph mode -- ncu cannot profile
# kernels under conditional graph nodes; the kernels are identical) with
# dram__bytes_read.sum + dram__bytes_write.sum and its duration, caches NOT
# flushed between kernels (--cache-control none) so L2 reuse is as in a run.
# The step's own time comes from the same script without ncu, in the normal
# conditional-graph mode.   usage: tools/step_traffic.sh C2 [C3 C4 ...]
for W in "${@:-C2}"; do
  timeout 600 python tools/profile_step.py $W > gpurun_out/traffic_graph_$W.log 2>&1
  IRK_NO_COND_GRAPH=1 timeout 600 python tools/profile_step.py $W > gpurun_out/traffic_plain_$W.log 2>&1
  IRK_NO_COND_GRAPH=1 timeout 1800 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --cache-control none --profile-from-start off --csv \
    --log-file gpurun_out/traffic_$W.csv python tools/profile_step.py $W > gpurun_out/traffic_ncu_$W.log 2>&1
  echo "$W ncu_rc=$? graph: $(head -1 gpurun_out/traffic_graph_$W.log) plain: $(head -1 gpurun_out/traffic_plain_$W.log)"
  python tools/traffic_summary.py gpurun_out/traffic_$W.csv gpurun_out/traffic_graph_$W.log $W \
    > gpurun_out/traffic_summary_$W.txt 2>&1; tail -4 gpurun_out/traffic_summary_$W.txt
done
