#!/bin/bash
# Full ncu captures of the hot kernels of one C2 step (host-driven graph mode,
# since ncu cannot profile kernel nodes under conditional graph nodes).
TAG=${1:-full}
export IRK_NO_COND_GRAPH=1
timeout 300 python tools/profile_step.py > gpurun_out/plain_full.log 2>&1 || exit 1
for spec in ${SPECS:-"dgsdot:k_dgs_dot:15:1" "dgsupdate:k_dgs_update:15:1" "dia:k_spmv_dia:10:2" "stageop:k_stage_op:10:1" "sell:k_spmv_sell:10:2"}; do
  IFS=: read name kern skip cnt <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base demangled \
    -k regex:$kern -s $skip -c $cnt -o gpurun_out/${TAG}_$name python tools/profile_step.py \
    > gpurun_out/ncu_${TAG}_$name.log 2>&1
  echo "$name rc=$?"
done
