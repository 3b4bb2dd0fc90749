#!/bin/bash
# One ncu --set full capture of the first V-cycle's SpMV-type kernels of a C2
# step (host-driven graph mode; ncu cannot profile under conditional nodes).
TAG=${1:-vc}
export IRK_NO_COND_GRAPH=1
timeout 300 python tools/profile_step.py > gpurun_out/plain_$TAG.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:'k_spmv|k_dense|k_sweep|k_stage_op|k_up_cls|k_tail' -s 1 -c 12 -o gpurun_out/${TAG} python tools/profile_step.py \
  > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"
