#!/bin/bash
# Round-2 profiling pass that fits gpurun's 64 MiB return limit: the C2 step
# traffic (tools/step_traffic.sh), the launch list of the bench command
# (host-driven graphs: ncu cannot see kernels under conditional nodes) and
# `ncu --set full` captures of the hot kernels exported to CSV on the box.
bash tools/step_traffic.sh C2 > gpurun_out/traffic_r2_C2.txt 2>&1; tail -3 gpurun_out/traffic_r2_C2.txt
IRK_NO_COND_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_bench_r2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/ncu_bench_r2.log 2>&1; echo launch_rc=$?
SPECS="dgsdot:k_dgs_dot:15:1 dgsupdate:k_dgs_update:15:1 cls:k_spmv_cls:2:2 sell:k_spmv_sell:2:2" bash tools/ncu_full.sh r2full
for f in gpurun_out/r2full_*.ncu-rep; do
  ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null
  ncu -i $f --page details --csv > ${f%.ncu-rep}_details.csv 2>/dev/null
  rm -f $f
done
rm -f gpurun_out/traffic_C2.csv.gz; gzip -f gpurun_out/traffic_C2.csv
ls -la gpurun_out | tail -20
