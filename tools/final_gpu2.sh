# round-end records: library build variants A/B, block-Jacobi check, benches, bench launch list
ROUNDS=2 IRK_AB_REPS=5 bash tools/ab_libs.sh 2>&1 | tee gpurun_out/ab_libs_r2c.txt
ARGS="1024 3 0" bash tools/ab.sh jac_comp= jac_rec=IRK_COMPOSE=0 2>&1 | tee gpurun_out/ab_jacobi_r2c.txt
ARGS="1024 7 3" bash tools/ab.sh s7_comp= s7_rec=IRK_COMPOSE=0 2>&1 | tee -a gpurun_out/ab_jacobi_r2c.txt
timeout 900 python bench.py > gpurun_out/bench_C2_r2c.log 2>&1; echo "C2 rc=$?"
for w in C4 C3 C1; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/bench_${w}_r2c.log 2>&1; echo "$w rc=$?"; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r2c.log 2>&1; echo "ref rc=$?"
IRK_NO_COND_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_bench_r2c.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench_r2c.log 2>&1; echo "ncu rc=$?"
