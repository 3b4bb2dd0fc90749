# Round-end records on the final code (one gpurun call): tests, smoke, full-size parity, whole-step traffic,
# benches of every BASELINE workload, reference arm, bench launch list, phase times, ncu --set full of a V-cycle, C5 sweep.
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_final.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_final.log
timeout 1500 python tools/fullsize_parity.py C2 C4 C3 > gpurun_out/fullsize_parity_r2d.jsonl 2> gpurun_out/fullsize_parity_r2d.err; echo "parity rc=$?"
bash tools/step_traffic.sh C2 C4 C3 2>&1 | tail -12
timeout 900 python bench.py > gpurun_out/bench_C2_r2d.log 2>&1; echo "C2 rc=$?"
for w in C4 C3 C1; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/bench_${w}_r2d.log 2>&1; echo "$w rc=$?"; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r2d.log 2>&1; echo "ref rc=$?"
IRK_NO_COND_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_bench_r2d.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench_r2d.log 2>&1; echo "ncu rc=$?"
python tools/phase_times.py > gpurun_out/phases_r2d.txt 2>&1
bash tools/ncu_vcycle.sh vc_r2d
timeout 1200 python tools/c5_sweep.py --json gpurun_out/c5_sweep_r2d.jsonl > gpurun_out/c5_sweep_r2d.csv 2> gpurun_out/c5_sweep_r2d.err; echo "c5 rc=$?"
