set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_final.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_final.log
timeout 1500 python tools/fullsize_parity.py C2 C4 C3 > gpurun_out/fullsize_parity_r2c.jsonl 2> gpurun_out/fullsize_parity_r2c.err; echo "parity rc=$?"
bash tools/step_traffic.sh C2 C4 C3 2>&1 | grep -v "^+" | tail -12
