#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the
# small device workloads of tools/san_cases.py; one log per tool under
# gpurun_out/ (summarised in profiles/r2/sanitizer.txt).
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1200 compute-sanitizer --tool $tool $extra --error-exitcode 7 \
    python tools/san_cases.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_$tool.log
done
