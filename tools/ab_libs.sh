#!/bin/bash
# Same-box A/B of several builds of the library (IRK_LIB): for each build dir
# under build_ab/ (and the in-tree lib as "head"), the DCGS2 dot timing and one
# C2 step (tools/profile_step.py, conditional-graph mode).
for lib in head build_ab/*/lib/libirkdev.so; do
  if [ "$lib" = head ]; then unset IRK_LIB; name=head; else export IRK_LIB=$PWD/$lib; name=$(basename $(dirname $(dirname $lib))); fi
  echo "== $name"
  timeout 300 python tools/dgs_time.py 2>&1 | tail -1
  for r in 1 2; do timeout 300 python tools/profile_step.py 2>/dev/null | head -1; done
done
