#!/bin/bash
# Same-box A/B of several builds of the library (IRK_LIB): the in-tree lib
# ("head") and every build under build_ab/<name>/lib, interleaved ROUNDS times;
# each line is one process: one C2 step + IRK_AB_REPS repeats (min / median).
# DGS=1 adds the isolated DCGS2 block-dot timing.
export IRK_AB_REPS=${IRK_AB_REPS:-10}
for round in $(seq 1 ${ROUNDS:-2}); do
  for lib in head build_ab/*/lib/libirkdev.so; do
    if [ "$lib" = head ]; then unset IRK_LIB; name=head; else export IRK_LIB=$PWD/$lib; name=$(basename $(dirname $(dirname $lib))); fi
    [ -n "$DGS" ] && echo "$name $(timeout 300 python tools/dgs_time.py 2>&1 | tail -1)"
    echo "$name: $(timeout 300 python tools/profile_step.py $ARGS 2>/dev/null | head -1)"
  done
done
