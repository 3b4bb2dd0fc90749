#!/bin/bash
# A/B step times (conditional-graph mode, 1 warm step then 1 timed step) for
# environment variants; each line: label, iterations, ms.
run() { echo -n "$1: "; env $2 timeout 300 python tools/profile_step.py 2>/dev/null | head -1; }
run default ""
run no_persist "IRK_NO_L2_PERSIST=1"
run no_tail "IRK_TAIL_ROWS=0"
run no_tail_no_persist "IRK_TAIL_ROWS=0 IRK_NO_L2_PERSIST=1"
run tail400 "IRK_TAIL_ROWS=400"
run tail400_no_persist "IRK_TAIL_ROWS=400 IRK_NO_L2_PERSIST=1"
