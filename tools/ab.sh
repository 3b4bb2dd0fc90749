#!/bin/bash
# A/B step times (conditional-graph mode, 1 warm step then 1 timed step) for
# environment variants; each line: label, iterations, ms.
# ARGS (optional): profile_step.py arguments (cells s kind).
run() { echo -n "$1: "; env $2 timeout 300 python tools/profile_step.py $ARGS 2>/dev/null | head -1; }
for v in "${@:-default=}"; do run "${v%%=*}" "${v#*=}"; done
