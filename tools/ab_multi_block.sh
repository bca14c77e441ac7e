#!/bin/bash
# Conv-layer and block timing (tools/ab_conv.py, CUDA events) of several library builds:
# LIBS="dir dir ..." ("-" = in-tree), CASES="config precision B|..." (B = 0: the config's batch)
cd "$(dirname "$0")/.."
LIBS=${LIBS:-"tools/oldlib -"}
CASES=${CASES:-"3 3xtf32 0|5 3xtf32 32|4 3xtf32 0"}
IFS='|' read -ra cs <<< "$CASES"
for c in "${cs[@]}"; do
  set -- $c
  for l in $LIBS; do
    if [ "$l" = "-" ]; then
      timeout 300 python tools/ab_conv.py --config $1 --precision $2 --B $3 2>&1 | tail -2 | sed "s|^|in-tree |"
    else
      CL_LIB_PATH=$PWD/$l/libclifford_b200.so timeout 300 python tools/ab_conv.py --config $1 --precision $2 --B $3 2>&1 | tail -2 | sed "s|^|$l |"
    fi
  done
done
