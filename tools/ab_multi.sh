#!/bin/bash
# Kernel-only A/B of several library builds (under gpurun): LIBS="dir dir ..."
# (each holding libclifford_b200.so; "-" = the in-tree build), alternating,
# over CASES ("precision B config" triples), ROUNDS times.
cd "$(dirname "$0")/.."
LIBS=${LIBS:-"tools/oldlib -"}
CASES=${CASES:-"bf16 16 4|tf32 16 4|bf16 32 5|tf32 32 5"}
ROUNDS=${ROUNDS:-2}
IFS='|' read -ra cs <<< "$CASES"
for c in "${cs[@]}"; do
  for r in $(seq $ROUNDS); do
    for l in $LIBS; do
      if [ "$l" = "-" ]; then
        echo "in-tree $(timeout 300 python tools/conv_kernel_time.py $c 2>&1 | tail -1)"
      else
        echo "$l $(CL_LIB_PATH=$PWD/$l/libclifford_b200.so timeout 300 python tools/conv_kernel_time.py $c 2>&1 | tail -1)"
      fi
    done
  done
done
