#!/bin/bash
# Kernel-only A/B of two library builds (under gpurun): ALT=<dir with
# libclifford_b200.so> vs the in-tree build, alternating, over CASES
# ("precision B config" triples).
cd "$(dirname "$0")/.."
ALT=${ALT:-tools/oldlib}
CASES=${CASES:-"bf16 16 4|tf32 16 4|fp32 16 4|3xtf32 16 4|bf16 32 5|tf32 32 5|fp32 32 5|bf16 32 3|tf32 32 3|fp32 32 3|fp32 8 1|bf16 8 1"}
IFS='|' read -ra cs <<< "$CASES"
for c in "${cs[@]}"; do
  for r in 1 2; do
    echo "ALT $(CL_LIB_PATH=$PWD/$ALT/libclifford_b200.so timeout 300 python tools/conv_kernel_time.py $c 2>&1 | tail -1)"
    echo "NEW $(timeout 300 python tools/conv_kernel_time.py $c 2>&1 | tail -1)"
  done
done
