#!/bin/bash
# Kernel-only times of one conv under diagnostic-library switches (under gpurun):
# CASE="bf16 16 4" VARS="-|CL_DBG_SKIP=4|..." tools/ab_kernel_env.sh
cd "$(dirname "$0")/.."
export CL_LIB_PATH=$PWD/paper_2507_01040_b200/lib/libclifford_b200_ab.so
IFS='|' read -ra vs <<< "${VARS:--}"
IFS='|' read -ra cs <<< "${CASES:-bf16 16 4}"
for c in "${cs[@]}"; do for v in "${vs[@]}"; do
  env $([ "$v" = "-" ] || echo $v) timeout 300 python tools/conv_kernel_time.py $c 2>&1 | tail -1
done; done
