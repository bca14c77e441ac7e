#!/bin/bash
# Diagnostic pass (under gpurun): the int8 MMA issue-shape probe (sustained,
# power-capped) and the CL_DBG_CLK cycle counters + plans of the 16-bit / tf32
# convs (diagnostic library).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/diag_smi.csv ) &
SMI=$!
timeout 300 tools/probe/mma_concat ${KSTEPS:-3000000} > gpurun_out/diag_concat.txt 2>&1
kill $SMI
export CL_LIB_PATH=$PWD/paper_2507_01040_b200/lib/libclifford_b200_ab.so
for a in "bf16 16 4" "tf32 16 4" "fp32 16 4" "bf16 32 5" "fp32 32 5"; do
  echo "== $a"; CL_DBG_CLK=1 timeout 300 python tools/conv_kernel_time.py $a 3 2>&1 | tail -3
done > gpurun_out/diag_clk.txt 2>&1
