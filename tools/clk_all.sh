#!/bin/bash
# CL_DBG_CLK cycle counters (MMA-warp / producer waits, epilogue time per tile) of the conv in several modes (under gpurun; diagnostic build)
cd "$(dirname "$0")/.."
export CL_LIB_PATH=${CL_LIB_PATH:-$(cd "$(dirname "$0")/.." && pwd)/paper_2507_01040_b200/lib/libclifford_b200_ab.so}  # A/B switches: diagnostic build
for cfg in "4 bf16 16" "4 tf32 16" "4 fp32 16" "5 bf16 32" "5 tf32 32" "5 3xtf32 32" "5 fp32 32" "3 bf16 32" "3 fp32 32"; do
  set -- $cfg
  echo "== cfg$1 $2 B=$3"; CL_DBG_CLK=1 timeout 300 python tools/time_vs_ncu.py $2 $3 $1 2>&1 | tail -2
done
