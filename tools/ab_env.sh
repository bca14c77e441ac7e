#!/bin/bash
# A/B over env settings: ENVS="A=1 B=2|C=3" (| separates variants; "-" = none)
cd "$(dirname "$0")/.."
export CL_LIB_PATH=${CL_LIB_PATH:-$(cd "$(dirname "$0")/.." && pwd)/paper_2507_01040_b200/lib/libclifford_b200_ab.so}  # A/B switches: diagnostic build
IFS='|' read -ra VARS <<< "${ENVS:--}"
for v in "${VARS[@]}"; do
  for c in ${CFGS:-5}; do
    B=$([ $c = 5 ] && echo 64 || echo 0)
    env $([ "$v" = "-" ] || echo $v) python tools/ab_conv.py --config $c --precision ${PREC:-fp32} --B $B | sed "s|^|[$v] |"
  done
done
