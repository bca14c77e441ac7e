#!/bin/bash
# conv layer + block timings for a few configs / precisions (tools/ab_conv.py)
cd "$(dirname "$0")/.."
for prec in ${PRECS:-bf16 tf32 fp32}; do
  python tools/ab_conv.py --config 3 --precision $prec --B 32
  python tools/ab_conv.py --config 5 --precision $prec --B 64
done
