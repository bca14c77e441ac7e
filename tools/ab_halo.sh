#!/bin/bash
# A/B: halo reuse on vs off for the non-int8 modes (block configs)
cd "$(dirname "$0")/.."
export CL_LIB_PATH=${CL_LIB_PATH:-$(cd "$(dirname "$0")/.." && pwd)/paper_2507_01040_b200/lib/libclifford_b200_ab.so}  # A/B switches: diagnostic build
CFGS=${CFGS:-"5 3"}
PRECS=${PRECS:-"bf16 tf32 3xtf32"}
for cfg in $CFGS; do
  for prec in $PRECS; do
    for v in on off; do
      if [ $v = off ]; then export CL_NO_HALO=1; else unset CL_NO_HALO; fi
      r=$(timeout 300 python bench.py --config $cfg --precision $prec --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1)
      echo "cfg$cfg $prec halo=$v $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["unit"], d["ms_per_step"], d.get("roofline",{}).get("frac"))' 2>&1)"
    done
  done
done
unset CL_NO_HALO
