# B-operand bandwidth experiment: conv time with and without the B stage loads (CL_DBG_SKIP=1, results garbage)
export CL_LIB_PATH=${CL_LIB_PATH:-$(cd "$(dirname "$0")/.." && pwd)/paper_2507_01040_b200/lib/libclifford_b200_ab.so}  # A/B switches: diagnostic build
for cfg in "5 bf16 64" "5 tf32 64" "4 bf16 16" "5 fp32 64"; do
  set -- $cfg
  for v in "" "CL_DBG_SKIP=1"; do
    echo "== cfg$1 $2 B=$3 $v"; env $v timeout 300 python tools/time_vs_ncu.py $2 $3 $1 2>&1 | tail -1
  done
done
