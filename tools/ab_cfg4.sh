export CL_LIB_PATH=${CL_LIB_PATH:-$(cd "$(dirname "$0")/.." && pwd)/paper_2507_01040_b200/lib/libclifford_b200_ab.so}  # A/B switches: diagnostic build
for v in "-" "CL_TPS=2" "CL_TPS=4" "CL_KS=2" "CL_KS=8" "CL_NO_PAIR=1" "CL_NO_HALO=1" "CL_DBG_SKIP=4"; do
  for p in bf16 tf32; do
    echo "[$v] $p $(env $([ "$v" = "-" ] || echo $v) timeout 300 python tools/time_vs_ncu.py $p 16 4 2>&1 | tail -1)"
  done
done
