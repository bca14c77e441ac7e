python -m pytest tests/test_gpu_parity.py -q -x -k "long_reductions or huge_batch" 2>&1 | tail -15
export CL_LIB_PATH=$PWD/paper_2507_01040_b200/lib/libclifford_b200_ab.so
for a in "bf16 16 4" "tf32 16 4" "fp32 16 4" "bf16 32 5" "tf32 32 5"; do echo "== $a"; CL_DBG_CLK=1 python tools/time_vs_ncu.py $a 2>&1 | tail -3; done
bash tools/ab_cfg4.sh 2>&1 | tail -20
