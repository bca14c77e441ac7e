python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for a in "bf16 16 4" "tf32 16 4" "fp32 16 4" "3xtf32 16 4" "bf16 32 5" "tf32 32 5" "fp32 32 5" "bf16 32 3" "fp32 32 3"; do python tools/conv_kernel_time.py $a 2>&1 | tail -1; done
