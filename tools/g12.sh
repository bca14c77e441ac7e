python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for a in "fp32 16 4" "fp32 32 5" "fp32 32 3" "fp32 8 1" "bf16 16 4" "tf32 16 4" "3xtf32 16 4" "bf16 32 5"; do python tools/conv_kernel_time.py $a 2>&1 | tail -1; done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
