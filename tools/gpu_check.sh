# round-2 GPU check: full GPU test suite, then a short default bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > gpurun_out/t_pytest.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/t_pytest.log
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/t_bench.log 2>&1; echo "bench rc=$?"
  tail -3 gpurun_out/t_bench.log | cut -c1-3000
fi
