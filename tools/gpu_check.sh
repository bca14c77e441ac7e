set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -x -q -m gpu > gpurun_out/t1_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/t1_pytest.log
BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/t1_share2.log 2>&1; echo "share2 rc=$?"
tail -3 gpurun_out/t1_share2.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/t1_bench.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/t1_bench.log
