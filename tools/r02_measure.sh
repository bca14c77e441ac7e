#!/bin/bash
# Round-2 measurement pass (under gpurun): every bench line with clock records,
# the full-size parity errors in every mode, ncu captures of the block's fused
# conv2 and of cfg4 in the 16-bit / tf32 modes, and the bench launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/round_numbers.sh
python -m pytest tests/test_gpu_configs.py -q -s -m gpu > gpurun_out/configs_errors.log 2>&1
echo "configs rc=$?" >> gpurun_out/status.txt
JOBS="blk2 cfg4bf16 cfg4tf32 blk2full" bash tools/prof_all.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_launches_cfg5_fp32.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e \
  > gpurun_out/r02_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/status.txt
