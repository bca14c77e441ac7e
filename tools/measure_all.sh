#!/bin/bash
# Full measurement pass (under gpurun): the GPU suite, every bench line
# with clock records, ncu of the current headline kernel and cfg4 16-bit modes,
# the bench launch list and the default bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/m2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/m2_status.txt
tail -3 gpurun_out/m2_pytest.log >> gpurun_out/m2_status.txt
bash tools/round_numbers.sh
cp gpurun_out/numbers.jsonl gpurun_out/m2_numbers.jsonl
rm -f gpurun_out/ncu/status.txt
JOBS="cfg4bf16 cfg4tf32 x3 bf16 blk2full" bash tools/prof_all.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/m2_launches_cfg5_fp32.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e \
  > gpurun_out/m2_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/m2_status.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/m2_bench.json 2> gpurun_out/m2_bench.err
echo "bench rc=$?" >> gpurun_out/m2_status.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/m2_ref.json 2> gpurun_out/m2_ref.err
echo "ref rc=$?" >> gpurun_out/m2_status.txt
