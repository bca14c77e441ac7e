#!/bin/bash
# ncu --set full captures of the current kernels (run under gpurun from the repo root).
# Each driver first runs plain (must exit 0), then once under ncu (B200_PROFILING.md).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ncu
NCU="ncu --set full --clock-control none --import-source on -c 1"
run() {  # name kernel-regex driver-args...
  local name=$1 kre=$2; shift 2
  timeout 300 python "$@" > gpurun_out/ncu/$name.plain.log 2>&1 && \
    timeout 1200 $NCU ${NCU_EXTRA:-} -k regex:$kre -f -o /tmp/ncu_$name python "$@" > gpurun_out/ncu/$name.ncu.log 2>&1
  echo "$name rc=$?" >> gpurun_out/ncu/status.txt
  # the .ncu-rep stays on the box (gpurun_out is capped at 64 MiB): bring back the raw
  # metrics and the details page (KEEP_REP=1 also copies the report)
  ncu -i /tmp/ncu_$name.ncu-rep --page raw --csv > gpurun_out/ncu/$name.raw.csv 2>/dev/null
  ncu -i /tmp/ncu_$name.ncu-rep --page details --csv > gpurun_out/ncu/$name.details.csv 2>/dev/null
  [ -n "$SOURCE" ] && ncu -i /tmp/ncu_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/$name.sass.csv 2>/dev/null
  [ -n "$KEEP_REP" ] && cp /tmp/ncu_$name.ncu-rep gpurun_out/ncu/
}
for job in ${JOBS:-act bf16 tf32 x3 cfg4 cfg3 cfg1}; do
  case $job in
    act)  run act_cfg2_linear act_kernel tools/prof_conv.py --config 2 --B 64 --act --reps 2 ;;
    bf16) run conv_cfg5_bf16_B32 conv_tc tools/prof_conv.py --config 5 --B 32 --precision bf16 --reps 1 ;;
    tf32) run conv_cfg5_tf32_B32 conv_tc tools/prof_conv.py --config 5 --B 32 --precision tf32 --reps 1 ;;
    x3)   run conv_cfg5_3xtf32_B32 conv_tc tools/prof_conv.py --config 5 --B 32 --precision 3xtf32 --reps 1 ;;
    cfg4) run conv_cfg4_fp32_B16 conv_tc tools/prof_conv.py --config 4 --B 16 --precision fp32 --reps 1 ;;
    cfg3) run conv_cfg3_bf16_B32 conv_tc tools/prof_conv.py --config 3 --B 32 --precision bf16 --reps 1 ;;
    fp32) run conv_cfg5_fp32_B64 conv_tc tools/prof_conv.py --config 5 --B 64 --precision fp32 --reps 1 ;;
    slice) run slice_cfg5_fp32_B64 slice_input tools/prof_conv.py --config 5 --B 64 --precision fp32 --reps 1 ;;
    fp32full) run conv_cfg5_fp32_B256 conv_tc tools/prof_conv.py --config 5 --B 256 --precision fp32 --reps 1 ;;
    cfg1) run conv_cfg1_fp32_B8 conv_tc tools/prof_conv.py --config 1 --B 8 --precision fp32 --reps 3 ;;
    # the block's conv2 (fused residual): skip conv1, capture the second conv_tc launch
    blk2) NCU_EXTRA="--launch-skip 1" run block_cfg5_fp32_B64_conv2 conv_tc tools/prof_block.py --config 5 --B 64 --precision fp32 ;;
    blk2full) NCU_EXTRA="--launch-skip 1" run block_cfg5_fp32_B256_conv2 conv_tc tools/prof_block.py --config 5 --B 256 --precision fp32 ;;
    # cfg3 block convs (2-D): conv1 with the fused gate, conv2 (--launch-skip 1) with the fused residual
    blk3x3c1) run block_cfg3_3xtf32_conv1 conv_tc tools/prof_block.py --config 3 --B 32 --precision 3xtf32 ;;
    blk3x3c2) NCU_EXTRA="--launch-skip 1" run block_cfg3_3xtf32_conv2 conv_tc tools/prof_block.py --config 3 --B 32 --precision 3xtf32 ;;
    blk3bf16c2) NCU_EXTRA="--launch-skip 1" run block_cfg3_bf16_conv2 conv_tc tools/prof_block.py --config 3 --B 32 --precision bf16 ;;
    cfg3fp32) run conv_cfg3_fp32_B32 conv_tc tools/prof_conv.py --config 3 --B 32 --precision fp32 --reps 1 ;;
    cfg4bf16) run conv_cfg4_bf16_B16 conv_tc tools/prof_conv.py --config 4 --B 16 --precision bf16 --reps 1 ;;
    cfg4tf32) run conv_cfg4_tf32_B16 conv_tc tools/prof_conv.py --config 4 --B 16 --precision tf32 --reps 1 ;;
  esac
done
