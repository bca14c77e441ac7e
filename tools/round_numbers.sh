#!/bin/bash
# Every bench line of DESIGN.md §6 (run under gpurun from the repo root):
# the headline (cfg5 fp32, with e2e and the CPU baseline), cfg5 in the other
# modes, cfg4 / cfg4b / cfg3 / cfg1 in all modes, cfg2 in all activation modes.
cd "$(dirname "$0")/.."
out=gpurun_out/numbers.jsonl
: > $out
run() { timeout 900 python bench.py "$@" 2>>gpurun_out/numbers.err | tail -1 >> $out; }
run --config 5
for p in 3xtf32 tf32 bf16; do run --config 5 --precision $p --no-cpu --no-e2e; done
for c in 4 40 3 1; do for p in fp32 3xtf32 tf32 bf16; do run --config $c --precision $p --no-cpu --no-e2e; done; done
run --config 2 --all-modes --no-cpu --no-e2e
