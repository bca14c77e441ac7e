"""Profiling driver: one block of a BASELINE config (conv1 with the fused
activation, conv2 with the fused residual); prints nothing measured."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
import paper_2507_01040_b200 as M  # noqa: E402
from paper_2507_01040_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--B", type=int, default=16)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
torch.cuda.set_device(0)
spec = W.CONFIGS[a.config]
f1, b1 = W.conv_params(spec, 1)
f2, b2 = W.conv_params(spec, 2)
aw, ab = W.act_params(spec)
blk = M.make_basic_block(M.Signature(spec.g), a.B, spec.C, spec.C, spec.C, spec.d, f1, b1, spec.mode, f2, b2,
                         act_weight=aw, act_bias=ab, padding=spec.padding, residual=True, precision=a.precision)
x = W.make_input(spec, 0, a.B)
for _ in range(a.reps):
    y = M.block_forward(x, blk)
torch.cuda.synchronize()
print("done", tuple(y.shape))
