"""Profiling driver: one conv layer of a BASELINE config, launched a few times
(used under ncu; prints nothing measured -- numbers under ncu are not bench values)."""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2507_01040_b200 as M
from paper_2507_01040_b200 import workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--B", type=int, default=16)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--act", action="store_true", help="profile the standalone activation (cfg2)")
a = ap.parse_args()
torch.cuda.set_device(0)
spec = W.CONFIGS[a.config]
if a.act:
    wgt, bias = W.act_params(spec)
    cfg = M.make_activation_config(M.Signature(spec.g), spec.mode, tuple(range(spec.nb)), wgt, bias)
    x = W.make_input(spec, 0, a.B)
    for _ in range(a.reps):
        y = M.activation_forward(x, cfg)
else:
    f, b = W.conv_params(spec, 1)
    layer = M.make_conv_layer(M.Dims(a.B, spec.C, spec.C, spec.d, spec.d_filter, spec.k), M.Signature(spec.g),
                              f, b, precision=a.precision, padding=spec.padding)
    x = W.make_input(spec, 0, a.B)
    for _ in range(a.reps):
        y = M.conv_forward(x, layer)
torch.cuda.synchronize()
print("done", tuple(y.shape))
