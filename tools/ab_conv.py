"""A/B timing helper: one BASELINE config's conv layer and block, CUDA-event
timed (run once per env setting, e.g. CL_NO_HALO=1)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_01040_b200 as M  # noqa: E402
from paper_2507_01040_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--precision", default="bf16")
ap.add_argument("--B", type=int, default=0)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
torch.cuda.set_device(0)
spec = W.CONFIGS[a.config]
B = a.B or spec.B
x = W.make_input(spec, 0, B)
f1, b1 = W.conv_params(spec, 1)
layer = M.make_conv_layer(M.Dims(B, spec.C, spec.C, spec.d, spec.d_filter, spec.k), M.Signature(spec.g), f1, b1,
                          precision=a.precision, padding=spec.padding)


from bench import ClockSampler  # noqa: E402

clocks = {}


def timeit(fn, name):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as cs:
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
    clocks[name] = cs.summary().get("sm_mhz")
    return e0.elapsed_time(e1) / a.iters


y = torch.empty(layer.output_shape(), device="cuda")
res = {"conv_ms": timeit(lambda: M.conv_forward(x, layer, out=y), "conv")}
if spec.kind == "block":
    f2, b2 = W.conv_params(spec, 2)
    aw, ab = W.act_params(spec)
    blk = M.make_basic_block(M.Signature(spec.g), B, spec.C, spec.C, spec.C, spec.d, f1, b1, spec.mode, f2, b2,
                             act_weight=aw, act_bias=ab, padding=spec.padding, residual=True, precision=a.precision)
    yb = torch.empty_like(x)
    res["block_ms"] = timeit(lambda: M.block_forward(x, blk, out=yb), "block")
tag = "halo=off" if os.environ.get("CL_NO_HALO") else "halo=on"
print(f"cfg{a.config} {a.precision} B={B} {tag}", " ".join(f"{k}={v:.3f}" for k, v in res.items()),
      "sm_mhz", clocks, flush=True)
