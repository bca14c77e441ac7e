"""Kernel-only time of one BASELINE conv layer (the tensor-core launch alone,
operand prepared once; cl_conv_time_kernel) plus its plan. For A/B sweeps
with the diagnostic library: CL_LIB_PATH=.../libclifford_b200_ab.so CL_KS=8 ...

  python tools/conv_kernel_time.py <precision> <B> <config> [reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_01040_b200 as M  # noqa: E402
from paper_2507_01040_b200 import _ops, workloads as W  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg = int(sys.argv[3]) if len(sys.argv) > 3 else 4
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
torch.cuda.set_device(0)
spec = W.CONFIGS[cfg]
f1, b1 = W.conv_params(spec, 1)
layer = M.make_conv_layer(M.Dims(B, spec.C, spec.C, spec.d, spec.d_filter, spec.k), M.Signature(spec.g), f1, b1,
                          precision=prec, padding=spec.padding)
x = W.make_input(spec, 0, B)
y = torch.empty(layer.output_shape(), device="cuda")
ms = min(_ops.op("conv_time_kernel", layer.handle(), x, B, reps, y) for _ in range(3))
names = "basis halo pair ks gs tps stages n_tile n_ntiles tx ty tz smem epx bcls tmem".split()
plan = dict(zip(names, _ops.op("conv_plan_info", list(spec.g), spec.C, spec.C, spec.d, spec.d_filter,
                                1 if spec.padding == "same" else 0, M.conv.PRECISIONS[prec])))
tf = M.conv_flops(layer.dims, layer) / ms / 1e9
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("CL_") and k != "CL_LIB_PATH") or "-"
print(f"[{env}] cfg{cfg} {prec} B={B}: {ms:.4f} ms  {tf:.0f} alg TF/s  plan(halo={plan['halo']} pair={plan['pair']} "
      f"ks={plan['ks']} tps={plan['tps']} stages={plan['stages']} n_tile={plan['n_tile']})", flush=True)
