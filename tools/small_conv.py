"""cfg1-sized conv latency: whole conv_forward (operand prep + tensor-core kernel)
and the tensor-core kernel alone (cl_conv_time_kernel), per precision, CUDA events,
warm. Run once per env variant (e.g. CL_NO_PAIR=1)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_01040_b200 as M  # noqa: E402
from paper_2507_01040_b200 import _lib, workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
torch.cuda.set_device(0)
spec = W.CONFIGS[cfg]
lib = _lib.load()
x = W.make_input(spec, 0, spec.B)
f, b = W.conv_params(spec, 1)
tag = " ".join(k for k in os.environ if k.startswith("CL_")) or "default"
for prec in ["fp32", "bf16", "tf32", "3xtf32"]:
    layer = M.make_conv_layer(M.Dims(spec.B, spec.C, spec.C, spec.d, spec.d_filter, spec.k), M.Signature(spec.g), f, b,
                              precision=prec, padding=spec.padding)
    y = torch.empty(layer.output_shape(), device="cuda")
    for _ in range(20):
        M.conv_forward(x, layer, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 200
    e0.record()
    for _ in range(n):
        M.conv_forward(x, layer, out=y)
    e1.record()
    torch.cuda.synchronize()
    t_fwd = e0.elapsed_time(e1) / n * 1e3
    # host cost of one call: launches queued back to back without a sync
    import time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        M.conv_forward(x, layer, out=y)
    t_host = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    ms = ctypes.c_float()
    _lib.check(lib.cl_conv_time_kernel(ctypes.c_void_p(layer.handle()), ctypes.c_void_p(x.data_ptr()),
                                       ctypes.c_void_p(y.data_ptr()), spec.B, n,
                                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), ctypes.byref(ms)))
    print(f"[{tag}] cfg{cfg} {prec:6s} conv_forward {t_fwd:8.2f} us (host {t_host:6.2f} us/call)   kernel alone {ms.value * 1e3:8.2f} us", flush=True)
