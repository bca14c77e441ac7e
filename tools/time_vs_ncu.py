"""Event-timed conv launches of one layer (compare with ncu's gpu__time_duration)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2507_01040_b200 as M  # noqa: E402
from paper_2507_01040_b200 import workloads as W  # noqa: E402
prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
cfg = int(sys.argv[3]) if len(sys.argv) > 3 else 5
torch.cuda.set_device(0)
spec = W.CONFIGS[cfg]
f1, b1 = W.conv_params(spec, 1)
layer = M.make_conv_layer(M.Dims(B, spec.C, spec.C, spec.d, spec.d_filter, spec.k), M.Signature(spec.g), f1, b1,
                          precision=prec, padding=spec.padding)
x = W.make_input(spec, 0, B)
y = torch.empty(layer.output_shape(), device="cuda")
for i in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    M.conv_forward(x, layer, out=y)
    e1.record()
    torch.cuda.synchronize()
    print(f"iter {i}: {e0.elapsed_time(e1):.3f} ms", flush=True)
