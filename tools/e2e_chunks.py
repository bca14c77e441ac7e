"""e2e (pinned host in / out) time of the cfg5 block per host-pipeline chunk size.

    python tools/e2e_chunks.py [precision] [chunk ...]     (0 = the library's automatic size)
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2507_01040_b200 as M  # noqa: E402
from paper_2507_01040_b200 import workloads as W  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
chunks = [int(c) for c in sys.argv[2:]] or [0, 4, 12, 16, 24, 32]
torch.cuda.set_device(0)
spec = W.CONFIGS[5]
f1, b1 = W.conv_params(spec, 1)
f2, b2 = W.conv_params(spec, 2)
aw, ab = W.act_params(spec)
blk = M.make_basic_block(M.Signature(spec.g), spec.B, spec.C, spec.C, spec.C, spec.d, f1, b1, spec.mode, f2, b2,
                         act_weight=aw, act_bias=ab, padding=spec.padding, residual=True, precision=prec)
x = W.make_input(spec, 0, spec.B)
xh = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
xh.copy_(x)
del x
yh = torch.empty(xh.shape, dtype=torch.float32, pin_memory=True)
for c in chunks:
    M.block_forward(xh, blk, chunk=c, out=yh)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        M.block_forward(xh, blk, chunk=c, out=yh)
        float(yh.view(-1)[0])
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    print(f"chunk {c:3d}: {t * 1e3:7.1f} ms  {spec.B / t:6.1f} samples/s", flush=True)
