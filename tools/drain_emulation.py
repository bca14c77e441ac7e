"""3xTF32 accuracy vs accumulation-chain length, measured on the B200's own
tensor cores (no kernel change needed): a conv whose filter is zero except
for one group of (tap, input-channel) entries gives exactly the partial sum
the tensor core would hold if its TMEM accumulator were drained after that
group (adding zero products leaves the accumulator unchanged). Summing the
group partials in fp32 / fp64 on the host emulates periodic draining.

  python tools/drain_emulation.py [C] [d]

Prints max_rel_error (floor 1e-2, the reference metric) against the fp64
oracle for: one accumulator (the current kernel), drain per tap, drain per
(tap, channel group of 16 / 8 / 4 channels)."""

import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2507_01040_b200 as M  # noqa: E402

C = int(sys.argv[1]) if len(sys.argv) > 1 else 32
d = int(sys.argv[2]) if len(sys.argv) > 2 else 12
g, k, nb, df, B = (1, 1, 1), 3, 8, 3, 2
rng = np.random.default_rng(0)
fan = C * nb * 27
x = rng.standard_normal((B, C, d ** 3, nb)).astype(np.float32)
f = rng.uniform(-1, 1, (nb, C, C, 27)).astype(np.float32) / np.float32(np.sqrt(fan))
b = (rng.standard_normal((nb, C)) * 0.01).astype(np.float32)
ref = O.conv_ref(x, f, b, g, d, df, 0)
dims = M.Dims(B, C, C, d, df, k)
xd = torch.from_numpy(x).cuda()
zero_b = np.zeros_like(b)


def conv(filt, bias, prec="3xtf32"):
    layer = M.make_conv_layer(dims, M.Signature(g), filt, bias, precision=prec)
    return M.conv_forward(xd, layer).cpu().numpy()


out = {"C": C, "K": C * nb * 27, "K_basis": C * 4 * 27}
out["one_accumulator"] = O.max_rel_error(conv(f, b), ref)
out["fp32_exact_mode"] = O.max_rel_error(conv(f, b, "fp32"), ref)
for cg in (C, 16, 8, 4):
    if cg > C:
        continue
    parts = []
    for q in range(27):
        for c0 in range(0, C, cg):
            fq = np.zeros_like(f)
            fq[:, c0:c0 + cg, :, q] = f[:, c0:c0 + cg, :, q]
            parts.append(conv(fq, zero_b))
    s32 = np.zeros_like(parts[0])
    for p in parts:
        s32 = (s32 + p).astype(np.float32)
    s64 = np.sum(np.stack(parts).astype(np.float64), axis=0)
    bias_bc = b.T[None, :, None, :]
    out[f"drain_tap_x_{cg}ch_fp32sum"] = O.max_rel_error((s32 + bias_bc).astype(np.float32), ref)
    out[f"drain_tap_x_{cg}ch_fp64sum"] = O.max_rel_error((s64 + bias_bc).astype(np.float32), ref)
print(out)
