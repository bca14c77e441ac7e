"""Small cases of every kernel family for compute-sanitizer (one tool per gpurun call):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py

conv k=1/2/3 in every precision (valid and same), the standalone activation,
2-D / 3-D blocks, the host (chunked H2D/compute/D2H) path and the linear layer.
Each result is checked against the oracle (the checker only)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_2507_01040_b200 as M  # noqa: E402

torch.cuda.set_device(0)
rng = np.random.default_rng(7)
TOL = {"fp32": 1e-4, "3xtf32": 1e-3, "tf32": 2e-2, "bf16": 2e-2}
n = 0


def conv_case(g, B, C, d, df, prec, padding):
    global n
    k = len(g)
    nb = 1 << k
    x = rng.standard_normal((B, C, d ** k, nb)).astype(np.float32)
    f = rng.uniform(-1, 1, (nb, C, C, df ** k)).astype(np.float32) / np.float32(np.sqrt(C * nb * df ** k))
    b = (rng.standard_normal((nb, C)) * 0.01).astype(np.float32)
    layer = M.make_conv_layer(M.Dims(B, C, C, d, df, k), M.Signature(g), f, b, precision=prec, padding=padding)
    y = M.conv_forward(torch.from_numpy(x).cuda(), layer).cpu().numpy()
    yh = M.conv_forward(x, layer)  # host path
    pad = (df - 1) // 2 if padding == "same" else 0
    ref = O.conv_ref(x, f, b, g, d, df, pad)
    fl = 1e-2 if prec == "fp32" else float(np.abs(ref).max())
    e = O.max_rel_error(y, ref, floor=fl)
    assert e <= TOL[prec], (g, prec, padding, e)
    assert np.array_equal(np.asarray(yh), y)
    n += 1


for g in [(1,), (1, 1), (1, 1, 1), (1, -1, 0)]:
    for prec in ["fp32", "3xtf32", "tf32", "bf16"]:
        for padding in ["valid", "same"]:
            d = {1: 20, 2: 9, 3: 6}[len(g)]
            conv_case(g, 3, 5, d, 3, prec, padding)

for g in [(1,), (1, 1), (1, 1, 1)]:
    nb = 1 << len(g)
    C, B, P = 6, 3, 37
    x = rng.standard_normal((B, C, P, nb)).astype(np.float32)
    for mode in (0, 1, 2):
        w = rng.uniform(-0.5, 0.5, (C, nb)).astype(np.float32) if mode == 0 else None
        bb = (rng.standard_normal(C) * 0.1).astype(np.float32) if mode == 0 else None
        cfg = M.make_activation_config(M.Signature(g), mode, tuple(range(nb)), w, bb)
        y = M.activation_forward(torch.from_numpy(x).cuda(), cfg).cpu().numpy()
        ref = O.activation_ref(x, mode, tuple(range(nb)), w, bb)
        assert O.max_abs_error(y, ref) <= 1e-5
        n += 1

for g, d, prec in [((1, 1), 10, "fp32"), ((1, 1), 10, "bf16"), ((1, 1, 1), 6, "fp32"), ((1, 1, 1), 6, "bf16")]:
    k = len(g)
    nb = 1 << k
    B, C = 2, 8
    fan = C * nb * 3 ** k
    f1 = rng.uniform(-1, 1, (nb, C, C, 3 ** k)).astype(np.float32) / np.float32(np.sqrt(fan))
    f2 = rng.uniform(-1, 1, (nb, C, C, 3 ** k)).astype(np.float32) / np.float32(np.sqrt(fan))
    b1 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    b2 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    x = rng.standard_normal((B, C, d ** k, nb)).astype(np.float32)
    blk = M.make_basic_block(M.Signature(g), B, C, C, C, d, f1, b1, 2, f2, b2, padding="same", residual=True,
                             precision=prec)
    y = M.block_forward(torch.from_numpy(x).cuda(), blk).cpu().numpy()
    yh = M.block_forward(x, blk)
    ref = O.block_ref(x, g, d, f1, b1, 2, tuple(range(nb)), None, None, f2, b2, padding="same", residual=True)
    fl = 1e-2 if prec == "fp32" else float(np.abs(ref).max())
    assert O.max_rel_error(y, ref, floor=fl) <= TOL[prec]
    assert np.array_equal(np.asarray(yh), y)
    n += 1

torch.cuda.synchronize()
print(f"sanitize cases ok: {n}")
