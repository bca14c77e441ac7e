"""Ad-hoc GPU parity probe (prints errors per case; not collected by pytest)."""
import sys
import time
import traceback

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as O
import paper_2507_01040_b200 as M


def conv_case(g, B, ci, co, d, df, prec, padding="valid", seed=0):
    rng = np.random.default_rng(seed)
    k = len(g)
    nb = 1 << k
    x = rng.standard_normal((B, ci, d ** k, nb)).astype(np.float32)
    fan = ci * nb * df ** k
    f = rng.uniform(-1, 1, (nb, ci, co, df ** k)).astype(np.float32) / np.float32(np.sqrt(fan))
    b = (rng.standard_normal((nb, co)) * 0.01).astype(np.float32)
    dims = M.Dims(B, ci, co, d, df, k)
    layer = M.make_conv_layer(dims, M.Signature(tuple(g)), f, b, precision=prec, padding=padding)
    y = M.conv_forward(torch.from_numpy(x).cuda(), layer).cpu().numpy()
    pad = (df - 1) // 2 if padding == "same" else 0
    ref = O.conv_ref(x, f, b, tuple(g), d, df, pad)
    e1 = O.max_rel_error(y, ref)
    e2 = O.max_rel_error(y, ref, floor=float(np.abs(ref).max()))
    return e1, e2


def main():
    torch.cuda.init()
    print("device", torch.cuda.get_device_name(0))
    lib = M._lib.load()
    # expand kernel
    for g in [(1, 1), (1, -1, 0), (1,), (0, 1)]:
        k = len(g)
        nb = 1 << k
        rng = np.random.default_rng(1)
        f = rng.standard_normal((nb, 3, 2, 3 ** k)).astype(np.float32)
        dims = M.Dims(1, 3, 2, 4, 3, k)
        layer = M.make_conv_layer(dims, M.Signature(g), f, np.zeros((nb, 2), np.float32))
        W = M.build_expanded_kernel(layer).cpu().numpy()
        ok = np.array_equal(W, O.expanded_kernel(f, g))
        print("expand", g, "bit-exact" if ok else "MISMATCH")
    cases = [
        ((1, 1), 2, 4, 4, 8, 3, "3xtf32"),
        ((1, 1, 1), 2, 32, 32, 16, 3, "3xtf32"),
        ((1, 1), 2, 4, 4, 8, 3, "fp32"),
        ((1, 1), 2, 4, 4, 8, 3, "tf32"),
        ((1, 1), 2, 4, 4, 8, 3, "bf16"),
        ((1, 1, 1), 2, 4, 4, 6, 3, "fp32"),
        ((1, 1, 1), 2, 4, 4, 6, 3, "tf32"),
        ((1, 1, 1), 2, 4, 4, 6, 3, "bf16"),
        ((1, 1), 8, 16, 16, 32, 3, "fp32"),
        ((1, 1), 8, 16, 16, 32, 3, "tf32"),
        ((1, 1), 8, 16, 16, 32, 3, "bf16"),
        ((1, -1, 0), 2, 32, 32, 12, 3, "fp32"),
        ((1, 1, 1), 2, 32, 32, 16, 3, "fp32"),
        ((1, 1), 2, 64, 64, 32, 3, "fp32"),
    ]
    for c in cases:
        try:
            t = time.time()
            e1, e2 = conv_case(*c)
            print("conv", c, f"mre={e1:.3e} mre_maxfloor={e2:.3e}", f"{time.time()-t:.1f}s", flush=True)
        except Exception:
            traceback.print_exc()
            print("conv", c, "FAILED", flush=True)
    for c in [((1, 1), 2, 4, 4, 8, 3, "fp32", "same"), ((1, 1, 1), 2, 8, 8, 6, 3, "fp32", "same"),
              ((1, 1), 2, 8, 8, 8, 3, "bf16", "same")]:
        try:
            e1, e2 = conv_case(*c)
            print("conv", c, f"mre={e1:.3e} mre_maxfloor={e2:.3e}", flush=True)
        except Exception:
            traceback.print_exc()
    # activation
    for k in (2, 3):
        nb = 1 << k
        for mode in (0, 1, 2):
            rng = np.random.default_rng(3)
            C = 13
            ki = tuple(rng.permutation(nb)[: nb // 2 + 1])
            w = rng.uniform(-0.5, 0.5, (C, len(ki))).astype(np.float32) if mode == 0 else None
            bb = (rng.standard_normal(C) * 0.1).astype(np.float32) if mode == 0 else None
            cfg = M.make_activation_config(M.Signature((1,) * k), mode, ki, w, bb)
            x = rng.standard_normal((3, C, 7, nb)).astype(np.float32)
            y = M.activation_forward(torch.from_numpy(x).cuda(), cfg).cpu().numpy()
            ref = O.activation_ref(x, mode, ki, w, bb)
            print("act", k, mode, ki, f"mae={O.max_abs_error(y, ref):.3e}")
    print("launches", M._lib.launch_count())


if __name__ == "__main__":
    main()
