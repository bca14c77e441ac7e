"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the reference package `mvkernels` (numpy + numba CPU code) and
records small input/output pairs for every function on the hot path. The
resulting `golden.npz` is committed; the GPU box never reads /root/reference.
Reference call sites used: algebra.product_table / blade_product
(algebra.py:87-129), specialize.schedule_for / schedule_to_text
(specialize.py:66-74, :334-346), conv.conv_reference / build_expanded_kernel /
conv_flops (conv.py:151-202, :384-387), activation.activation_reference and
activation_forward('specialized') (activation.py:338-416), serve._forward
(serve.py:102-119, spatial fold), bench.max_rel_error (bench.py:74-88),
layout.write_tensor (layout.py:183-196), layout.gather_index_table
(layout.py:137-146).
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

import mvkernels as mk
from mvkernels import activation as act
from mvkernels import serve

HERE = os.path.dirname(os.path.abspath(__file__))


def gkey(g):
    return "_".join(str(v) for v in g)


def main():
    rng = np.random.default_rng(20250701)
    out: dict[str, np.ndarray] = {}

    # 1. blade product tables + schedules for all 36 signatures
    sigs = mk.all_valid_signatures(3)
    out["sig_list"] = np.array([gkey(s.g) for s in sigs])
    for s in sigs:
        t = mk.product_table(s)
        out[f"table_target_{gkey(s.g)}"] = np.array(t.target)
        out[f"table_coeff_{gkey(s.g)}"] = np.array(t.coeff)
        sch = mk.schedule_for(s)
        out[f"sched_{gkey(s.g)}"] = np.array(
            [[tm.out_blade, tm.a_blade, tm.b_blade, int(tm.negate)] for tm in sch.terms],
            dtype=np.int64,
        )
    out["sched_text_1"] = np.array(mk.schedule_to_text(mk.schedule_for(mk.Signature((1,)))))
    out["sched_text_1_1_labels"] = np.array(
        mk.schedule_to_text(mk.schedule_for(mk.Signature((1, 1))), labels=True))

    # 2. expanded kernels + conv oracle outputs
    conv_cases = [
        # (g, B, C_in, C_out, d_image, d_filter)
        ((1,), 2, 3, 2, 9, 3),
        ((-1,), 3, 2, 2, 5, 2),
        ((1, 1), 2, 3, 5, 6, 3),
        ((1, -1), 2, 2, 2, 6, 2),
        ((0, 1), 1, 4, 3, 5, 3),
        ((-1, -1), 2, 5, 4, 7, 3),
        ((1, 1, 1), 2, 2, 3, 5, 3),
        ((1, -1, 0), 2, 3, 2, 5, 3),
        ((-1, 0, 1), 1, 2, 2, 4, 2),
        ((0, 0, 1), 1, 3, 2, 4, 2),
    ]
    for n, (g, B, ci, co, di, df) in enumerate(conv_cases):
        sig = mk.Signature(g)
        dims = mk.Dims(B=B, C_in=ci, C_out=co, d_image=di, d_filter=df, k=len(g))
        x = rng.standard_normal(dims.input_shape()).astype(np.float32)
        f = (rng.standard_normal(dims.filters_shape()) * 0.3).astype(np.float32)
        b = (rng.standard_normal(dims.bias_shape()) * 0.1).astype(np.float32)
        layer = mk.make_conv_layer(dims, sig, f, b, W=1)
        out[f"conv{n}_g"] = np.array(g, dtype=np.int64)
        out[f"conv{n}_dims"] = np.array([B, ci, co, di, df, len(g)], dtype=np.int64)
        out[f"conv{n}_x"] = x
        out[f"conv{n}_f"] = f
        out[f"conv{n}_b"] = b
        out[f"conv{n}_y"] = mk.conv_reference(x, layer)
        out[f"conv{n}_W"] = mk.build_expanded_kernel(layer)
        out[f"conv{n}_flops"] = np.array(mk.conv_flops(dims, layer.schedule))
        out[f"conv{n}_in_index"] = np.array(layer.in_index)
        # the reference's own fastest CPU path, for context only
        out[f"conv{n}_y_specialized"] = mk.conv_forward(x, layer, "specialized")

    # 3. activation: all modes, k in {1,2,3}, K in {1, N_B/2, N_B}, shuffled indices
    n = 0
    for k in (1, 2, 3):
        sig = mk.Signature((1,) * k)
        nb = sig.n_blades
        for mode in (0, 1, 2):
            for K in sorted({1, max(1, nb // 2), nb}):
                idx = np.arange(nb)
                rng.shuffle(idx)
                ki = tuple(int(i) for i in idx[:K])
                C = 13
                w = bvec = None
                if mode == 0:
                    w = (rng.standard_normal((C, K)) / np.sqrt(K)).astype(np.float32)
                    bvec = (rng.standard_normal(C) * 0.1).astype(np.float32)
                cfg = mk.make_activation_config(sig, mode, ki, w, bvec)
                x = (rng.standard_normal((3, C, nb)) * 2).astype(np.float32)
                out[f"act{n}_meta"] = np.array([k, mode, K], dtype=np.int64)
                out[f"act{n}_ki"] = np.array(ki, dtype=np.int64)
                out[f"act{n}_x"] = x
                if mode == 0:
                    out[f"act{n}_w"] = w
                    out[f"act{n}_bias"] = bvec
                out[f"act{n}_y"] = act.activation_reference(x, cfg)
                out[f"act{n}_y_specialized"] = act.activation_forward(x, cfg, "specialized")
                n += 1
    out["act_count"] = np.array(n)

    # 4. spatial activation through the server fold (serve.py:108-117)
    for mode in (0, 1, 2):
        sig = mk.Signature((1, 1, 1))
        C, P = 8, 6
        ki = tuple(range(8))
        w = bvec = None
        if mode == 0:
            w = rng.uniform(-0.5, 0.5, (C, 8)).astype(np.float32)
            bvec = (rng.standard_normal(C) * 0.1).astype(np.float32)
        cfg = mk.make_activation_config(sig, mode, ki, w, bvec)
        x = rng.standard_normal((2, C, P, 8)).astype(np.float32)
        out[f"sact{mode}_x"] = x
        if mode == 0:
            out[f"sact{mode}_w"] = w
            out[f"sact{mode}_bias"] = bvec
        out[f"sact{mode}_y"] = serve._forward("activation", cfg, x, "reference")

    # 5. blocks composed from reference primitives (block.ts:134-148 semantics;
    #    'same' + residual per DESIGN.md D1)
    for name, g, padding, residual, mode in [
        ("blk2v", (1, 1), "valid", False, 0),
        ("blk2s", (1, 1), "same", True, 0),
        ("blk3s", (1, 1, 1), "same", True, 2),
        ("blk3v", (1, -1, 0), "valid", False, 1),
    ]:
        k = len(g)
        nb = 1 << k
        B, C, d = 2, 3, 6
        sig = mk.Signature(g)
        pad = 1 if padding == "same" else 0
        x = rng.standard_normal((B, C, d ** k, nb)).astype(np.float32)
        fan = C * nb * 9 if k == 2 else C * nb * 27
        f1 = rng.uniform(-1, 1, (nb, C, C, 3 ** k)).astype(np.float32) / np.float32(np.sqrt(fan))
        b1 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
        f2 = rng.uniform(-1, 1, (nb, C, C, 3 ** k)).astype(np.float32) / np.float32(np.sqrt(fan))
        b2 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
        aw = ab = None
        if mode == 0:
            aw = rng.uniform(-0.5, 0.5, (C, nb)).astype(np.float32)
            ab = (rng.standard_normal(C) * 0.1).astype(np.float32)
        acfg = mk.make_activation_config(sig, mode, tuple(range(nb)), aw, ab)

        def conv(xx, dd, f, b):
            if pad:
                xs = xx.reshape((B, C) + (dd,) * k + (nb,))
                xs = np.pad(xs, [(0, 0), (0, 0)] + [(1, 1)] * k + [(0, 0)])
                xx = xs.reshape(B, C, (dd + 2) ** k, nb)
                dd = dd + 2
            dims = mk.Dims(B=B, C_in=C, C_out=C, d_image=dd, d_filter=3, k=k)
            return mk.conv_reference(xx, mk.make_conv_layer(dims, sig, f, b, W=1)), dd - 2

        y1, d1 = conv(x, d, f1, b1)
        y2 = serve._forward("activation", acfg, y1, "reference")
        y3, d3 = conv(y2, d1, f2, b2)
        if residual:
            y3 = (y3 + x).astype(np.float32)
        out[f"{name}_meta"] = np.array(list(g) + [0] * (3 - k) + [k, pad, int(residual), mode, B, C, d])
        for nm, v in [("x", x), ("f1", f1), ("b1", b1), ("f2", f2), ("b2", b2), ("y", y3)]:
            out[f"{name}_{nm}"] = v
        if mode == 0:
            out[f"{name}_aw"] = aw
            out[f"{name}_ab"] = ab

    # 6. parity metric known answers (bench.py:74-96)
    a = rng.standard_normal(50)
    b = a + rng.standard_normal(50) * 1e-3
    out["mre_a"] = a
    out["mre_b"] = b
    out["mre_default"] = np.array(mk.max_rel_error(a, b))
    out["mre_floor1"] = np.array(mk.max_rel_error(a, b, floor=1.0))
    out["mae"] = np.array(mk.max_abs_error(a, b))

    # 7. flop models (activation.py:419-433)
    out["act_flops"] = np.array([act.activation_flops(5, 7, nb, K, m)
                                 for nb, K in ((4, 4), (8, 8), (8, 3)) for m in (0, 1, 2)])
    out["act_flops_unit"] = np.array(act.activation_flops(1, 1, 4, 2, 0))

    # 8. MVTF bytes (layout.py:183-196)
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "t.mvtf")
        arr = rng.standard_normal((2, 3, 4)).astype(np.float32)
        mk.write_tensor(p, arr, mk.LayoutTag.CONV_INPUT, 2)
        out["mvtf_arr"] = arr
        out["mvtf_bytes"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)

    # 9. Clifford linear layer (linear.py:58-102): fp64 oracle and the gemm variant
    lrng = np.random.default_rng(7)
    lin_cases = [((1,), 5, 3, 4), ((1, 1), 7, 6, 5), ((0, 1), 3, 2, 3), ((1, 1, 1), 9, 5, 4),
                 ((1, -1, 0), 4, 3, 6), ((-1, 0, 1), 2, 8, 8)]
    for n, (g, B, ci, co) in enumerate(lin_cases):
        sig = mk.Signature(g)
        nb = sig.n_blades
        w = (lrng.standard_normal((nb, co, ci)) / np.sqrt(ci * nb)).astype(np.float32)
        b = (lrng.standard_normal((nb, co)) * 0.1).astype(np.float32)
        x = lrng.standard_normal((B, ci, nb)).astype(np.float32)
        layer = mk.make_linear_layer(sig, w, b)
        out[f"lin{n}_g"] = np.array(g, dtype=np.int64)
        out[f"lin{n}_x"] = x
        out[f"lin{n}_w"] = w
        out[f"lin{n}_b"] = b
        out[f"lin{n}_y"] = mk.linear_reference(x, layer)
        out[f"lin{n}_y_gemm"] = mk.linear_forward(x, layer, "gemm")
        out[f"lin{n}_flops"] = np.array(mk.linear_flops(B, ci, co, layer.schedule))
    out["lin_count"] = np.array(len(lin_cases))

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    sys.exit(main())
