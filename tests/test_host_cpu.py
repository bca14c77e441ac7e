"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares; host-side algebra (the same C code that builds the device
kernels) matches the reference golden tables; host validation mirrors the
reference's exceptions; MVTF wire format; FLOP models. No GPU compute."""

import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2507_01040_b200 as M
from paper_2507_01040_b200 import _lib, errors as E

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "clifford_b200.h")).read()
    return sorted(set(re.findall(r"\b(cl_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 19
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert lib.cl_version().startswith(b"clifford_b200")


def test_library_is_sm100a_native():
    # the fatbin carries sm_100a SASS with tcgen05 / TMA instructions
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UTCHMMA" in out or "UTCQMMA" in out or "UTCIMMA" in out
    assert "UTMALDG" in out


def test_product_tables_via_c_abi(golden):
    for s in golden["sig_list"]:
        g = tuple(int(v) for v in str(s).split("_"))
        tgt, cof = M.product_table(M.Signature(g))
        np.testing.assert_array_equal(tgt, golden[f"table_target_{s}"])
        np.testing.assert_array_equal(cof, golden[f"table_coeff_{s}"])
        assert M.schedule_terms(M.Signature(g)) == len(golden[f"sched_{s}"])


def test_blade_product_known_answers():
    assert M.blade_product(1, 1, M.Signature((1, 1))) == (0, 1)
    assert M.blade_product(1, 1, M.Signature((-1, 1))) == (0, -1)
    assert M.blade_product(1, 1, M.Signature((0, 1))) == (0, 0)
    assert M.blade_product(2, 1, M.Signature((1, 1))) == (3, -1)
    assert M.blade_product(3, 3, M.Signature((1, 1))) == (0, -1)


def test_signature_validation():
    with pytest.raises(E.InvalidSignature):
        M.validate_signature((0, 0))
    with pytest.raises(E.InvalidMetricValue):
        M.validate_signature((1, 2))
    with pytest.raises(E.InvalidSignature):
        M.validate_signature(())
    assert M.validate_signature((1.0, -1.0, 0.0)).g == (1, -1, 0)
    g = (_lib.C.c_int32 * 2)(0, 0)
    assert _lib.load().cl_validate_signature(g, 2) == 1
    g = (_lib.C.c_int32 * 2)(1, 2)
    assert _lib.load().cl_validate_signature(g, 2) == 2
    with pytest.raises(E.InvalidMetricValue):
        _lib.check(2)


def test_dims_and_layer_validation():
    with pytest.raises(E.ShapeMismatch):
        M.Dims(1, 1, 1, 3, 4, 2)
    with pytest.raises(E.ShapeMismatch):
        M.Dims(0, 1, 1, 3, 1, 2)
    d = M.Dims(2, 3, 4, 6, 3, 2)
    assert d.input_shape() == (2, 3, 36, 4) and d.output_shape() == (2, 4, 16, 4)
    sig = M.Signature((1, 1))
    f = np.zeros(d.filters_shape(), np.float32)
    b = np.zeros(d.bias_shape(), np.float32)
    with pytest.raises(E.ShapeMismatch):
        M.make_conv_layer(d, M.Signature((1, 1, 1)), f, b)
    with pytest.raises(E.ShapeMismatch):
        M.make_conv_layer(d, sig, f[:, :2], b)
    with pytest.raises(E.ShapeMismatch):
        M.make_conv_layer(d, sig, f, b[:, :1])
    with pytest.raises(E.ShapeMismatch):
        M.make_conv_layer(d, sig, f, b, W=0)
    layer = M.make_conv_layer(d, sig, f, b, padding="same")
    assert layer.d_out == 6 and layer.output_shape() == (2, 4, 36, 4)
    assert not layer.filters.flags.writeable


def test_activation_config_validation():
    s2 = M.Signature((1, 1))
    with pytest.raises(E.ModeConfigMismatch):
        M.make_activation_config(s2, M.AggMode.LINEAR, (0, 1))
    with pytest.raises(E.ModeConfigMismatch):
        M.make_activation_config(s2, M.AggMode.SUM, (0, 1), weight=np.ones((3, 2)), bias=np.ones(3))
    with pytest.raises(E.IndexOutOfRange):
        M.make_activation_config(s2, M.AggMode.SUM, (1, 1))
    with pytest.raises(E.IndexOutOfRange):
        M.make_activation_config(s2, M.AggMode.MEAN, (0, 4))
    with pytest.raises(E.ShapeMismatch):
        M.make_activation_config(s2, M.AggMode.LINEAR, (0, 1), weight=np.ones((3, 3)), bias=np.ones(3))
    cfg = M.make_activation_config(M.Signature((1,)), 1, (0,))
    assert cfg.agg_mode is M.AggMode.SUM and cfg.K == 1


def test_flop_models(golden):
    for n in range(10):
        g = tuple(int(v) for v in golden[f"conv{n}_g"])
        B, ci, co, di, df, k = (int(v) for v in golden[f"conv{n}_dims"])
        assert M.conv_flops(M.Dims(B, ci, co, di, df, k), M.Signature(g)) == int(golden[f"conv{n}_flops"])
    got = [M.activation_flops(5, 7, nb, K, m) for nb, K in ((4, 4), (8, 8), (8, 3)) for m in (0, 1, 2)]
    np.testing.assert_array_equal(got, golden["act_flops"])
    # BASELINE config FLOP counts
    assert M.conv_flops(M.Dims(8, 16, 16, 32, 3, 2), M.Signature((1, 1))) == 531_302_400
    assert M.conv_flops(M.Dims(16, 32, 32, 32, 3, 3), M.Signature((1, 1, 1))) == 1_528_934_400_000
    assert M.conv_flops(M.Dims(16, 32, 32, 32, 3, 3), M.Signature((1, -1, 0))) == 1_146_728_448_000
    assert M.conv_flops(M.Dims(256, 64, 64, 32, 3, 3), M.Signature((1, 1, 1)), padding="same") == 118_751_550_767_104


def test_mvtf_roundtrip(tmp_path, golden):
    p = tmp_path / "t.mvtf"
    M.write_tensor(p, golden["mvtf_arr"], M.LayoutTag.CONV_INPUT, 2)
    assert p.read_bytes() == golden["mvtf_bytes"].tobytes()
    tf = M.read_tensor(p)
    np.testing.assert_array_equal(tf.data, golden["mvtf_arr"])
    assert tf.tag == M.LayoutTag.CONV_INPUT and tf.k == 2
    good = p.read_bytes()
    # malformed files (tests/test_layout.py:133-165 of the reference): bad magic,
    # truncated header, unknown version / dtype code, short or long payload
    import struct
    bad = [b"XXXX" + good[4:], good[:10], good[:4] + struct.pack("<I", 2) + good[8:],
           good[:8] + struct.pack("<I", 7) + good[12:], good[:-4], good + b"\0\0\0\0"]
    for raw in bad:
        p.write_bytes(raw)
        with pytest.raises(E.ShapeMismatch):
            M.read_tensor(p)
    # float64 payloads are representable (and rejected by the server, not here)
    M.write_tensor(p, np.zeros((2, 3)), M.LayoutTag.GENERIC, 0)
    assert M.read_tensor(p).data.dtype == np.float64
    with pytest.raises(E.ShapeMismatch):
        M.write_tensor(p, np.zeros(3, np.int32))


def test_no_oracle_in_product():
    # the product package must never import the oracle (no CPU fallback)
    pkg = os.path.join(ROOT, "paper_2507_01040_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith(".py"):
                src = open(os.path.join(dp, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_linear_validation_and_flops(golden):
    s2 = M.Signature((1, 1))
    with pytest.raises(E.ShapeMismatch):
        M.make_linear_layer(s2, np.zeros((3, 2, 2)), np.zeros((4, 2)))
    with pytest.raises(E.ShapeMismatch):
        M.make_linear_layer(s2, np.zeros((4, 2, 3)), np.zeros((4, 3)))
    layer = M.make_linear_layer(s2, np.zeros((4, 2, 3)), np.zeros((4, 2)))
    assert (layer.C_in, layer.C_out) == (3, 2)
    for n in range(int(golden["lin_count"])):
        g = tuple(int(v) for v in golden[f"lin{n}_g"])
        x, w = golden[f"lin{n}_x"], golden[f"lin{n}_w"]
        assert M.linear_flops(x.shape[0], x.shape[1], w.shape[1], M.Signature(g)) == int(golden[f"lin{n}_flops"])


def _basis(g):
    lib = _lib.load()
    ncol, w = _lib.C.c_int(), _lib.C.c_int()
    T = (_lib.C.c_int8 * 64)()
    ok = lib.cl_basis_info(_lib.int32_array(g), len(g), _lib.C.byref(ncol), _lib.C.byref(w), T)
    return ok, ncol.value, w.value, np.array(list(T), np.int64).reshape(8, 8)


@pytest.mark.parametrize("g", O.all_signatures(3))
def test_change_of_basis_is_exact_block_diagonalisation(g):
    """x' = T x turns left multiplication by any multivector into
    ncol identical w x w blocks (checked against the oracle's Cayley tensor);
    for the degenerate signatures the blocks are lower block-triangular."""
    ok, ncol, w, T = _basis(g)
    k = len(g)
    expect = k >= 2 and all(g) and not (k == 2 and g == (-1, -1)) and g not in [(-1, -1, -1), (1, 1, -1), (1, -1, 1), (-1, 1, 1)]
    # degenerate k = 3 with one null generator whose complement pair is M2(R) (not the quaternions)
    expect = expect or (k == 3 and g.count(0) == 1 and tuple(v for v in g if v) != (-1, -1))
    if not ok:
        assert not expect, f"no basis found for {g}"
        return
    nb = 1 << k
    T = T[:nb, :nb]
    np.testing.assert_array_equal(T @ T.T, 2 * np.eye(nb, dtype=np.int64))
    cay = O.cayley(g)
    rng = np.random.default_rng(0)
    f = rng.standard_normal(nb)
    L = np.einsum("i,ijt->tj", f, cay)  # (f x)[t] = sum_j L[t, j] x[j]
    A = T @ L @ T.T / 2
    for c in range(ncol):
        for c2 in range(ncol):
            blk = A[c * w:(c + 1) * w, c2 * w:(c2 + 1) * w]
            if c == c2:
                np.testing.assert_allclose(blk, A[:w, :w], atol=1e-12)
            else:
                np.testing.assert_allclose(blk, 0, atol=1e-12)


PLAN_KEYS = ["basis", "halo", "pair", "ks", "gs", "tps", "stages", "n_tile", "n_ntiles", "tx", "ty", "tz",
             "smem", "epx", "bcls", "tmem_cols"]


def plan_info(g, C_in, C_out, d, df, padding, prec):
    lib = _lib.load()
    out = (_lib.C.c_int64 * 16)()
    _lib.check(lib.cl_conv_plan_info(_lib.int32_array(g), len(g), C_in, C_out, d, df, padding, prec, out))
    return dict(zip(PLAN_KEYS, list(out)))


@pytest.mark.parametrize("prec", [0, 1, 2, 3])
def test_planner_cfg5_layer(prec):
    """cfg5's conv (3-D, C=64, 32^3 same): change of basis, halo reuse and the
    2-SM pair in every mode; int8 keeps one accumulator
    slot (4 levels x 128 columns = all of TMEM); 3xTF32 rotates three 128-column
    slots (the A_hi*B_hi accumulation groups, drained every 192 reduction
    elements) in front of the tile-long cross-term accumulator (4 x 128 = 512)."""
    p = plan_info((1, 1, 1), 64, 64, 32, 3, 1, prec)
    assert p["basis"] == 1 and p["halo"] == 1 and p["pair"] == 1
    assert (p["tx"], p["ty"], p["tz"]) == (4, 16, 1)  # one 8-row core-matrix group per halo row
    assert p["smem"] <= 232448 and p["stages"] >= 4 and p["tmem_cols"] == 512
    assert p["epx"] == 4  # 32-byte pixels as 8-byte TMA elements
    if prec == 0:
        assert p["n_tile"] == 128 and p["n_ntiles"] == 2 and p["bcls"] == 1
    elif prec == 3:
        assert p["n_tile"] == 128 and p["n_ntiles"] == 2 and p["ks"] * p["tps"] * 8 <= 192
    else:
        assert p["n_tile"] == 256 and p["n_ntiles"] == 1


def test_planner_variants():
    # degenerate signature: the block-triangular basis (cfg4b), epilogue pattern class 2
    p = plan_info((1, -1, 0), 32, 32, 32, 3, 0, 0)
    assert p["basis"] == 1 and p["bcls"] == 2
    # quaternion pair + null generator: no basis, 32-byte protocol rows, no halo for tf32
    p = plan_info((-1, -1, 0), 8, 8, 12, 3, 0, 1)
    assert p["basis"] == 0 and p["halo"] == 0 and p["epx"] == 0
    # 3xTF32 pairs only with halo reuse
    assert plan_info((-1, -1, 0), 8, 8, 12, 3, 0, 3)["pair"] == 0
    assert plan_info((1, 1, 1), 16, 16, 12, 3, 1, 3)["pair"] == 1
    # 1-D: no halo (a tile row spans samples)
    assert plan_info((1,), 16, 16, 64, 3, 0, 0)["halo"] == 0
    # fp32 K limit (4 s32 levels): Unsupported beyond K = 32000 is checked at create; the planner still plans
    with pytest.raises(E.ConfigInvalid):
        plan_info((1, 1), 4, 4, 8, 3, 0, 7)


# ---- reference-API host helpers ----------------

def test_schedule_for_matches_reference_golden(golden):
    """specialize.schedule_for (specialize.py:49-69) term by term, all 36 signatures."""
    for s in golden["sig_list"]:
        g = tuple(int(v) for v in str(s).split("_"))
        sch = M.schedule_for(M.Signature(g))
        got = np.array([[t.out_blade, t.a_blade, t.b_blade, int(t.negate)] for t in sch.terms], np.int64)
        np.testing.assert_array_equal(got, golden[f"sched_{s}"])
        assert M.schedule_flop_count(sch) == M.schedule_flop_count(M.Signature(g)) == 2 * len(sch)


def test_product_table_object_and_cayley():
    sig = M.Signature((1, -1, 0))
    t = M.product_table(sig)
    assert isinstance(t, M.BladeProductTable) and t.sig == sig
    tgt, cof = t  # tuple unpacking still works
    assert tgt is t.target and cof is t.coeff and not t.coeff.flags.writeable
    np.testing.assert_array_equal(M.cayley_tensor(sig), O.cayley(sig.g))


def test_gather_index_table_golden(golden):
    for n in range(10):
        B, ci, co, di, df, k = (int(v) for v in golden[f"conv{n}_dims"])
        dims = M.Dims(B, ci, co, di, df, k)
        np.testing.assert_array_equal(M.gather_index_table(dims), golden[f"conv{n}_in_index"])
    # 2-D, d_image 4, 3x3 filter: output (0,0) reads rows 0..2 of a 4-wide image
    t = M.gather_index_table(M.Dims(1, 1, 1, 4, 3, 2))
    assert t.shape == (4, 9) and list(t[0]) == [0, 1, 2, 4, 5, 6, 8, 9, 10]


def test_conv_layer_reference_fields():
    rng = np.random.default_rng(3)
    dims = M.Dims(2, 3, 4, 6, 3, 2)
    f = rng.standard_normal(dims.filters_shape()).astype(np.float32)
    b = rng.standard_normal(dims.bias_shape()).astype(np.float32)
    layer = M.make_conv_layer(dims, M.Signature((0, 1)), f, b, W=4, U=2)
    assert layer.L == 8 and len(layer.schedule) == 12
    np.testing.assert_array_equal(layer.in_index, O.gather_index_table(6, 3, 2))
    # the reference call shape conv_flops(dims, layer.schedule) (conv.py:384-387)
    assert M.conv_flops(dims, layer.schedule) == M.conv_flops(dims, layer) == \
        O.conv_flops(2, 3, 4, 4, 3, (0, 1))


def test_reference_cpu_variants_are_not_aliases():
    """variant="reference" (or any reference CPU variant) must not silently run
    the B200 kernel: a harness verifying variants against "reference" would
    otherwise compare the B200 output with itself."""
    rng = np.random.default_rng(0)
    nb = 4
    dims = M.Dims(2, 2, 2, 6, 3, 2)
    f = rng.standard_normal(dims.filters_shape()).astype(np.float32)
    b = np.zeros(dims.bias_shape(), np.float32)
    layer = M.make_conv_layer(dims, M.Signature((1, 1)), f, b)
    x = np.zeros(dims.input_shape(), np.float32)
    for v in ("reference", "kernelized", "packed", "specialized"):
        with pytest.raises(ValueError, match="not provided by the B200 path"):
            M.conv_forward(x, layer, v)
    with pytest.raises(ValueError, match="unknown conv variant"):
        M.conv_forward(x, layer, "nonsense")
    cfg = M.make_activation_config(M.Signature((1, 1)), 1, (0, 1))
    for v in ("reference", "hoisted", "packed", "specialized"):
        with pytest.raises(ValueError, match="not provided"):
            M.activation_forward(np.zeros((1, 1, nb), np.float32), cfg, v)
    lin = M.make_linear_layer(M.Signature((1, 1)), np.zeros((nb, 2, 2), np.float32), np.zeros((nb, 2), np.float32))
    for v in ("reference", "gemm"):
        with pytest.raises(ValueError, match="not provided"):
            M.linear_forward(np.zeros((1, 2, nb), np.float32), lin, v)


def test_numpy_out_is_validated_before_the_c_abi():
    """A caller-supplied numpy `out` goes straight to the C-ABI: wrong shape,
    dtype, layout or a read-only array must raise ShapeMismatch first."""
    rng = np.random.default_rng(1)
    dims = M.Dims(2, 2, 3, 6, 3, 2)
    layer = M.make_conv_layer(dims, M.Signature((1, 1)), rng.standard_normal(dims.filters_shape()).astype(np.float32),
                              np.zeros(dims.bias_shape(), np.float32))
    x = np.zeros(dims.input_shape(), np.float32)
    shape = layer.output_shape()
    ro = np.zeros(shape, np.float32)
    ro.flags.writeable = False
    bad = [np.zeros(shape[:-1] + (shape[-1] + 1,), np.float32), np.zeros(shape, np.float16),
           np.zeros(shape[::-1], np.float32).T, ro, [0.0]]
    for out in bad:
        with pytest.raises(E.ShapeMismatch):
            M.conv_forward(x, layer, out=out)
    cfg = M.make_activation_config(M.Signature((1, 1)), 2, (0, 1, 2, 3))
    with pytest.raises(E.ShapeMismatch):
        M.activation_forward(np.zeros((2, 3, 4), np.float32), cfg, out=np.zeros((2, 3, 5), np.float32))
    blk = M.make_basic_block(M.Signature((1, 1)), 1, 2, 2, 2, 6, np.zeros((4, 2, 2, 9), np.float32),
                             np.zeros((4, 2), np.float32), 1, np.zeros((4, 2, 2, 9), np.float32),
                             np.zeros((4, 2), np.float32))
    with pytest.raises(E.ShapeMismatch):
        M.block_forward(np.zeros(blk.input_shape(), np.float32), blk, out=np.zeros((1, 2, 36, 4), np.float64))
    lin = M.make_linear_layer(M.Signature((1,)), np.zeros((2, 3, 2), np.float32), np.zeros((2, 3), np.float32))
    with pytest.raises(E.ShapeMismatch):
        M.linear_forward(np.zeros((4, 2, 2), np.float32), lin, out=np.zeros((4, 2, 2), np.float32))


def test_reference_patch_applies_to_baseline_ref(tmp_path):
    """tests/reference_b200.patch applies cleanly to
    the unmodified reference package in baseline/_ref."""
    import shutil
    import subprocess
    ref = os.path.join(ROOT, "baseline", "_ref", "mvkernels")
    if not os.path.isdir(ref):
        pytest.skip("baseline/_ref not installed")
    shutil.copytree(ref, tmp_path / "mvkernels")
    r = subprocess.run(["patch", "-p1", "--dry-run", "-d", str(tmp_path), "-i",
                        os.path.join(ROOT, "tests", "reference_b200.patch")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_production_library_ignores_the_environment():
    """The CL_* A/B timing switches and the fault injection are compiled only
    into the diagnostic build (libclifford_b200_ab.so); the production library
    contains no getenv of them."""
    from paper_2507_01040_b200 import build as B
    prod = open(B.LIB, "rb").read()
    ab = open(B.LIB_AB, "rb").read()
    for name in (b"CL_NO_PAIR", b"CL_NO_HALO", b"CL_DBG_SKIP", b"CL_DBG_FLIP_COEFF", b"CL_TPS", b"CL_NO_GRAPH"):
        assert name not in prod, name
        assert name in ab, name


def test_torch_operator_registration():
    """The C-ABI is registered as PyTorch operators (the package's binding):
    host-only operators run without a GPU and C-ABI failures come back as the
    reference's exception classes."""
    import torch
    from paper_2507_01040_b200 import _ops
    o = _ops.ops()
    assert o is torch.ops.clifford_b200
    assert torch.ops.clifford_b200.version().startswith("clifford_b200")
    assert list(_ops.op("blade_product", 2, 1, [1, 1])) == [3, -1]
    assert _ops.op("schedule_terms", [1, -1, 0]) == 48
    with pytest.raises(E.InvalidSignature):
        _ops.op("validate_signature", [0, 0])
    with pytest.raises(E.InvalidMetricValue):
        _ops.op("validate_signature", [1, 2])
    with pytest.raises(E.IndexOutOfRange):
        _ops.op("blade_product", 9, 1, [1, 1])
    with pytest.raises(E.ShapeMismatch, match="CUDA tensor"):
        _ops.op("conv_forward", 0, torch.zeros(4), 1, torch.zeros(4))
    for name in ("conv_create", "conv_forward", "conv_forward_host", "act_forward", "act_preactivation",
                 "act_gather", "block_forward", "block_forward_host", "linear_create", "expand_kernel"):
        assert hasattr(o, name), name


def test_geometric_product_and_metrics():
    """Host helpers re-exported for drop-in callers (algebra.py:155-173,
    bench.py:74-96), checked against the oracle and known answers."""
    rng = np.random.default_rng(3)
    for g in [(1, 1), (1, -1, 0), (-1,), (0, 1, 1)]:
        sig = M.Signature(g)
        a = rng.standard_normal((5, sig.n_blades)).astype(np.float32)
        b = rng.standard_normal((5, sig.n_blades)).astype(np.float32)
        got = M.geometric_product(a, b, M.product_table(sig))
        assert got.dtype == np.float32
        want = np.einsum("...i,ijt,...j->...t", a.astype(np.float64), O.cayley(g), b.astype(np.float64))
        np.testing.assert_allclose(got, want.astype(np.float32), rtol=1e-6, atol=1e-7)
    with pytest.raises(E.DimensionMismatch):
        M.geometric_product(np.zeros(3), np.zeros(4), M.product_table(M.Signature((1, 1))))
    assert M.max_rel_error(np.array([1.0, 0.0]), np.array([1.0, 0.001])) == pytest.approx(0.001 / 0.011)
    assert M.max_abs_error(np.zeros(3), np.array([0.0, -2.0, 1.0])) == 2.0
    assert M.max_rel_error(np.zeros(0), np.zeros(0)) == 0.0
    with pytest.raises(E.VerificationFailed):
        M.max_abs_error(np.zeros(2), np.zeros(3))
    assert float(M.sigmoid(4.0)) == pytest.approx(0.98201379003790844, abs=1e-15)  # tests/test_activation.py:38-40
    assert float(M.sigmoid(0.0)) == 0.5
    assert float(M.sigmoid(-1000.0)) == 0.0
