"""GPU parity: the B200 path (through the C-ABI) against the CPU oracle.

Tolerances (D3, the reference's own metric bench.py:74-88):
  * expanded kernel: bit-exact (+-0 equal)
  * conv/block fp32 (int8-slice exact accumulation): max_rel_error(floor=1e-2) <= 1e-4
  * conv 3xTF32: max_rel_error(floor=max|ref|) <= 1e-5 (normwise; 5e-5 for full-size
    blocks, tests/test_gpu_configs.py)
  * conv TF32 / BF16: max_rel_error(floor=max|ref|) <= 2e-2 (stated bound)
  * activation: max_abs_error <= 1e-5 (activation.py:7, tests/test_activation.py:160-173)
"""

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2507_01040_b200 as M  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def make_conv(rng, g, B, ci, co, d, df, prec="fp32", padding="valid", fscale=None):
    k = len(g)
    nb = 1 << k
    x = rng.standard_normal((B, ci, d ** k, nb)).astype(np.float32)
    fan = ci * nb * df ** k
    bound = fscale if fscale is not None else 1.0 / np.sqrt(fan)
    f = rng.uniform(-bound, bound, (nb, ci, co, df ** k)).astype(np.float32)
    b = (rng.standard_normal((nb, co)) * 0.01).astype(np.float32)
    layer = M.make_conv_layer(M.Dims(B, ci, co, d, df, k), M.Signature(tuple(g)), f, b,
                              precision=prec, padding=padding)
    pad = (df - 1) // 2 if padding == "same" else 0
    return x, f, b, layer, pad


def run_dev(fn, x, *a):
    return fn(torch.from_numpy(x).cuda(), *a).cpu().numpy()


def assert_conv_close(y, ref, prec, K=0):
    """fp32 and 3xTF32 are the FP32-accurate modes. fp32 (exact int8-digit
    accumulation) meets the reference metric (max_rel_error, floor 1e-2,
    bench.py:74-88) <= 1e-4 everywhere. 3xTF32 drains its tensor-core
    A_hi*B_hi accumulator every 192 reduction elements into fp32 registers (DESIGN.md
    "3xTF32 accumulation groups"), so its error no longer grows with K:
    normwise <= 2e-6 (fp32-class; measured 1e-7 .. 4e-7). The floor-1e-2
    metric is absolute near zero, so for fp32-class arithmetic it scales with
    the output magnitude: <= 1e-4 is asserted on the BASELINE configs at full
    size (test_gpu_configs.py, unit-scale outputs), <= 3e-4 on these small
    cases with up to 12x-scaled channels (the reference's own fp32 path: 3.6e-4
    at cfg4)."""
    if prec == "fp32":
        assert O.max_rel_error(y, ref) <= 1e-4, O.max_rel_error(y, ref)
    elif prec == "3xtf32":
        e_ref = O.max_rel_error(y, ref)
        e = O.max_rel_error(y, ref, floor=float(np.abs(ref).max()) + 1e-30)
        assert e_ref <= 3e-4 and e <= 2e-6, (e_ref, e, K)
    else:
        e = O.max_rel_error(y, ref, floor=float(np.abs(ref).max()) + 1e-30)
        assert e <= 2e-2, e


# ---- (1) kernel construction: bit-exact for all 36 signatures ----------------

@pytest.mark.parametrize("g", O.all_signatures(3))
def test_expanded_kernel_bit_exact_all_signatures(g):
    rng = np.random.default_rng(abs(hash(g)) % 2 ** 32)
    k = len(g)
    nb = 1 << k
    f = rng.standard_normal((nb, 3, 2, 2 ** k)).astype(np.float32)
    layer = M.make_conv_layer(M.Dims(1, 3, 2, 3, 2, k), M.Signature(g), f, np.zeros((nb, 2), np.float32))
    W = M.build_expanded_kernel(layer).cpu().numpy()
    assert np.array_equal(W, O.expanded_kernel(f, g))


def test_expanded_kernel_golden(golden):
    for n in range(10):
        g = tuple(int(v) for v in golden[f"conv{n}_g"])
        B, ci, co, di, df, k = (int(v) for v in golden[f"conv{n}_dims"])
        layer = M.make_conv_layer(M.Dims(B, ci, co, di, df, k), M.Signature(g),
                                  golden[f"conv{n}_f"], golden[f"conv{n}_b"])
        W = M.build_expanded_kernel(layer).cpu().numpy()
        assert np.array_equal(W, golden[f"conv{n}_W"]), n


# ---- (2) convolution -------------------------------------------------------------

@pytest.mark.parametrize("prec", ["fp32", "3xtf32", "tf32", "bf16"])
def test_conv_golden_cases(golden, prec):
    for n in range(10):
        g = tuple(int(v) for v in golden[f"conv{n}_g"])
        B, ci, co, di, df, k = (int(v) for v in golden[f"conv{n}_dims"])
        layer = M.make_conv_layer(M.Dims(B, ci, co, di, df, k), M.Signature(g),
                                  golden[f"conv{n}_f"], golden[f"conv{n}_b"], precision=prec)
        y = run_dev(M.conv_forward, golden[f"conv{n}_x"], layer)
        assert_conv_close(y, golden[f"conv{n}_y"], prec)


SIGS = [(1,), (-1,), (1, 1), (-1, 1), (0, 1), (1, 1, 1), (1, -1, 0), (-1, 0, 1), (0, 0, 1)]


@pytest.mark.parametrize("prec", ["fp32", "3xtf32", "tf32", "bf16"])
@pytest.mark.parametrize("g", SIGS)
@pytest.mark.parametrize("padding", ["valid", "same"])
def test_conv_signatures(prec, g, padding):
    rng = np.random.default_rng(7)
    k = len(g)
    d = {1: 40, 2: 9, 3: 6}[k]
    x, f, b, layer, pad = make_conv(rng, g, 2, 5, 6, d, 3, prec, padding)
    y = run_dev(M.conv_forward, x, layer)
    assert_conv_close(y, O.conv_ref(x, f, b, g, d, 3, pad), prec)


@pytest.mark.parametrize("prec", ["fp32", "3xtf32", "tf32", "bf16"])
@pytest.mark.parametrize("shape", [
    ((1, 1), 1, 1, 1, 4, 1),      # 1x1 conv, single channel
    ((1, 1), 3, 7, 3, 5, 5),      # d_out = 1
    ((1, 1), 2, 3, 9, 40, 3),     # odd channels, several x tiles
    ((1, 1), 1, 64, 64, 16, 3),
    ((1, 1, 1), 1, 3, 5, 7, 1),
    ((1, 1, 1), 2, 16, 16, 9, 3),
    ((1, 1, 1), 1, 5, 3, 4, 4),   # even filter, valid
    ((1, -1), 3, 33, 17, 11, 3),  # N not a multiple of 32
    ((1,), 37, 3, 5, 9, 3),       # 1-D: tile rows span samples; odd channels
    ((-1,), 3, 16, 16, 300, 5),   # 1-D: several position tiles
    ((1, 1), 3, 20, 12, 23, 7),   # 2-D wide filter: halo 14 x 22
    ((1, 1, 1), 3, 9, 40, 10, 5), # 3-D d_f = 5 under the change of basis: halo 8 x 20 x 5
    ((1, -1, 0), 1, 24, 72, 8, 3),  # degenerate basis, two N tiles (int8), ghost tile of a CTA pair
    ((0, 0, 1), 2, 6, 10, 6, 2),  # no basis in 3-D: 32-byte protocol rows (tf32 modes)
])
def test_conv_edge_shapes(prec, shape):
    g, B, ci, co, d, df = shape
    rng = np.random.default_rng(11)
    x, f, b, layer, pad = make_conv(rng, g, B, ci, co, d, df, prec)
    y = run_dev(M.conv_forward, x, layer)
    assert_conv_close(y, O.conv_ref(x, f, b, g, d, df, pad), prec, K=ci * (1 << len(g)) * df ** len(g))


def test_conv_identity_filter():
    # tests/test_conv.py:31-35: scalar-1 filter, zero bias -> identity
    dims = M.Dims(B=2, C_in=3, C_out=3, d_image=4, d_filter=1, k=2)
    f = np.zeros(dims.filters_shape(), np.float32)
    f[0] = np.eye(3, dtype=np.float32)[:, :, None]
    layer = M.make_conv_layer(dims, M.Signature((1, 1)), f, np.zeros(dims.bias_shape(), np.float32))
    x = np.random.default_rng(0).standard_normal(dims.input_shape()).astype(np.float32)
    np.testing.assert_allclose(run_dev(M.conv_forward, x, layer), x, rtol=1e-6, atol=1e-7)


def test_conv_bias_broadcast():
    # tests/test_conv.py:37-45 (k=2 here): zero input -> bias everywhere
    dims = M.Dims(B=2, C_in=2, C_out=3, d_image=4, d_filter=3, k=2)
    rng = np.random.default_rng(1)
    f = rng.standard_normal(dims.filters_shape()).astype(np.float32)
    bias = rng.standard_normal(dims.bias_shape()).astype(np.float32)
    layer = M.make_conv_layer(dims, M.Signature((-1, 1)), f, bias)
    out = run_dev(M.conv_forward, np.zeros(dims.input_shape(), np.float32), layer)
    np.testing.assert_allclose(out, np.broadcast_to(bias.T[None, :, None, :], out.shape), atol=1e-7)


def test_conv_empty_batch():
    rng = np.random.default_rng(0)
    _, f, b, _, _ = make_conv(rng, (1, 1), 1, 2, 2, 5, 3)
    layer = M.make_conv_layer(M.Dims(1, 2, 2, 5, 3, 2), M.Signature((1, 1)), f, b)
    h = layer.handle()
    from paper_2507_01040_b200 import _lib
    import ctypes
    assert _lib.load().cl_conv_forward(ctypes.c_void_p(h), None, None, 0, None) == 0


def test_conv_host_path_numpy():
    rng = np.random.default_rng(5)
    x, f, b, layer, pad = make_conv(rng, (1, 1, 1), 3, 4, 4, 8, 3, "fp32", "same")
    y = M.conv_forward(x, layer)  # numpy in -> host path of the C-ABI
    assert isinstance(y, np.ndarray)
    assert_conv_close(y, O.conv_ref(x, f, b, (1, 1, 1), 8, 3, pad), "fp32")


def test_conv_host_path_ragged_chunks():
    # B = 37 through the host pipeline: ramped chunks 1, 2, 4, 5 x 4, 3, 4, 2, 1
    # over three streams; per-sample results are batch-independent, so bit-exact
    rng = np.random.default_rng(6)
    x, f, b, layer, pad = make_conv(rng, (1, 1), 37, 3, 5, 9, 3, "fp32", "same")
    y_host = M.conv_forward(x, layer)
    y_dev = run_dev(M.conv_forward, x, layer)
    assert np.array_equal(y_host, y_dev)
    assert_conv_close(y_host, O.conv_ref(x, f, b, (1, 1), 9, 3, pad), "fp32")


def test_conv_batch_independence():
    rng = np.random.default_rng(9)
    x, f, b, layer, _ = make_conv(rng, (1, 1), 5, 4, 4, 12, 3)
    y = run_dev(M.conv_forward, x, layer)
    one = M.make_conv_layer(M.Dims(1, 4, 4, 12, 3, 2), M.Signature((1, 1)), f, b)
    for i in (0, 4):
        np.testing.assert_array_equal(run_dev(M.conv_forward, x[i:i + 1], one)[0], y[i])


def test_conv_linearity():
    # tests/test_conv.py:143-152: conv(a x1 + x2) - bias = a (conv(x1)-bias) + (conv(x2)-bias)
    rng = np.random.default_rng(3)
    x1, f, _, _, _ = make_conv(rng, (1, 1, 1), 2, 4, 4, 6, 3)
    x2 = rng.standard_normal(x1.shape).astype(np.float32)
    layer = M.make_conv_layer(M.Dims(2, 4, 4, 6, 3, 3), M.Signature((1, 1, 1)), f, np.zeros((8, 4), np.float32))
    a = np.float32(0.75)
    lhs = run_dev(M.conv_forward, (a * x1 + x2).astype(np.float32), layer)
    rhs = a * run_dev(M.conv_forward, x1, layer) + run_dev(M.conv_forward, x2, layer)
    assert O.max_rel_error(lhs, rhs) <= 1e-4


def test_conv_shape_errors():
    rng = np.random.default_rng(0)
    x, f, b, layer, _ = make_conv(rng, (1, 1), 2, 3, 3, 6, 3)
    with pytest.raises(M.errors.ShapeMismatch):
        M.conv_forward(torch.zeros((2, 3, 35, 4), device="cuda"), layer)
    with pytest.raises(ValueError):
        M.conv_forward(torch.from_numpy(x).cuda(), layer, "nonsense")


# ---- (3) activation -----------------------------------------------------------------

def test_activation_golden(golden):
    for n in range(int(golden["act_count"])):
        k, mode, K = (int(v) for v in golden[f"act{n}_meta"])
        ki = tuple(int(v) for v in golden[f"act{n}_ki"])
        w = golden[f"act{n}_w"] if mode == 0 else None
        b = golden[f"act{n}_bias"] if mode == 0 else None
        cfg = M.make_activation_config(M.Signature((1,) * k), mode, ki, w, b)
        y = run_dev(M.activation_forward, golden[f"act{n}_x"], cfg)
        assert O.max_abs_error(y, golden[f"act{n}_y"]) <= 1e-5, n


def test_activation_spatial_golden(golden):
    for mode in (0, 1, 2):
        w = golden[f"sact{mode}_w"] if mode == 0 else None
        b = golden[f"sact{mode}_bias"] if mode == 0 else None
        cfg = M.make_activation_config(M.Signature((1, 1, 1)), mode, tuple(range(8)), w, b)
        y = run_dev(M.activation_forward, golden[f"sact{mode}_x"], cfg)
        assert O.max_abs_error(y, golden[f"sact{mode}_y"]) <= 1e-5


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("C,P,B", [(1, 1, 1), (13, 7, 3), (64, 1000, 2), (3, 4097, 1), (5, 3, 300), (7, 1, 1500)])
def test_activation_shapes(k, mode, C, P, B):
    nb = 1 << k
    rng = np.random.default_rng(k * 100 + mode)
    ki = tuple(int(i) for i in rng.permutation(nb)[: max(1, nb - mode)])
    w = rng.uniform(-0.5, 0.5, (C, len(ki))).astype(np.float32) if mode == 0 else None
    b = (rng.standard_normal(C) * 0.1).astype(np.float32) if mode == 0 else None
    cfg = M.make_activation_config(M.Signature((1,) * k), mode, ki, w, b)
    x = (rng.standard_normal((B, C, P, nb)) * 3).astype(np.float32)
    y = run_dev(M.activation_forward, x, cfg)
    assert O.max_abs_error(y, O.activation_ref(x, mode, ki, w, b)) <= 1e-5
    # flat (B, C, N_B) form
    y3 = run_dev(M.activation_forward, x[:, :, 0, :].copy(), cfg)
    assert O.max_abs_error(y3, O.activation_ref(x[:, :, 0, :], mode, ki, w, b)) <= 1e-5


def test_activation_sigmoid_accuracy():
    # tests/test_activation.py:48-59: gate within 1e-6 of the fp64 sigmoid on [-30, 30]
    s_vals = np.linspace(-30, 30, 4001).astype(np.float32)
    x = np.ones((1, s_vals.size, 4), np.float32)
    x[0, :, 0] = s_vals
    cfg = M.make_activation_config(M.Signature((1, 1)), 1, (0,))
    gate = run_dev(M.activation_forward, x, cfg)[0, :, 1]
    want = 1.0 / (1.0 + np.exp(-s_vals.astype(np.float64)))
    assert np.max(np.abs(gate - want)) < 1e-6


def test_activation_host_path():
    rng = np.random.default_rng(2)
    cfg = M.make_activation_config(M.Signature((1, 1)), 2, (0, 1, 2, 3))
    x = rng.standard_normal((4, 6, 33, 4)).astype(np.float32)
    y = M.activation_forward(x, cfg)
    assert O.max_abs_error(y, O.activation_ref(x, 2, (0, 1, 2, 3))) <= 1e-5


# ---- (4) block ------------------------------------------------------------------------

def _block_from_golden(golden, name, prec="fp32"):
    meta = golden[f"{name}_meta"]
    k = int(meta[3])
    g = tuple(int(v) for v in meta[:k])
    pad, residual, mode, B, C, d = (int(v) for v in meta[4:10])
    aw = golden[f"{name}_aw"] if mode == 0 else None
    ab = golden[f"{name}_ab"] if mode == 0 else None
    blk = M.make_basic_block(M.Signature(g), B, C, C, C, d, golden[f"{name}_f1"], golden[f"{name}_b1"], mode,
                             golden[f"{name}_f2"], golden[f"{name}_b2"], act_weight=aw, act_bias=ab,
                             padding="same" if pad else "valid", residual=bool(residual), precision=prec)
    return blk


@pytest.mark.parametrize("name", ["blk2v", "blk2s", "blk3s", "blk3v"])
@pytest.mark.parametrize("prec", ["fp32", "3xtf32", "bf16"])
def test_block_golden(golden, name, prec):
    blk = _block_from_golden(golden, name, prec)
    y = run_dev(M.block_forward, golden[f"{name}_x"], blk)
    ref = golden[f"{name}_y"]
    assert_conv_close(y, ref, prec)


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("g,mode,padding,residual", [
    ((1, 1), 0, "same", True), ((1, 1, 1), 2, "same", True), ((1, 1), 1, "valid", False),
    ((1, -1, 0), 0, "valid", True), ((1,), 0, "same", True), ((-1,), 1, "valid", False)])
def test_block_random(g, mode, padding, residual, prec):
    rng = np.random.default_rng(4)
    k = len(g)
    nb = 1 << k
    B, C, d = 2, 6, {1: 30, 2: 10, 3: 8}[k]
    fan = C * nb * 3 ** k
    f1 = rng.uniform(-1, 1, (nb, C, C, 3 ** k)).astype(np.float32) / np.float32(np.sqrt(fan))
    f2 = rng.uniform(-1, 1, (nb, C, C, 3 ** k)).astype(np.float32) / np.float32(np.sqrt(fan))
    b1 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    b2 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    aw = rng.uniform(-0.5, 0.5, (C, nb)).astype(np.float32) if mode == 0 else None
    ab = (rng.standard_normal(C) * 0.1).astype(np.float32) if mode == 0 else None
    x = rng.standard_normal((B, C, d ** k, nb)).astype(np.float32)
    blk = M.make_basic_block(M.Signature(g), B, C, C, C, d, f1, b1, mode, f2, b2, act_weight=aw, act_bias=ab,
                             padding=padding, residual=residual, precision=prec)
    y = run_dev(M.block_forward, x, blk)
    ref = O.block_ref(x, g, d, f1, b1, mode, tuple(range(nb)), aw, ab, f2, b2, padding=padding, residual=residual)
    assert_conv_close(y, ref, prec)
    yh = M.block_forward(x, blk)  # host path, chunked
    assert np.array_equal(yh, y)


@pytest.mark.parametrize("prec", ["fp32", "3xtf32", "tf32", "bf16"])
@pytest.mark.parametrize("g,C", [((1, 1), 8), ((1, -1), 12), ((1, 1), 16), ((1, 1, 1), 9)])
def test_block_residual_wide_channels(g, C, prec):
    """Residual fusion with C_out >= 8: under the 2-D change of basis (3xTF32 /
    fp32 modes) one 16-column epilogue chunk covers 8 output channels, each
    with its own residual (advisor finding: channels 4-7 once re-used 0-3's)."""
    rng = np.random.default_rng(40 + C)
    k = len(g)
    nb = 1 << k
    B, d = 2, {2: 10, 3: 6}[k]
    fan = C * nb * 3 ** k
    f1 = rng.uniform(-1, 1, (nb, C, C, 3 ** k)).astype(np.float32) / np.float32(np.sqrt(fan))
    f2 = rng.uniform(-1, 1, (nb, C, C, 3 ** k)).astype(np.float32) / np.float32(np.sqrt(fan))
    b1 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    b2 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    x = (rng.standard_normal((B, C, d ** k, nb)) * (1 + np.arange(C)[None, :, None, None])).astype(np.float32)
    blk = M.make_basic_block(M.Signature(g), B, C, C, C, d, f1, b1, 2, f2, b2, padding="same", residual=True,
                             precision=prec)
    y = run_dev(M.block_forward, x, blk)
    ref = O.block_ref(x, g, d, f1, b1, 2, tuple(range(nb)), None, None, f2, b2, padding="same", residual=True)
    assert_conv_close(y, ref, prec, K=C * nb * 3 ** k)


def test_launch_counter_moves():
    from paper_2507_01040_b200 import _lib
    n0 = _lib.launch_count()
    cfg = M.make_activation_config(M.Signature((1, 1)), 1, (0, 1, 2, 3))
    M.activation_forward(torch.zeros((1, 1, 4), device="cuda"), cfg)
    torch.cuda.synchronize()
    assert _lib.launch_count() > n0


# ---- Clifford linear layer --------------------------------------------

@pytest.mark.parametrize("prec", ["fp32", "3xtf32", "tf32", "bf16"])
def test_linear_golden(golden, prec):
    for n in range(int(golden["lin_count"])):
        g = tuple(int(v) for v in golden[f"lin{n}_g"])
        layer = M.make_linear_layer(M.Signature(g), golden[f"lin{n}_w"], golden[f"lin{n}_b"], precision=prec)
        y = run_dev(M.linear_forward, golden[f"lin{n}_x"], layer)
        assert_conv_close(y, golden[f"lin{n}_y"], prec)


@pytest.mark.parametrize("g", [(1,), (1, 1), (1, 1, 1), (0, 1, -1)])
@pytest.mark.parametrize("B,ci,co", [(1, 1, 1), (300, 64, 48), (129, 7, 33)])
def test_linear_shapes(g, B, ci, co):
    rng = np.random.default_rng(B + ci)
    nb = 1 << len(g)
    w = (rng.standard_normal((nb, co, ci)) / np.sqrt(ci * nb)).astype(np.float32)
    b = (rng.standard_normal((nb, co)) * 0.1).astype(np.float32)
    x = rng.standard_normal((B, ci, nb)).astype(np.float32)
    layer = M.make_linear_layer(M.Signature(g), w, b)
    y = run_dev(M.linear_forward, x, layer)
    assert_conv_close(y, O.linear_ref(x, w, b, g), "fp32")
    yh = M.linear_forward(x, layer)  # host path
    np.testing.assert_array_equal(yh, y)


# ---- seeded shape fuzz over all signatures, precisions, paddings ----------------

def _fuzz_cases(n=48, seed=2507):
    rng = np.random.default_rng(seed)
    sigs = O.all_signatures(3)
    out = []
    for _ in range(n):
        g = sigs[rng.integers(len(sigs))]
        k = len(g)
        df = int(rng.integers(1, 5 if k == 3 else 6))
        padding = "same" if (df % 2 == 1 and rng.random() < 0.5) else "valid"
        d = int(rng.integers(df, {1: 70, 2: 20, 3: 9}[k]))
        out.append((g, int(rng.integers(1, 4)), int(rng.integers(1, 12)), int(rng.integers(1, 12)), d, df, padding,
                    ["fp32", "3xtf32", "tf32", "bf16"][int(rng.integers(4))]))
    return out


@pytest.mark.parametrize("n,case", list(enumerate(_fuzz_cases())),
                         ids=lambda c: f"{c[0]}-B{c[1]}-{c[2]}x{c[3]}-d{c[4]}-f{c[5]}-{c[6]}-{c[7]}" if isinstance(c, tuple) else str(c))
def test_conv_fuzz(n, case):
    g, B, ci, co, d, df, padding, prec = case
    rng = np.random.default_rng(1000 + n)  # deterministic per case
    x, f, b, layer, pad = make_conv(rng, g, B, ci, co, d, df, prec, padding)
    y = run_dev(M.conv_forward, x, layer)
    assert_conv_close(y, O.conv_ref(x, f, b, g, d, df, pad), prec, K=ci * (1 << len(g)) * df ** len(g))


def _block_fuzz_cases(n=16, seed=107):
    rng = np.random.default_rng(seed)
    sigs = [g for g in O.all_signatures(3) if len(g) >= 2]
    out = []
    for _ in range(n):
        g = sigs[rng.integers(len(sigs))]
        out.append((g, int(rng.integers(0, 3)), ["same", "valid"][int(rng.integers(2))], bool(rng.integers(2)),
                    int(rng.integers(1, 4)), int(rng.integers(2, 10)),
                    ["fp32", "3xtf32", "tf32", "bf16"][int(rng.integers(4))]))
    return out


@pytest.mark.parametrize("n,case", list(enumerate(_block_fuzz_cases())),
                         ids=lambda c: "-".join(str(v) for v in c) if isinstance(c, tuple) else str(c))
def test_block_fuzz(n, case):
    """Blocks over random signatures (incl. degenerate and change-of-basis ones),
    activation modes, padding, residual on/off and all four precisions."""
    g, mode, padding, residual, B, C, prec = case  # valid + residual: the input is cropped to the output window
    rng = np.random.default_rng(2000 + n)
    k = len(g)
    nb = 1 << k
    d = {2: 11, 3: 7}[k]
    fan = C * nb * 3 ** k
    f1 = rng.uniform(-1, 1, (nb, C, C, 3 ** k)).astype(np.float32) / np.float32(np.sqrt(fan))
    f2 = rng.uniform(-1, 1, (nb, C, C, 3 ** k)).astype(np.float32) / np.float32(np.sqrt(fan))
    b1 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    b2 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    aw = rng.uniform(-0.5, 0.5, (C, nb)).astype(np.float32) if mode == 0 else None
    ab = (rng.standard_normal(C) * 0.1).astype(np.float32) if mode == 0 else None
    x = rng.standard_normal((B, C, d ** k, nb)).astype(np.float32)
    blk = M.make_basic_block(M.Signature(g), B, C, C, C, d, f1, b1, mode, f2, b2, act_weight=aw, act_bias=ab,
                             padding=padding, residual=residual, precision=prec)
    y = run_dev(M.block_forward, x, blk)
    ref = O.block_ref(x, g, d, f1, b1, mode, tuple(range(nb)), aw, ab, f2, b2, padding=padding, residual=residual)
    assert_conv_close(y, ref, prec, K=C * nb * 3 ** k)


def test_graph_replay_small_forwards():
    """Small conv / block forwards are replayed from a captured CUDA graph from the
    second call with the same buffers on: results stay bit-identical to the first
    (direct) call, follow new input CONTENT in the same buffer, and stay on the
    oracle."""
    rng = np.random.default_rng(21)
    g = (1, 1)
    x, f, b, layer, pad = make_conv(rng, g, 4, 6, 5, 10, 3, "fp32", "same")
    xd = torch.from_numpy(x).cuda()
    y = torch.empty(layer.output_shape(), device="cuda")
    outs = []
    for _ in range(4):  # direct, capture + replay, replay, replay
        M.conv_forward(xd, layer, out=y)
        outs.append(y.cpu().numpy().copy())
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    x2 = rng.standard_normal(x.shape).astype(np.float32)
    xd.copy_(torch.from_numpy(x2))
    M.conv_forward(xd, layer, out=y)
    ref2 = O.conv_ref(x2, f, b, g, 10, 3, pad)
    assert O.max_rel_error(y.cpu().numpy(), ref2) <= 1e-4
    # a block: conv1 (fused gate) -> conv2 (fused residual) replayed the same way
    C, d, nb = 4, 8, 4
    f1 = rng.uniform(-0.2, 0.2, (nb, C, C, 9)).astype(np.float32)
    f2 = rng.uniform(-0.2, 0.2, (nb, C, C, 9)).astype(np.float32)
    b1 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    b2 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    blk = M.make_basic_block(M.Signature(g), 3, C, C, C, d, f1, b1, 1, f2, b2, padding="same", residual=True)
    xb = rng.standard_normal((3, C, d * d, nb)).astype(np.float32)
    xbd = torch.from_numpy(xb).cuda()
    yb = torch.empty_like(xbd)
    res = []
    for _ in range(3):
        M.block_forward(xbd, blk, out=yb)
        res.append(yb.cpu().numpy().copy())
    assert np.array_equal(res[1], res[0]) and np.array_equal(res[2], res[0])
    ref = O.block_ref(xb, g, d, f1, b1, 1, tuple(range(nb)), None, None, f2, b2, padding="same", residual=True)
    assert O.max_rel_error(res[2], ref) <= 1e-4


# ---- exact-mode limits lifted: long reductions (K > 32000) and huge batches ----

@pytest.mark.parametrize("g,B,ci,co,d,df,padding", [
    ((1, 1, 1), 1, 512, 4, 4, 3, "valid"),   # 3-D, C_in = 512: K = 27 * 512 * 4 (basis) = 55296 -> 2 groups
    ((1, 1, 1), 2, 320, 9, 5, 3, "same"),    # K = 34560 -> 2 groups, several N / M tiles
    ((1, -1), 1, 1900, 3, 5, 3, "same"),     # 2-D halo path: K = 9 * 1900 * 2 = 34200
    ((1, 0, -1), 1, 200, 5, 4, 3, "valid"),  # degenerate signature: K = 27 * 200 * 4 or 8 > 32000
])
def test_exact_mode_long_reductions(g, B, ci, co, d, df, padding):
    """The exact mode's s32 level accumulators hold reductions up to K = 32000;
    longer ones are split into accumulation groups drained into exact int64
    partial sums (ConvPlan::drain) instead of being rejected."""
    rng = np.random.default_rng(ci)
    x, f, b, layer, pad = make_conv(rng, g, B, ci, co, d, df, "fp32", padding)
    y = run_dev(M.conv_forward, x, layer)
    e = O.max_rel_error(y, O.conv_ref(x, f, b, g, d, df, pad))
    assert e <= 1e-4, e
    # the same digits summed in one s32 group would overflow in the worst case only; a
    # reduction of exactly-representable integers checks the int64 combine bit-exactly
    xi = np.round(x * 4).astype(np.float32)
    fi = np.round(f * 1024).astype(np.float32)
    li = M.make_conv_layer(M.Dims(B, ci, co, d, df, len(g)), M.Signature(g), fi, np.zeros_like(b), padding=padding)
    yi = run_dev(M.conv_forward, xi, li)
    ri = O.conv_ref(xi, fi, np.zeros_like(b), g, d, df, pad)
    assert np.array_equal(yi, ri)


@pytest.mark.parametrize("g,B,ci,co,d,df,padding", [
    ((1, 1, 1), 1, 512, 4, 4, 3, "valid"),   # 3-D halo path: K = 55296 -> 864 accumulation groups
    ((1, -1), 1, 1900, 3, 5, 3, "same"),     # 2-D halo path: K = 34200
    ((1, 1), 2, 7, 5, 12, 5, "same"),        # K = 700: groups not aligned with the taps
    ((1,), 3, 300, 4, 30, 3, "valid"),       # 1-D (per-tap A loads, 1-SM, splitter per stage)
])
def test_3xtf32_accumulation_groups(g, B, ci, co, d, df, padding):
    """3xTF32 drains its A_hi*B_hi TMEM accumulator every 192 reduction elements
    into fp32 registers and keeps the cross terms in their own tile-long
    accumulator (x3_drain_groups): the error must not grow with K (one truncating
    accumulator reached 7e-3 under the reference metric at K = 13824)."""
    rng = np.random.default_rng(ci + 3)
    x, f, b, layer, pad = make_conv(rng, g, B, ci, co, d, df, "3xtf32", padding)
    y = run_dev(M.conv_forward, x, layer)
    ref = O.conv_ref(x, f, b, g, d, df, pad)
    e = O.max_rel_error(y, ref, floor=float(np.abs(ref).max()))
    assert e <= 1e-6 and O.max_rel_error(y, ref) <= 1e-4, (e, O.max_rel_error(y, ref))


@pytest.mark.parametrize("prec", ["bf16", "tf32", "3xtf32", "fp32"])
@pytest.mark.parametrize("df,ci,co,d", [(5, 20, 70, 7), (2, 12, 9, 6), (3, 64, 72, 5), (4, 3, 33, 6)])
def test_halo_multi_tap_stages(prec, df, ci, co, d):
    """3-D halo plans store each CTA's taps of a channel group contiguously and
    load a multi-tap B stage as ONE request (a pair's box always covers tps
    taps; a short last stage over-reads into the next block or past the end of
    the image, zero-filled): tap counts not divisible by the taps per stage
    (Q = 125, 8, 27, 64), several channel groups and several N tiles."""
    rng = np.random.default_rng(df * 100 + ci)
    g = (1, 1, 1)
    padding = "same" if df % 2 else "valid"  # same padding needs an odd filter (conv.py)
    x, f, b, layer, pad = make_conv(rng, g, 2, ci, co, d, df, prec, padding)
    y = run_dev(M.conv_forward, x, layer)
    assert_conv_close(y, O.conv_ref(x, f, b, g, d, df, pad), prec, K=ci * 8 * df ** 3)


def test_linear_huge_batch_and_long_reduction():
    """linear_forward on B = 100000 samples (the per-sample absmax grid is 1-D,
    no 65535-sample limit) and a C_in whose reduction exceeds 32000."""
    rng = np.random.default_rng(8)
    g, nb = (1, 1, 1), 8
    for B, ci, co in [(100_000, 16, 8), (300, 4100, 5)]:
        w = (rng.standard_normal((nb, co, ci)) / np.sqrt(ci * nb)).astype(np.float32)
        b = (rng.standard_normal((nb, co)) * 0.1).astype(np.float32)
        x = rng.standard_normal((B, ci, nb)).astype(np.float32)
        layer = M.make_linear_layer(M.Signature(g), w, b)
        y = run_dev(M.linear_forward, x, layer)
        idx = np.r_[0:50, B - 50:B]
        assert O.max_rel_error(y[idx], O.linear_ref(x[idx], w, b, g)) <= 1e-4
        yh = M.linear_forward(x, layer)  # host path
        np.testing.assert_array_equal(yh, y)


def test_misaligned_buffers_are_copied_or_rejected():
    """A contiguous CUDA view with a 4-byte storage offset is realigned (copied)
    by the Python shim; a misaligned `out` is rejected with ShapeMismatch by the
    C-ABI instead of faulting (a misaligned-address fault poisons the context)."""
    rng = np.random.default_rng(12)
    x, f, b, layer, pad = make_conv(rng, (1, 1), 2, 3, 3, 7, 3, "fp32")
    flat = torch.zeros(x.size + 1, device="cuda")
    flat[1:] = torch.from_numpy(x.ravel()).cuda()
    xv = flat[1:].view(x.shape)
    assert xv.data_ptr() % 16 != 0 and xv.is_contiguous()
    y = M.conv_forward(xv, layer).cpu().numpy()
    assert O.max_rel_error(y, O.conv_ref(x, f, b, (1, 1), 7, 3, pad)) <= 1e-4
    out_flat = torch.zeros(int(np.prod(layer.output_shape())) + 1, device="cuda")
    with pytest.raises(M.errors.ShapeMismatch, match="aligned"):
        M.conv_forward(torch.from_numpy(x).cuda(), layer, out=out_flat[1:].view(layer.output_shape()))
    for prec in ("bf16", "tf32"):
        lp = M.make_conv_layer(M.Dims(2, 3, 3, 7, 3, 2), M.Signature((1, 1)), f, b, precision=prec)
        assert_conv_close(M.conv_forward(xv, lp).cpu().numpy(), O.conv_ref(x, f, b, (1, 1), 7, 3, pad), prec)
    torch.cuda.synchronize()  # the context is healthy
