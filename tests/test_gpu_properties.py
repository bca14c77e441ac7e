"""Size-independent properties the reference tests pin (on the B200 path):
conv translation consistency (tests/test_conv.py:154-174, extended to 3-D and
every precision), activation output bound, gate scale covariance and
blade-uniform gating (tests/test_activation.py:210-237)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
import paper_2507_01040_b200 as M  # noqa: E402

TOL = {"fp32": (1e-6, 1e-6), "3xtf32": (1e-4, 1e-5), "tf32": (2e-3, 1e-4), "bf16": (2e-2, 1e-3)}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _conv(g, B, ci, co, d, df, f, b, prec):
    return M.make_conv_layer(M.Dims(B, ci, co, d, df, len(g)), M.Signature(g), f, b, precision=prec)


@pytest.mark.parametrize("prec", ["fp32", "3xtf32", "tf32", "bf16"])
@pytest.mark.parametrize("g,B,ci,co,d,df", [((1,), 2, 1, 1, 8, 3), ((1, -1), 1, 1, 2, 6, 2),
                                            ((1, 1), 2, 5, 3, 12, 3), ((1, 1, 1), 2, 3, 4, 7, 3),
                                            ((1, -1, 0), 1, 2, 2, 6, 2)])
def test_conv_translation_consistency(prec, g, B, ci, co, d, df):
    """Valid conv of the input shifted by one pixel along every axis equals the
    full output shifted the same way (test_conv.py:154-174)."""
    k = len(g)
    nb = 1 << k
    rng = np.random.default_rng(d * 10 + k)
    x = np.clip(rng.standard_normal((B, ci) + (d,) * k + (nb,)), -5, 5).astype(np.float32)
    # the per-sample max lies inside the cropped region, so the fp32 mode's
    # power-of-two scale (and with it every digit) is the same in both runs
    x[(slice(None), slice(None)) + (1,) * k + (slice(None),)] = 8.0
    f = rng.uniform(-1, 1, (nb, ci, co, df ** k)).astype(np.float32) / np.float32(np.sqrt(ci * nb * df ** k))
    b = (rng.standard_normal((nb, co)) * 0.01).astype(np.float32)
    full = M.conv_forward(torch.from_numpy(x.reshape(B, ci, d ** k, nb)).cuda(),
                          _conv(g, B, ci, co, d, df, f, b, prec)).cpu().numpy()
    do = d - df + 1
    full = full.reshape((B, co) + (do,) * k + (nb,))
    xs = np.ascontiguousarray(x[(slice(None), slice(None)) + (slice(1, None),) * k + (slice(None),)])
    crop = M.conv_forward(torch.from_numpy(xs.reshape(B, ci, (d - 1) ** k, nb)).cuda(),
                          _conv(g, B, ci, co, d - 1, df, f, b, prec)).cpu().numpy()
    crop = crop.reshape((B, co) + (do - 1,) * k + (nb,))
    rtol, atol = TOL[prec]
    np.testing.assert_allclose(crop, full[(slice(None), slice(None)) + (slice(1, None),) * k + (slice(None),)],
                               rtol=rtol, atol=atol)


def _act(rng, k, C, mode):
    nb = 1 << k
    ki = tuple(int(i) for i in rng.permutation(nb)[: max(1, nb // 2)])
    w = rng.uniform(-0.5, 0.5, (C, len(ki))).astype(np.float32) if mode == 0 else None
    b = (rng.standard_normal(C) * 0.1).astype(np.float32) if mode == 0 else None
    return M.make_activation_config(M.Signature((1,) * k), mode, ki, w, b)


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_activation_bounds_and_blade_uniform_gate(k, mode):
    """|out| <= |in|, and out / x is the same for every blade of a multivector
    (test_activation.py:210-216, :229-237)."""
    rng = np.random.default_rng(100 * k + mode)
    nb = 1 << k
    cfg = _act(rng, k, 6, mode)
    x = rng.standard_normal((3, 6, 50, nb)).astype(np.float32)
    x[np.abs(x) < 1e-3] = 1.0
    y = M.activation_forward(torch.from_numpy(x).cuda(), cfg).cpu().numpy()
    assert np.all(np.abs(y) <= np.abs(x))
    ratio = y / x
    np.testing.assert_allclose(ratio, np.broadcast_to(ratio[..., :1], ratio.shape), rtol=1e-6)


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("alpha", [0.125, 0.5, 3.0, 8.0])
def test_activation_gate_scale_covariance(mode, alpha):
    """Sum / Mean pre-activations scale with the input (test_activation.py:218-227):
    s(alpha x) = alpha s(x), read back as logit(out / x) where the gate is not saturated."""
    rng = np.random.default_rng(int(alpha * 8) + mode)
    cfg = _act(rng, 3, 4, mode)
    x = (rng.standard_normal((2, 4, 5, 8)) * 0.3).astype(np.float32)
    x[np.abs(x) < 1e-2] = 0.5

    def s_of(xx):
        y = M.activation_forward(torch.from_numpy(xx).cuda(), cfg).cpu().numpy().astype(np.float64)
        r = (y / xx)[..., 0]
        return np.log(r / (1 - r))

    s1 = s_of(x)
    s2 = s_of((np.float32(alpha) * x).astype(np.float32))
    ok = np.abs(alpha * s1) < 6
    np.testing.assert_allclose(s2[ok], alpha * s1[ok], rtol=1e-3, atol=1e-4)


def _finite_close(y, ref, prec):
    """Same finiteness pattern as the oracle (both directions), and the finite
    entries within the mode's bound."""
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(y), fin), (int((np.isfinite(y) != fin).sum()), prec)
    yz, rz = np.where(fin, y, 0), np.where(fin, ref, 0)
    if prec == "fp32":
        assert O.max_rel_error(yz, rz) <= 1e-4
    else:
        tol = {"3xtf32": 1e-4}.get(prec, 2e-2)
        assert O.max_rel_error(yz, rz, floor=float(np.abs(rz).max())) <= tol


@pytest.mark.parametrize("prec", ["fp32", "3xtf32", "tf32", "bf16"])
@pytest.mark.parametrize("g,padding", [((1, 1), "valid"), ((1, 1, 1), "same"), ((1, -1, 0), "valid"), ((1,), "same"),
                                       ((0, 1), "same")])
def test_conv_non_finite_inputs(prec, g, padding):
    """A NaN / Inf input turns exactly the outputs the fp64 oracle gives as
    non-finite into non-finite ones -- the receptive fields of the bad inputs,
    all channels and blades -- and nothing else: oracle finite <=> B200 finite,
    finite values within the mode's bound. (The exact mode scales samples by
    their finite max, slices Inf / NaN as 0 and poisons their receptive fields
    afterwards; the fp32-accumulator modes propagate them through the MMAs.)"""
    k = len(g)
    nb = 1 << k
    rng = np.random.default_rng(5)
    B, C, d, df = 4, 3, {1: 30, 2: 7, 3: 6}[k], 3
    x = rng.standard_normal((B, C, d ** k, nb)).astype(np.float32)
    x[1, 0, 7, 1] = np.nan
    x[2, 2, 3, 0] = np.inf
    x[3, 1, d ** k - 1, nb - 1] = -np.inf  # a corner: clipped receptive fields
    f = rng.uniform(-1, 1, (nb, C, C, df ** k)).astype(np.float32) / np.float32(np.sqrt(C * nb * df ** k))
    b = (rng.standard_normal((nb, C)) * 0.01).astype(np.float32)
    layer = M.make_conv_layer(M.Dims(B, C, C, d, df, k), M.Signature(g), f, b, precision=prec, padding=padding)
    y = M.conv_forward(torch.from_numpy(x).cuda(), layer).cpu().numpy()
    pad = 1 if padding == "same" else 0
    with np.errstate(invalid="ignore", over="ignore"):
        ref = O.conv_ref(x, f, b, g, d, df, pad)
    bad = ~np.isfinite(ref)
    assert bad[1].any() and bad[2].any() and bad[3].any() and not bad[0].any()
    assert bad[1].sum() < bad[1].size  # the poisoned set is a receptive field, not the whole sample
    _finite_close(y, ref, prec)


@pytest.mark.parametrize("prec", ["fp32", "3xtf32", "bf16"])
def test_block_non_finite_input(prec):
    """Block: a NaN input poisons conv1's receptive field, the gate keeps it
    (NaN), conv2 widens it (the fused absmax of y1 carries a non-finite flag to
    conv2 in the exact mode), the residual adds it; everything else stays
    finite and accurate -- the oracle's pattern in both directions."""
    rng = np.random.default_rng(9)
    g, B, C, d, nb = (1, 1, 1), 3, 4, 7, 8
    fan = C * nb * 27
    f1 = rng.uniform(-1, 1, (nb, C, C, 27)).astype(np.float32) / np.float32(np.sqrt(fan))
    f2 = rng.uniform(-1, 1, (nb, C, C, 27)).astype(np.float32) / np.float32(np.sqrt(fan))
    b1 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    b2 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    x = rng.standard_normal((B, C, d ** 3, nb)).astype(np.float32)
    x[1, 1, 0, 3] = np.nan
    x[2, 0, 171, 5] = np.inf
    blk = M.make_basic_block(M.Signature(g), B, C, C, C, d, f1, b1, 2, f2, b2, padding="same", residual=True,
                             precision=prec)
    y = M.block_forward(torch.from_numpy(x).cuda(), blk).cpu().numpy()
    with np.errstate(invalid="ignore", over="ignore"):
        ref = O.block_ref(x, g, d, f1, b1, 2, tuple(range(nb)), None, None, f2, b2, padding="same", residual=True)
    bad = ~np.isfinite(ref)
    assert bad[1].any() and bad[2].any() and not bad[0].any() and bad[1].sum() < bad[1].size
    _finite_close(y, ref, prec)


@pytest.mark.parametrize("k", [2, 3])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_activation_non_kernel_blades_never_reach_the_gate(k, mode):
    """K < N_B: an Inf / NaN in a NON-kernel blade must not touch the gate --
    the reference never reads those blades (activation.py:142-162) -- so only
    that blade itself is non-finite in the output; a non-finite kernel blade
    poisons the whole multivector as in the reference. (The gate fused into
    a block's conv1 epilogue uses the same kernel-blade select.)"""
    nb = 1 << k
    rng = np.random.default_rng(20 + k * 3 + mode)
    ki = (1, 0) if k == 2 else (5, 2, 0)
    C = 5
    w = rng.uniform(-0.5, 0.5, (C, len(ki))).astype(np.float32) if mode == 0 else None
    b = (rng.standard_normal(C) * 0.1).astype(np.float32) if mode == 0 else None
    cfg = M.make_activation_config(M.Signature((1,) * k), mode, ki, w, b)
    x = rng.standard_normal((3, C, 6, nb)).astype(np.float32)
    x[0, 1, 2, 3] = np.inf      # non-kernel blade
    x[1, 2, 0, nb - 1] = np.nan  # non-kernel blade
    x[2, 0, 4, ki[0]] = np.inf   # kernel blade
    y = M.activation_forward(torch.from_numpy(x).cuda(), cfg).cpu().numpy()
    with np.errstate(invalid="ignore", over="ignore"):
        ref = O.activation_ref(x, mode, ki, w, b)
    assert np.array_equal(np.isfinite(y), np.isfinite(ref))
    assert np.isfinite(y[0, 1, 2, :3]).all() and not np.isfinite(y[0, 1, 2, 3])
    fin = np.isfinite(ref)
    assert O.max_abs_error(np.where(fin, y, 0), np.where(fin, ref, 0)) <= 1e-5


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_gather_vpack_and_gate_preactivation(k, mode):
    """Device-backed gather_vpack / gate_preactivation (activation.py:99-117):
    numpy in -> numpy out, CUDA in -> CUDA out, flat and spatial forms, against
    the reference's formulas (kernel blades in kernel_indices order)."""
    nb = 1 << k
    rng = np.random.default_rng(100 + 7 * k + mode)
    ki = tuple(int(i) for i in rng.permutation(nb)[: max(1, nb - 1)])
    C = 6
    w = rng.uniform(-0.5, 0.5, (C, len(ki))).astype(np.float32) if mode == 0 else None
    b = (rng.standard_normal(C) * 0.1).astype(np.float32) if mode == 0 else None
    cfg = M.make_activation_config(M.Signature((1,) * k), mode, ki, w, b)
    x = rng.standard_normal((4, C, nb)).astype(np.float32)
    vp = M.gather_vpack(x, cfg)
    assert isinstance(vp, np.ndarray) and vp.shape == (4, C, len(ki))
    np.testing.assert_array_equal(vp, x[:, :, list(ki)])
    s = M.gate_preactivation(x, cfg)
    want = ((vp * w[None]).sum(axis=2) + b[None]) if mode == 0 else (vp.sum(axis=2) if mode == 1 else vp.mean(axis=2))
    assert s.shape == (4, C) and np.max(np.abs(s - want)) <= 1e-5
    xs = rng.standard_normal((2, C, 9, nb)).astype(np.float32)
    sd = M.gate_preactivation(torch.from_numpy(xs).cuda(), cfg)
    assert sd.is_cuda and tuple(sd.shape) == (2, C, 9)
    vps = xs[..., list(ki)]
    want = ((vps * w[None, :, None]).sum(-1) + b[None, :, None]) if mode == 0 else (
        vps.sum(-1) if mode == 1 else vps.mean(-1))
    assert np.max(np.abs(sd.cpu().numpy() - want)) <= 1e-5
    # the gate the forward applies is sigmoid(preactivation)
    y = M.activation_forward(x, cfg)
    np.testing.assert_allclose(y, x * M.sigmoid(s)[..., None].astype(np.float32), rtol=2e-6, atol=2e-6)


@pytest.mark.parametrize("g", [(1, 1), (1, 1, 1), (1, -1, 0)])
def test_exact_mode_heterogeneous_channel_scales(g):
    """The exact (fp32) mode is fixed point against a PER-SAMPLE power-of-two
    scale s_x >= max|x| (31-bit digits), with channels scaled x1e-3 ... x1e3
    in one sample. (a) Dense random filters (every output mixes all
    channels): the reference metric stays <= 1e-4. (b) Channel-diagonal
    filters (output channel c reads input channel c only) expose the small
    channels' loss; the error stays within the scheme's representation bound
    |dy| <= 8 sum_k (|W_k| s_x + |x_k| s_w) 2^-32 + ulp(y)/2 (s_w the filter
    column scale; the factor covers the change of basis: |T x| <= 2 max|x|,
    the transformed filter entries, and the power-of-two rounding of scales) -- DESIGN.md section 4 states this limit."""
    k = len(g)
    nb = 1 << k
    rng = np.random.default_rng(77)
    B, C, d, df = 2, 7, {2: 8, 3: 5}[k], 3
    Q = df ** k
    scales = (10.0 ** np.linspace(-3, 3, C)).astype(np.float32)
    x = (rng.standard_normal((B, C, d ** k, nb)) * scales[None, :, None, None]).astype(np.float32)
    f = rng.uniform(-1, 1, (nb, C, C, Q)).astype(np.float32) / np.float32(np.sqrt(C * nb * Q))
    b = np.zeros((nb, C), np.float32)
    xd = torch.from_numpy(x).cuda()
    dims = M.Dims(B, C, C, d, df, k)
    y = M.conv_forward(xd, M.make_conv_layer(dims, M.Signature(g), f, b, padding="same")).cpu().numpy()
    assert O.max_rel_error(y, O.conv_ref(x, f, b, g, d, df, 1)) <= 1e-4
    # (b) channel-diagonal filters
    fd = np.zeros_like(f)
    for c in range(C):
        fd[:, c, c, :] = f[:, c, c, :]
    y = M.conv_forward(xd, M.make_conv_layer(dims, M.Signature(g), fd, b, padding="same")).cpu().numpy()
    ref = O.conv_ref(x, fd, b, g, d, df, 1).astype(np.float64)
    s_x = 2.0 ** np.ceil(np.log2(np.abs(x).reshape(B, -1).max(axis=1) * 1.016))  # per sample
    W = O.expanded_kernel(fd, g).astype(np.float64)                               # (C*nb, C*nb, Q)
    s_w = 2.0 ** np.ceil(np.log2(np.abs(W).max(axis=(1, 2)) * 1.016))            # per output row
    absW = np.abs(W).sum(axis=(1, 2)).reshape(C, nb)                              # sum_k |W_k| per (co, t)
    # sum over the receptive field (all blades) of |x| of the same channel, zero padded
    ax = np.abs(x.astype(np.float64)).sum(axis=3).reshape((B, C) + (d,) * k)
    axp = np.pad(ax, [(0, 0), (0, 0)] + [(1, 1)] * k)
    box = np.zeros_like(ax)
    for q in np.ndindex(*(df,) * k):
        box += axp[(slice(None), slice(None)) + tuple(slice(qi, qi + d) for qi in q)]
    box = box.reshape(B, C, d ** k)
    bound = 8.0 * 2.0 ** -32 * (absW[None, :, None, :] * s_x[:, None, None, None]
                                + box[..., None] * s_w.reshape(C, nb)[None, :, None, :])
    bound += np.abs(ref) * 2.0 ** -24 + 1e-38
    err = np.abs(y.astype(np.float64) - ref)
    assert np.all(err <= bound), float(np.max(err / bound))
    # the bound is what the x1e-3 channel can get: report it against fp32's own precision
    rel_small = float(np.max(err[:, 0]) / np.max(np.abs(ref[:, 0])))
    assert rel_small < 1e-2, rel_small
