"""Size-independent properties the reference tests pin (on the B200 path):
conv translation consistency (tests/test_conv.py:154-174, extended to 3-D and
every precision), activation output bound, gate scale covariance and
blade-uniform gating (tests/test_activation.py:210-237)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

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


@pytest.mark.parametrize("prec", ["fp32", "3xtf32", "tf32", "bf16"])
@pytest.mark.parametrize("g", [(1, 1), (1, 1, 1), (1, -1, 0)])
def test_conv_non_finite_inputs(prec, g):
    """A NaN / Inf in a sample's input never turns into finite garbage: every
    output the fp64 oracle gives as non-finite is non-finite here too (the
    exact mode's per-sample scale becomes NaN, so that whole sample is NaN),
    and the other samples are untouched."""
    import oracle as O
    k = len(g)
    nb = 1 << k
    rng = np.random.default_rng(5)
    B, C, d, df = 3, 3, 6, 3
    x = rng.standard_normal((B, C, d ** k, nb)).astype(np.float32)
    x[1, 0, 7, 1] = np.nan
    x[2, 2, 3, 0] = np.inf
    f = rng.uniform(-1, 1, (nb, C, C, df ** k)).astype(np.float32) / np.float32(np.sqrt(C * nb * df ** k))
    b = (rng.standard_normal((nb, C)) * 0.01).astype(np.float32)
    y = M.conv_forward(torch.from_numpy(x).cuda(), _conv(g, B, C, C, d, df, f, b, prec)).cpu().numpy()
    with np.errstate(invalid="ignore"):
        ref = O.conv_ref(x, f, b, g, d, df, 0)
    bad = ~np.isfinite(ref)
    assert bad[1].any() and bad[2].any()
    assert np.all(~np.isfinite(y[bad])), prec
    assert np.all(np.isfinite(y[0]))
    assert O.max_rel_error(y[:1], ref[:1], floor=float(np.abs(ref[0]).max())) <= {"fp32": 1e-6, "3xtf32": 1e-4}.get(prec, 2e-2)


def test_block_non_finite_input_exact_mode():
    """The block's fused absmax of y1 (conv1 epilogue) keeps a NaN too."""
    import oracle as O
    rng = np.random.default_rng(9)
    g, B, C, d, nb = (1, 1, 1), 2, 4, 6, 8
    fan = C * nb * 27
    f1 = rng.uniform(-1, 1, (nb, C, C, 27)).astype(np.float32) / np.float32(np.sqrt(fan))
    f2 = rng.uniform(-1, 1, (nb, C, C, 27)).astype(np.float32) / np.float32(np.sqrt(fan))
    b1 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    b2 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    x = rng.standard_normal((B, C, d ** 3, nb)).astype(np.float32)
    x[1, 1, 100, 3] = np.nan
    blk = M.make_basic_block(M.Signature(g), B, C, C, C, d, f1, b1, 2, f2, b2, padding="same", residual=True)
    y = M.block_forward(torch.from_numpy(x).cuda(), blk).cpu().numpy()
    with np.errstate(invalid="ignore"):
        ref = O.block_ref(x, g, d, f1, b1, 2, tuple(range(nb)), None, None, f2, b2, padding="same", residual=True)
    bad = ~np.isfinite(ref)
    assert bad[1].any() and np.all(~np.isfinite(y[bad]))
    assert O.max_rel_error(y[:1], ref[:1]) <= 1e-4
