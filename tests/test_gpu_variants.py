"""GPU parity of the kernel variants the planner can switch off (1-SM MMA,
per-tap A loads, per-pixel TMA lines, one tap per B stage, generic basis
inverse, separate absmax pass, generic digit slicing, the small-layer fused
absmax + slice launch and graph replay) and the dynamic tile order forced on
every launch (CL_DYN_TILES: 1-D / 2-D / 3-D, paired and 1-SM, the 3xTF32
splitter). The switches are
read once when the library loads -- and only by the diagnostic build
libclifford_b200_ab.so, loaded here through CL_LIB_PATH -- so each variant
runs in a fresh process;
the default variant is covered by test_gpu_parity.py. Same tolerances."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SNIPPET = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import torch
import oracle as O
from test_gpu_parity import make_conv, run_dev, assert_conv_close
import paper_2507_01040_b200 as M
torch.cuda.set_device(0)
rng = np.random.default_rng(11)
cases = [((1, 1, 1), 2, 5, 6, 6, 3, "same"), ((1, -1, 0), 1, 3, 4, 5, 3, "valid"), ((1, 1), 3, 6, 5, 9, 3, "same"),
         ((0, 0, 1), 2, 4, 3, 5, 2, "valid"), ((1,), 3, 4, 4, 40, 3, "valid")]
for prec in ("fp32", "3xtf32", "tf32", "bf16"):
    for g, B, ci, co, d, df, padding in cases:
        x, f, b, layer, pad = make_conv(rng, g, B, ci, co, d, df, prec, padding)
        y = run_dev(M.conv_forward, x, layer)
        assert_conv_close(y, O.conv_ref(x, f, b, g, d, df, pad), prec,
                          K=ci * (1 << len(g)) * df ** len(g))
# a block (conv -> activation -> conv + residual) in the exact mode
g, B, C, d = (1, 1, 1), 2, 4, 6
nb = 8
x = rng.standard_normal((B, C, d ** 3, nb)).astype(np.float32)
fan = C * nb * 27
f1 = rng.uniform(-1, 1, (nb, C, C, 27)).astype(np.float32) / np.float32(np.sqrt(fan))
f2 = rng.uniform(-1, 1, (nb, C, C, 27)).astype(np.float32) / np.float32(np.sqrt(fan))
b1 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
b2 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
blk = M.make_basic_block(M.Signature(g), B, C, C, C, d, f1, b1, 2, f2, b2, padding="same", residual=True)
y = M.block_forward(torch.from_numpy(x).cuda(), blk).cpu().numpy()
ref = O.block_ref(x, g, d, f1, b1, 2, tuple(range(nb)), None, None, f2, b2, padding="same", residual=True)
assert O.max_rel_error(y, ref) <= 1e-4, O.max_rel_error(y, ref)
print("ok")
"""


AB_LIB = os.path.join(ROOT, "paper_2507_01040_b200", "lib", "libclifford_b200_ab.so")


def _run(env_extra):
    # the switches exist only in the diagnostic build (the production library ignores the environment)
    env = dict(os.environ, CL_LIB_PATH=AB_LIB, **env_extra)
    code = SNIPPET.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("flags", [{"CL_NO_PAIR": "1"}, {"CL_NO_HALO": "1"}, {"CL_NO_TMA_MERGE": "1"},
                                   {"CL_TPS": "1"}, {"CL_NO_BASIS": "1"}, {"CL_NO_BASIS_2D": "1"},
                                   {"CL_NO_BCLS": "1", "CL_NO_FUSED_AMAX": "1", "CL_NO_SLICE_FIXED": "1"},
                                   {"CL_NO_FUSED_PREP": "1", "CL_NO_GRAPH": "1"},
                                   {"CL_DYN_TILES": "1"}, {"CL_DYN_TILES": "1", "CL_NO_PAIR": "1"}],
                         ids=lambda f: ",".join(f))
def test_variant_parity(flags):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    _run(flags)


FAULT_SNIPPET = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import torch
import oracle as O
from test_gpu_parity import make_conv, run_dev
import paper_2507_01040_b200 as M
torch.cuda.set_device(0)
rng = np.random.default_rng(3)
i, j = 1, 2  # CL_DBG_FLIP_COEFF: coeff(e1, e2) negated in kernel construction
for g in [(1, 1), (1, 1, 1)]:
    x, f, b, layer, pad = make_conv(rng, g, 2, 3, 4, 6, 3, "fp32", "same")
    W = M.build_expanded_kernel(layer).cpu().numpy()
    ref_W = O.expanded_kernel(f, g)
    nb = 1 << len(g)
    bad = np.zeros(ref_W.shape, bool)
    for t in range(nb):
        if t ^ j == i:  # W[(co, t), (ci, j), q] reads coeff(t ^ j, j)
            bad[t::nb, j::nb, :] = True
    assert np.array_equal(W[~bad], ref_W[~bad]) and np.array_equal(W[bad], -ref_W[bad]), "flip not where expected"
    for prec in ("fp32", "bf16"):
        x, f, b, layer, pad = make_conv(rng, g, 2, 3, 4, 6, 3, prec, "same")
        y = run_dev(M.conv_forward, x, layer)
        ref = O.conv_ref(x, f, b, g, 6, 3, pad)
        e = O.max_rel_error(y, ref, floor=float(np.abs(ref).max()))
        assert e > 2e-2, (g, prec, e)  # the parity bound of every mode catches the fault
print("detected")
"""


def test_fault_injection_is_detected():
    """Fault injection (the reference's parity_report schedule_transform, bench.py:566-576 /
    tests/test_bench.py:202-210): one negated product-table coefficient in the device's
    kernel construction must show up exactly in the expanded filter and break conv parity."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    env = dict(os.environ, CL_LIB_PATH=AB_LIB, CL_DBG_FLIP_COEFF="1,2")
    code = FAULT_SNIPPET.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("detected"), r.stdout[-2000:] + r.stderr[-4000:]
