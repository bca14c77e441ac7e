"""JSON-lines server (serve.py protocol) on the B200 path. Protocol and
validation paths run on CPU; forwards need the GPU."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
from paper_2507_01040_b200 import serve as S
from paper_2507_01040_b200.layout import LayoutTag, read_tensor, write_tensor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ping_and_unknown_op():
    h = S.Handles()
    assert S.handle_request({"op": "ping"}, h)["ok"]
    r = S.handle_request({"op": "nope"}, h)
    assert not r["ok"] and "unknown op" in r["error"]
    r = S.handle_request({"op": "forward", "handle": 9, "input": "x", "output": "y"}, h)
    assert not r["ok"] and r["error"].startswith("ShapeMismatch")


def test_create_errors_mirror_reference(tmp_path):
    h = S.Handles()
    f = tmp_path / "f.mvtf"
    b = tmp_path / "b.mvtf"
    write_tensor(f, np.zeros((4, 2, 2, 9), np.float32), LayoutTag.CONV_FILTERS, 2)
    write_tensor(b, np.zeros((4, 2), np.float32), LayoutTag.CONV_BIAS, 2)
    base = {"op": "create_conv", "B": 1, "Cin": 2, "Cout": 2, "dimage": 5, "dfilter": 3,
            "filters": str(f), "bias": str(b)}
    r = S.handle_request(dict(base, sig=[1, 2]), h)
    assert r["error"].startswith("InvalidMetricValue")
    r = S.handle_request(dict(base, sig=[0, 0]), h)
    assert r["error"].startswith("InvalidSignature")
    r = S.handle_request(dict(base, sig=[1, 1], Cin=3), h)
    assert r["error"].startswith("ShapeMismatch")
    assert S.handle_request(dict(base, sig=[1, 1]), h)["ok"]
    # float64 payloads are rejected (serve.py:36-42)
    write_tensor(b, np.zeros((4, 2), np.float64), LayoutTag.CONV_BIAS, 2)
    r = S.handle_request(dict(base, sig=[1, 1]), h)
    assert not r["ok"] and "float32" in r["error"]
    r = S.handle_request({"op": "create_activation", "sig": [1, 1], "mode": 0, "kernel_indices": [0, 1]}, h)
    assert r["error"].startswith("ModeConfigMismatch")


@pytest.mark.gpu
def test_conv_activation_block_roundtrip(tmp_path):
    import torch
    assert torch.cuda.is_available()
    rng = np.random.default_rng(3)
    h = S.Handles()
    g, B, C, d = (1, 1), 2, 3, 8
    nb = 4
    x = rng.standard_normal((B, C, d * d, nb)).astype(np.float32)
    f1 = (rng.uniform(-1, 1, (nb, C, C, 9)) / np.sqrt(C * nb * 9)).astype(np.float32)
    b1 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    paths = {}
    for name, arr, tag in [("x", x, LayoutTag.CONV_INPUT), ("f1", f1, LayoutTag.CONV_FILTERS),
                           ("b1", b1, LayoutTag.CONV_BIAS)]:
        paths[name] = str(tmp_path / f"{name}.mvtf")
        write_tensor(paths[name], arr, tag, 2)
    r = S.handle_request({"op": "create_conv", "sig": list(g), "B": B, "Cin": C, "Cout": C, "dimage": d,
                          "dfilter": 3, "filters": paths["f1"], "bias": paths["b1"], "padding": "same"}, h)
    hc = r["handle"]
    out = str(tmp_path / "y.mvtf")
    r = S.handle_request({"op": "forward", "handle": hc, "input": paths["x"], "output": out, "variant": "b200"}, h)
    assert r["ok"] and r["shape"] == [B, C, d * d, nb], r
    # the reference's CPU variant names are not aliases of the B200 path
    r = S.handle_request({"op": "forward", "handle": hc, "input": paths["x"], "output": out, "variant": "packed"}, h)
    assert not r["ok"] and "ValueError" in r["error"] and "packed" in r["error"], r
    y = read_tensor(out).data
    assert O.max_rel_error(y, O.conv_ref(x, f1, b1, g, d, 3, 1)) <= 1e-4
    # spatial activation
    r = S.handle_request({"op": "create_activation", "sig": list(g), "mode": 2, "kernel_indices": [0, 1, 2, 3]}, h)
    ha = r["handle"]
    r = S.handle_request({"op": "forward", "handle": ha, "input": out, "output": str(tmp_path / "a.mvtf")}, h)
    assert r["ok"]
    ya = read_tensor(tmp_path / "a.mvtf").data
    assert O.max_abs_error(ya, O.activation_ref(y, 2, (0, 1, 2, 3))) <= 1e-5
    # fused block from the three handles
    r = S.handle_request({"op": "create_block", "conv1": hc, "act": ha, "conv2": hc, "residual": True}, h)
    hb = r["handle"]
    r = S.handle_request({"op": "forward", "handle": hb, "input": paths["x"], "output": str(tmp_path / "z.mvtf")}, h)
    assert r["ok"]
    z = read_tensor(tmp_path / "z.mvtf").data
    ref = O.block_ref(x, g, d, f1, b1, 2, (0, 1, 2, 3), None, None, f1, b1, padding="same", residual=True)
    assert O.max_rel_error(z, ref) <= 1e-4


@pytest.mark.gpu
def test_stdio_subprocess(tmp_path):
    rng = np.random.default_rng(0)
    w = (rng.standard_normal((4, 3, 2)) * 0.3).astype(np.float32)
    b = (rng.standard_normal((4, 3)) * 0.1).astype(np.float32)
    x = rng.standard_normal((5, 2, 4)).astype(np.float32)
    for n, a in [("w", w), ("b", b), ("x", x)]:
        write_tensor(tmp_path / f"{n}.mvtf", a)
    reqs = [{"op": "ping"},
            {"op": "create_linear", "sig": [1, 1], "weight": str(tmp_path / "w.mvtf"), "bias": str(tmp_path / "b.mvtf")},
            {"op": "forward", "handle": 1, "input": str(tmp_path / "x.mvtf"), "output": str(tmp_path / "y.mvtf")},
            {"op": "close", "handle": 1}, {"op": "exit"}]
    p = subprocess.run([sys.executable, "-m", "paper_2507_01040_b200", "serve"], cwd=ROOT,
                       input="\n".join(json.dumps(r) for r in reqs) + "\n", capture_output=True, text=True,
                       timeout=300)
    resp = [json.loads(l) for l in p.stdout.splitlines()]
    assert len(resp) == 5 and all(r["ok"] for r in resp), resp
    y = read_tensor(tmp_path / "y.mvtf").data
    assert O.max_rel_error(y, O.linear_ref(x, w, b, (1, 1))) <= 1e-4
