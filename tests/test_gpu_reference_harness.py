"""The B200 path run through the REFERENCE's own harness.

baseline/_ref holds the unmodified reference package (`pip install --target
baseline/_ref`). This test copies it to a
scratch directory, applies tests/reference_b200.patch -- the one branch per
dispatcher plus the bench.VARIANTS entry a maintainer would add
 -- and runs, in a fresh process:

  * the reference's parity_report (bench.py:566-637): every one of the 36
    signatures, with the b200 variant checked against the reference's own
    conv_reference / linear_reference / activation_reference at the
    reference's tolerances (1e-4 max_rel_error, 1e-5 max_abs_error);
  * run_sweep with verify=True (bench.py:338-412): the reference's
    verify-before-time of "b200" against variant "reference" for conv1d/2d/3d,
    linear and activation sweeps;
  * the reference CLI (`python -m mvkernels bench --variants reference,b200
    --verify`), cli.py:71-111.
"""

import json
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref", "mvkernels")
PATCH = os.path.join(ROOT, "tests", "reference_b200.patch")

SCRIPT = r"""
import json, sys, warnings
sys.path.insert(0, sys.argv[1])   # patched reference copy
sys.path.insert(1, sys.argv[2])   # this repo (paper_2507_01040_b200)
warnings.simplefilter("ignore")
import mvkernels
assert mvkernels.__file__.startswith(sys.argv[1]), mvkernels.__file__
from mvkernels import bench, algebra, activation as act
out = {}
rep = bench.parity_report(seed=0)
b200 = [e for e in rep.entries if e.name.endswith("/b200")]
out["parity"] = {"ok": rep.ok, "n": len(rep.entries), "n_b200": len(b200),
                 "b200_fail": [(e.name, e.max_err) for e in b200 if not e.ok],
                 "b200_max_conv": max(e.max_err for e in b200 if e.name.startswith("conv")),
                 "b200_max_act": max(e.max_err for e in b200 if e.name.startswith("activation")),
                 "b200_max_lin": max(e.max_err for e in b200 if e.name.startswith("linear")),
                 "sigs": sorted({e.name.split("/")[1] for e in b200 if e.name.startswith("conv")})}
sweeps = []
for kind, sig, kw in [("conv1d", (1,), dict(d_image=40)), ("conv2d", (1, 1), dict(d_image=12)),
                      ("conv2d", (1, -1), dict(d_image=10, d_filter=5)),
                      ("conv3d", (1, 1, 1), dict(d_image=8)), ("conv3d", (1, -1, 0), dict(d_image=7)),
                      ("linear", (1, 1, 1), dict(B=40)), ("activation", (1, 1, 1), dict(B=64)),
                      ("activation", (1, 1), dict(B=16, mode=act.AggMode.LINEAR, K=3))]:
    cfg = bench.BenchConfig(kind=kind, sig=algebra.Signature(sig), variants=("reference", "b200"),
                            verify=True, reps=3, warmup=1, sweep_channels=(4, 8), **kw)
    recs = bench.run_sweep(cfg)   # raises VerificationFailed on a miss
    sweeps += [{"kind": kind, "sig": list(sig), "variant": r.variant, "C": r.C_in, "err": r.max_err,
                "verified": r.verified} for r in recs]
out["sweeps"] = sweeps
print("RESULT " + json.dumps(out))
"""


@pytest.fixture(scope="module")
def patched_ref(tmp_path_factory):
    if not os.path.isdir(REF):
        pytest.skip("baseline/_ref/mvkernels missing: install the reference with "
                    "`python -m pip install --no-index --no-build-isolation --no-deps --target baseline/_ref "
                    "<copy of /root/reference/pkg>` (DESIGN.md)")
    pytest.importorskip("numba")
    d = tmp_path_factory.mktemp("ref")
    shutil.copytree(REF, d / "mvkernels")
    r = subprocess.run(["patch", "-p1", "-d", str(d), "-i", PATCH], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    return str(d)


def test_reference_parity_report_and_sweeps_with_b200(patched_ref):
    r = subprocess.run([sys.executable, "-c", SCRIPT, patched_ref, ROOT], capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")][-1]
    res = json.loads(line[len("RESULT "):])
    p = res["parity"]
    assert p["b200_fail"] == [], p["b200_fail"]
    assert p["ok"], p
    assert len(p["sigs"]) == 36, p["sigs"]          # conv b200 on every valid signature
    assert p["n_b200"] == 36 + 36 + 9, p["n_b200"]  # conv + linear per signature, activation k x mode
    sw = [s for s in res["sweeps"] if s["variant"] == "b200"]
    assert len(sw) == 16 and all(s["verified"] for s in sw), sw
    print(json.dumps(p))


def test_reference_cli_bench_b200(patched_ref):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([patched_ref, ROOT]))
    r = subprocess.run([sys.executable, "-m", "mvkernels", "bench", "--kind", "conv3d", "--sig", "1,1,1",
                        "--B", "8", "--Cin", "8", "--Cout", "8", "--dimage", "8", "--dfilter", "3",
                        "--variants", "reference,b200", "--verify", "--reps", "3", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=patched_ref)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "b200" in r.stdout, r.stdout
