"""The reference's OWN fastest CPU path, timed on the host cores (bench.py
--impl reference, and the `cpu_baseline` of bench.py's own line).

What runs is the unmodified reference package installed under
baseline/_ref (`pip install --target baseline/_ref`):

  conv        conv_forward(x, layer, "specialized")          conv.py:371-381
  activation  activation_forward(x, cfg, "specialized") on the serve fold
              (B, C, P, N_B) -> (B*P, C, N_B)                activation.py:400-416,
                                                             serve.py:108-117
  block       conv1 -> act -> conv2 + residual, composed from those calls
              as SURVEY 7 D1 states ("same" padding = valid conv on the
              zero-padded input; block.ts:134-148 + residual)

The reference is single-threaded by design, so it is run the
way BASELINE.md section 4 prescribes: one process per host core, pinned with
sched_setaffinity, each on its own 8-sample batch (the packed kernels need
B % 8 == 0 with the AVX2 width, layout.py:103-104). The numba JIT is compiled
once in the parent before the workers fork (warm-up, excluded from timing as
the reference harness does, bench.py:258-262).

Bounded samples: cfg1 and cfg2 run at full size per worker. For cfg3/4/5
each worker times the same per-voxel work on a spatial sub-volume (s^k
output voxels, their halo included) and the per-sample time is extrapolated
per output voxel of each stage (conv cost per output voxel does not depend on
the volume: measured 7.3 / 7.7 GFLOP/s at s = 4 / 6 on a cfg5 conv).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
L = 8  # samples per worker batch (the reference's packing width on AVX2 hosts)


def unavailable() -> str | None:
    """None when the reference package and numba are importable, else why not."""
    if not os.path.isdir(os.path.join(REF_DIR, "mvkernels")):
        return "baseline/_ref/mvkernels is not installed (pip install --target baseline/_ref <reference>)"
    try:
        import numba  # noqa: F401
    except ImportError:
        return "numba (the reference's JIT) is not importable"
    return None


def _mv():
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import mvkernels
    if not os.path.abspath(mvkernels.__file__).startswith(REF_DIR):
        raise RuntimeError(f"mvkernels imported from {mvkernels.__file__}, not {REF_DIR}")
    from mvkernels import activation, conv, layout, algebra
    return conv, activation, layout, algebra


def _fold(y):
    B, C, P, nb = y.shape
    return np.ascontiguousarray(y.transpose(0, 2, 1, 3)).reshape(B * P, C, nb)


def _unfold(a, B, C, P, nb):
    return np.ascontiguousarray(a.reshape(B, P, C, nb).transpose(0, 2, 1, 3))


def sub_side(spec) -> int:
    """Output side s of the timed sub-volume (full size for cfg1)."""
    if spec.kind == "conv" and spec.cfg == 1:
        return spec.d - spec.d_filter + 1
    return {2: 16, 3: 4}.get(spec.k, spec.d)


class Work:
    """The reference layers of one bounded sample and its stages."""

    def __init__(self, spec, seed=0):
        conv, act, layout, algebra = _mv()
        self.spec = spec
        k, nb, C = spec.k, spec.nb, spec.C
        sig = algebra.Signature(tuple(spec.g))
        rng = np.random.default_rng(seed)
        self.s = s = sub_side(spec)
        d_full_out = spec.d if spec.padding == "same" else spec.d - spec.d_filter + 1
        self.full_vox = d_full_out ** k
        fan = C * nb * spec.Q

        def filt(dims):
            f = (rng.uniform(-1, 1, dims.filters_shape()) / np.sqrt(fan)).astype(np.float32)
            b = (rng.standard_normal(dims.bias_shape()) * 0.01).astype(np.float32)
            return conv.make_conv_layer(dims, sig, f, b)

        self.conv, self.act = conv, act
        if spec.kind == "activation":
            self.x = rng.standard_normal((L, C, spec.P, nb), dtype=np.float32)
            w = rng.uniform(-0.5, 0.5, (C, nb)).astype(np.float32) if spec.mode == 0 else None
            b = (rng.standard_normal(C) * 0.1).astype(np.float32) if spec.mode == 0 else None
            self.acfg = act.make_activation_config(sig, spec.mode, tuple(range(nb)), w, b)
        elif spec.kind == "conv":
            self.l1 = filt(layout.Dims(L, C, C, s + spec.d_filter - 1, spec.d_filter, k))
            self.x = rng.standard_normal(self.l1.dims.input_shape(), dtype=np.float32)
        else:  # block: conv1 on (s+4)^k -> (s+2)^k, act, conv2 -> s^k, + residual
            self.l1 = filt(layout.Dims(L, C, C, s + 4, 3, k))
            self.l2 = filt(layout.Dims(L, C, C, s + 2, 3, k))
            w = rng.uniform(-0.5, 0.5, (C, nb)).astype(np.float32) if spec.mode == 0 else None
            b = (rng.standard_normal(C) * 0.1).astype(np.float32) if spec.mode == 0 else None
            self.acfg = act.make_activation_config(sig, spec.mode, tuple(range(nb)), w, b)
            self.x = rng.standard_normal(self.l1.dims.input_shape(), dtype=np.float32)

    def step(self):
        """One timed step: per-stage seconds."""
        sp = self.spec
        t0 = time.perf_counter()
        if sp.kind == "activation":
            B, C, P, nb = self.x.shape
            a = self.act.activation_forward(_fold(self.x), self.acfg, "specialized")
            _unfold(a, B, C, P, nb)
            return [time.perf_counter() - t0]
        y1 = self.conv.conv_forward(self.x, self.l1, "specialized")
        t1 = time.perf_counter()
        if sp.kind == "conv":
            return [t1 - t0]
        B, C, P, nb = y1.shape
        a = _unfold(self.act.activation_forward(_fold(y1), self.acfg, "specialized"), B, C, P, nb)
        t2 = time.perf_counter()
        y2 = self.conv.conv_forward(a, self.l2, "specialized")
        k, s = sp.k, self.s
        xin = self.x.reshape((B, C) + (s + 4,) * k + (nb,))
        crop = xin[(slice(None), slice(None)) + (slice(2, 2 + s),) * k]
        y2 += crop.reshape(y2.shape)
        t3 = time.perf_counter()
        return [t1 - t0, t2 - t1, t3 - t2]

    def per_sample_seconds(self, st):
        """Full-size seconds per sample from one step's stage times."""
        sp, k, s = self.spec, self.spec.k, self.s
        if sp.kind == "activation":
            return st[0] / L
        if sp.kind == "conv":
            return st[0] * self.full_vox / s ** k / L
        return ((st[0] + st[1]) * self.full_vox / (s + 2) ** k + st[2] * self.full_vox / s ** k) / L

    def sample_desc(self):
        sp = self.spec
        if sp.kind == "activation":
            return f"{L} of {sp.B} samples (full size) per worker, serve fold + activation_forward(specialized)"
        if sp.kind == "conv" and sp.cfg == 1:
            return f"full cfg1 batch ({L} samples) per worker, conv_forward(specialized)"
        what = "conv_forward(specialized)" if sp.kind == "conv" else \
            "conv(specialized) -> fold + activation(specialized) -> conv(specialized) + residual"
        return (f"{L} samples x {self.s}^{sp.k} output voxels (with halo) per worker, {what}; "
                f"per-sample time extrapolated per output voxel to {self.full_vox} voxels")


_W = None


def _worker(args):
    core, steps, warmup = args
    try:
        os.sched_setaffinity(0, {core})
    except (AttributeError, OSError):
        pass
    for _ in range(warmup):
        _W.step()
    return [_W.step() for _ in range(steps)]


def time_reference(spec, steps: int, warmup: int, cores: int | None = None, seed: int = 0) -> dict:
    """Run the reference path on `cores` pinned processes (default: every
    core this process may use). Returns the aggregate throughput."""
    global _W
    avail = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else list(range(os.cpu_count()))
    use = avail[: cores or len(avail)]
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS"):
        os.environ[v] = "1"
    _W = Work(spec, seed)
    t0 = time.perf_counter()
    _W.step()  # numba JIT of every kernel used, in the parent (inherited by the forked workers)
    t_jit = time.perf_counter() - t0
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(len(use)) as pool:
        res = pool.map(_worker, [(c, steps, warmup) for c in use])
    wall = time.perf_counter() - t0
    per_sample = [[_W.per_sample_seconds(st) for st in r] for r in res]  # [worker][step]
    rate = sum(1.0 / float(np.mean(ps)) for ps in per_sample)            # samples/s over all workers
    step_s = float(np.mean([sum(st) for r in res for st in r]))
    out = {"samples_per_s": rate, "cores": len(use), "step_s": step_s, "wall_s": wall, "jit_s": t_jit,
           "per_sample_s": float(np.mean([np.mean(ps) for ps in per_sample])),
           "sample": _W.sample_desc(), "sub_side": _W.s}
    if spec.kind == "activation":
        out["gbs"] = rate * 2 * spec.C * spec.P * spec.nb * 4 / 1e9
    _W = None
    return out
