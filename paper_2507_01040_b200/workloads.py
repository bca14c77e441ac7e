"""Seeded synthetic workloads of BASELINE.json configs 1-5.

Inputs are generated on the device, per GLOBAL sample index, so values do
not depend on how the batch is sharded across ranks (D2). Small
parameter tensors are generated on the host with numpy SeedSequence
([seed, cfg, tensor_id]) and are identical on every rank.

Distributions (BASELINE.json configs; interpretations stated in DESIGN.md):
  input  ~ N(0, 1)
  conv filters ~ U(+-1/sqrt(C_in * N_B * Q)); cfg1 bias ~ N(0, 0.01^2);
  block conv biases ~ U(+-1/sqrt(fan_in)) with fan_in = C_in * N_B * Q
  activation Linear weights ~ U(+-0.5), Linear bias ~ N(0, 0.1^2)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEED = 20250701


@dataclass(frozen=True)
class ConfigSpec:
    cfg: int
    kind: str          # "conv" | "activation" | "block"
    g: tuple
    B: int
    C: int
    d: int
    d_filter: int = 3
    padding: str = "valid"
    mode: int = 0      # activation aggregation mode (block / activation configs)
    name: str = ""

    @property
    def k(self):
        return len(self.g)

    @property
    def nb(self):
        return 1 << len(self.g)

    @property
    def P(self):
        return self.d ** self.k

    @property
    def Q(self):
        return self.d_filter ** self.k


CONFIGS = {
    1: ConfigSpec(1, "conv", (1, 1), 8, 16, 32, name="cfg1: 2D conv g=(1,1) B=8 C=16 32^2 f=3 valid"),
    2: ConfigSpec(2, "activation", (1, 1), 64, 64, 64, mode=0,
                  name="cfg2: 2D activation (64,64,4096,4) over all 4 blades"),
    3: ConfigSpec(3, "block", (1, 1), 32, 64, 128, padding="same", mode=0,
                  name="cfg3: 2D block conv3x3-act(Linear)-conv3x3+res B=32 C=64 128^2"),
    4: ConfigSpec(4, "conv", (1, 1, 1), 16, 32, 32, name="cfg4: 3D conv g=(1,1,1) B=16 C=32 32^3 f=3 valid"),
    40: ConfigSpec(40, "conv", (1, -1, 0), 16, 32, 32, name="cfg4b: 3D conv g=(1,-1,0) B=16 C=32 32^3 f=3 valid"),
    5: ConfigSpec(5, "block", (1, 1, 1), 256, 64, 32, padding="same", mode=2,
                  name="cfg5: 3D block conv3^3-act(Mean)-conv3^3+res B=256 C=64 32^3"),
}


def _rng(*key):
    return np.random.default_rng(np.random.SeedSequence([SEED, *[int(k) for k in key]]))


def conv_params(spec: ConfigSpec, layer: int = 1):
    """(filters (N_B, C, C, Q), bias (N_B, C)) as float32 numpy."""
    nb, C, Q = spec.nb, spec.C, spec.Q
    fan = C * nb * Q
    r = _rng(spec.cfg, 10 + layer)
    bound = 1.0 / np.sqrt(fan)
    f = r.uniform(-bound, bound, (nb, C, C, Q)).astype(np.float32)
    if spec.kind == "conv":
        b = (r.standard_normal((nb, C)) * 0.01).astype(np.float32)
    else:
        b = r.uniform(-bound, bound, (nb, C)).astype(np.float32)
    return f, b


def act_params(spec: ConfigSpec):
    """(weight (C, N_B), bias (C,)) for Linear mode, else (None, None)."""
    if spec.mode != 0:
        return None, None
    r = _rng(spec.cfg, 20)
    w = r.uniform(-0.5, 0.5, (spec.C, spec.nb)).astype(np.float32)
    b = (r.standard_normal(spec.C) * 0.1).astype(np.float32)
    return w, b


def input_shape(spec: ConfigSpec, B=None):
    return (spec.B if B is None else B, spec.C, spec.P, spec.nb)


def make_input(spec: ConfigSpec, b0: int, nb_samples: int, device="cuda", out=None):
    """Samples [b0, b0+nb_samples) of the config input, generated on `device`."""
    import torch
    shape = (nb_samples, spec.C, spec.P, spec.nb)
    x = out if out is not None else torch.empty(shape, device=device, dtype=torch.float32)
    gen = torch.Generator(device=device)
    for i in range(nb_samples):
        gen.manual_seed(int(np.random.SeedSequence([SEED, spec.cfg, 0, b0 + i]).generate_state(1)[0]))
        x[i].normal_(0.0, 1.0, generator=gen)
    return x


def shard(B: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous batch slice [lo, hi) of rank `rank` (SURVEY 8e partitioning)."""
    base, rem = divmod(B, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)
