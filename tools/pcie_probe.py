"""Host<->device copy bandwidth from pinned memory (H2D, D2H, both at once), to
read the e2e line against: the cfg5 e2e step moves 17.2 GB each way."""
import os
import sys
import time

import torch

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else (2 << 30)
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


th = t(lambda: d.copy_(h, non_blocking=True))
td = t(lambda: h2.copy_(d2, non_blocking=True))
tb = t(both)
print(f"affinity {len(os.sched_getaffinity(0))} cpus; H2D {n / th / 1e9:.1f} GB/s, D2H {n / td / 1e9:.1f} GB/s, "
      f"both at once {n / tb / 1e9:.1f} + {n / tb / 1e9:.1f} GB/s", flush=True)
