"""Measure dense tensor-core GEMM peaks per MMA kind on this GPU with cuBLAS
(torch.matmul / torch._int_mm), the same way MEASURED_PEAKS.json's bf16 figure
is taken: 8192^3, best of 10 (burst) and back-to-back for ~4 s (sustained).
Writes profiles/<out>.json. These are the roofline denominators of the
tf32 / 3xtf32 / fp32 (int8 digit) conv modes."""
import json
import sys
import time

import torch

out = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_mode_peaks.json"
torch.cuda.set_device(0)
n = 8192
res = {"gpu": torch.cuda.get_device_name(0), "n": n}


def bench(fn, flops):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    t0 = time.time(); cnt = 0
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    while time.time() - t0 < 4.0:
        fn(); cnt += 1
        if cnt % 8 == 0:
            torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    sus = e0.elapsed_time(e1) / 1e3 / cnt
    return flops / best / 1e12, flops / sus / 1e12


f = 2.0 * n ** 3
a = torch.randn(n, n, device="cuda", dtype=torch.bfloat16); b = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
res["bf16_tflops"], res["bf16_tflops_sustained"] = bench(lambda: a @ b, f)
torch.backends.cuda.matmul.allow_tf32 = True
a32 = torch.randn(n, n, device="cuda"); b32 = torch.randn(n, n, device="cuda")
res["tf32_tflops"], res["tf32_tflops_sustained"] = bench(lambda: a32 @ b32, f)
ai = torch.randint(-64, 64, (n, n), device="cuda", dtype=torch.int8)
bi = torch.randint(-64, 64, (n, n), device="cuda", dtype=torch.int8)
res["int8_tops"], res["int8_tops_sustained"] = bench(lambda: torch._int_mm(ai, bi), f)
torch.backends.cuda.matmul.allow_tf32 = False
res["fp32_simt_tflops"], res["fp32_simt_tflops_sustained"] = bench(lambda: a32 @ b32, f)
res["how"] = "cuBLAS via torch (matmul bf16 / tf32 / fp32, _int_mm int8), 8192^3, best of 10 and ~4 s back-to-back"
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
