import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
import paper_2507_01040_b200 as M
rng = np.random.default_rng(0)
for g, B, C, d, prec in [((1, 1), 2, 4, 6, "fp32"), ((1, 1), 4, 16, 32, "fp32"), ((1, 1), 4, 16, 32, "tf32"), ((1, 1, 1), 4, 8, 8, "fp32")]:
    k = len(g); nb = 1 << k
    x = rng.standard_normal((B, C, d ** k, nb)).astype(np.float32)
    f = (rng.uniform(-1, 1, (nb, C, C, 3 ** k)) / np.sqrt(C * nb * 3 ** k)).astype(np.float32)
    b = np.zeros((nb, C), np.float32)
    layer = M.make_conv_layer(M.Dims(B, C, C, d, 3, k), M.Signature(g), f, b, precision=prec)
    y = M.conv_forward(torch.from_numpy(x).cuda(), layer).cpu().numpy()
    ref = O.conv_ref(x, f, b, g, d, 3, 0)
    print(g, B, C, d, prec, "per-sample err:", [f"{O.max_rel_error(y[i], ref[i], floor=1.0):.1e}" for i in range(B)])
