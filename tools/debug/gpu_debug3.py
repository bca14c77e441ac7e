"""Debug helper: run each golden conv case in fp32 and report CUDA errors."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2507_01040_b200 as M
n = int(sys.argv[1])
gd = np.load("tests/golden/golden.npz")
g = tuple(int(v) for v in gd[f"conv{n}_g"])
B, ci, co, di, df, k = (int(v) for v in gd[f"conv{n}_dims"])
layer = M.make_conv_layer(M.Dims(B, ci, co, di, df, k), M.Signature(g), gd[f"conv{n}_f"], gd[f"conv{n}_b"], precision=sys.argv[2] if len(sys.argv) > 2 else "fp32")
x = torch.from_numpy(gd[f"conv{n}_x"]).cuda()
try:
    y = M.conv_forward(x, layer).cpu().numpy()
    ref = gd[f"conv{n}_y"]
    print(n, g, (B, ci, co, di, df, k), "err", float(np.abs(y - ref).max() / (np.abs(ref).max() + 1e-30)))
except Exception as e:
    print(n, g, (B, ci, co, di, df, k), "EXC", str(e)[:300])
