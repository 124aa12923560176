"""Quick GPU check of the tcgen05 conv on tiny shapes (debug aid)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import oracle
from paper_2301_13659_b200 import spk
rng = np.random.default_rng(0)
for (B, T, Ci, H, W, Co, K, s, p) in [(1, 15, 1, 4, 4, 16, 1, 1, 0), (1, 15, 2, 6, 6, 16, 3, 1, 1), (2, 15, 6, 28, 28, 30, 5, 1, 2), (3, 15, 250, 4, 4, 200, 5, 1, 2)]:
    lat = rng.integers(0, T, (B, Ci, H, W)).astype(np.uint8)
    lat[rng.random(lat.shape) > 0.5] = T
    w = rng.uniform(0, 1, (Co, Ci, K, K)).astype(np.float32)
    ref = oracle.conv_event(lat, T, w, (s, s), (p, p))
    for prec in ["fp32", "exact"]:
        got = spk.conv(torch.from_numpy(lat).cuda(), torch.from_numpy(w).cuda(), T, s, p, prec=prec, epi="potential")
        torch.cuda.synchronize()
        got = got.cpu().numpy()
        err = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-6)
        print((B, T, Ci, H, W, Co, K), prec, "max rel err", err.max(), "mismatch frac", (err > 1e-5).mean(), flush=True)
        if err.max() > 1e-5:
            idx = np.argwhere(err > 1e-5)[:5]
            for i in idx: print("   ", tuple(i), got[tuple(i)], ref[tuple(i)])
