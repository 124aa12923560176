"""Event timestamps of CTA 0 of the tcgen05 conv (libspk built with -DSPK_CONV_TRACE)."""
import ctypes, os, sys
sys.path.insert(0, ".")
import numpy as np, torch
import synth
from paper_2301_13659_b200 import spk
from paper_2301_13659_b200.network import Network
cfg = synth.load_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
B = cfg["batch"]
net = Network(cfg, B)
net.img.copy_(torch.from_numpy(synth.images(cfg, 0, B)))
net.set_weights([torch.from_numpy(w) for w in synth.layer_weights(cfg)])
net.front()
L = spk.lib()
tr = np.zeros((12, 256), np.int64)
names = ["mma_commit_accf", "epi_wake", "epi_done", "mma_acce_wake", "fl_wake", "fl_done"]
for li in range(len(net.layers)):
    for rep in range(2):
        net.layer(li, pstar=(li == cfg.get("train_layer")))
        torch.cuda.synchronize()
    L.spk_debug_conv_trace(tr.ctypes.data_as(ctypes.c_void_p))
    t = tr - tr[0, 0]
    n = 256
    sl = slice(16, 200)
    d = lambda a, b, lag=0: np.median((t[b, sl.start + lag:sl.stop + lag] - t[a, sl]))
    print(f"layer {li}: per-tile period mma {np.median(np.diff(t[0, sl])):.0f}  epi {np.median(np.diff(t[2, sl])):.0f}  fl {np.median(np.diff(t[5, sl])):.0f} cycles")
    print(f"   commit->epi_wake {d(0, 1):.0f}  epi_wake->epi_done {d(1, 2):.0f}  epi_done->mma_acce_wake(+NB) "
          f"{np.median(t[3, sl.start + 4:sl.stop + 4] - t[2, sl]):.0f}  acce_wake->commit {d(3, 0):.0f}  "
          f"epi_done->fl_wake {d(2, 4):.0f}  fl_wake->fl_done {d(4, 5):.0f}")
    print("   first tiles (mma commit):", (t[0, :8]).tolist())
    print("   stages: prod granted", np.diff(t[6, 16:24]).tolist(), " mma stage-wake", np.diff(t[7, 16:40]).tolist())
    print("   mma stage wakes rel. to tile acce-wake:", [(t[7, k] - t[3, 0]) for k in range(0, 12)], "tile commits:", [(t[0, k] - t[3, 0]) for k in range(0, 4)], "acce wakes:", [(t[3, k] - t[3, 0]) for k in range(0, 4)])
    print("   prod granted -> mma wake (same stage):", (t[7, 16:32] - t[6, 16:32]).tolist())
    print("   mma wait3 duration per stage:", (t[7, 16:40] - t[9, 16:40]).tolist())
    print("   B copy issue -> mma wake (same B stage):", (t[7, 16:40] - t[8, 16:40]).tolist())
    print("   B copy issue deltas:", np.diff(t[8, 16:40]).tolist())
    print("   per stage: wait3", (t[7, 16:28] - t[9, 16:28]).tolist())
    print("   per stage: issue", (t[10, 16:28] - t[7, 16:28]).tolist())
    print("   per stage: commits", (t[11, 16:28] - t[10, 16:28]).tolist())
    print("   per stage: to next wait", (t[9, 17:29] - t[11, 16:28]).tolist())
    gpt = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # hand-offs per tile (to line up tile boundaries)
    if gpt:
        for i in range(1, 4):
            c, ew, ed, mw0, mw1 = t[0, i - 1], t[1, i - 1], t[2, i - 1], t[9, i * gpt], t[7, i * gpt]
            print(f"   tile {i-1}->{i}: accf commit issued {c}, epi wake +{ew - c}, epi done +{ed - c}, "
                  f"MMA starts waiting +{mw0 - c}, MMA wakes +{mw1 - c}")
