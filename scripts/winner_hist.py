"""Distribution of STDP winners over output maps for one train step (debug aid)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import synth
from paper_2301_13659_b200.network import Network
cfg = synth.load_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
B = cfg["batch"]
net = Network(cfg, B)
net.img.copy_(torch.from_numpy(synth.images(cfg, 0, B)))
net.set_weights([torch.from_numpy(w) for w in synth.layer_weights(cfg)])
net.train_step()
torch.cuda.synchronize()
win, nwin = net.win.cpu().numpy(), net.nwin.cpu().numpy()
maps = np.concatenate([win[b, :nwin[b], 2] for b in range(B)])
h = np.bincount(maps)
print("winners", len(maps), "maps hit", (h > 0).sum(), "max per map", h.max(), "top", np.sort(h)[-8:])
