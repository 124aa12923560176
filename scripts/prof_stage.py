"""Run one stage of a config's pipeline at full batch (for ncu captures of a single kernel).

    python scripts/prof_stage.py c5 rank_code      # front end then rank coding
    python scripts/prof_stage.py c4 wta            # forward to the trained layer, inhibit, then WTA
"""
import sys
sys.path.insert(0, ".")
import torch
import synth
from paper_2301_13659_b200 import spk
from paper_2301_13659_b200.network import Network

cfg = synth.load_config(sys.argv[1])
stage = sys.argv[2]
B = int(sys.argv[3]) if len(sys.argv) > 3 else cfg["batch"]
net = Network(cfg, B, prec="auto")
net.img.copy_(torch.from_numpy(synth.images_parallel(cfg, 0, B)))
net.set_weights([torch.from_numpy(w) for w in synth.layer_weights(cfg)])
fr = cfg["front"]
net.front()
torch.cuda.synchronize()
if stage == "rank_code":
    for _ in range(3):
        spk.rank_code(net.y, net.T, fr["thresh"], fr["sort"], out=net.lat0)
elif stage in ("wta", "inhibit"):
    tl = cfg["train_layer"]
    for li in range(tl):
        net.layer(li)
    net.layer(tl, pstar=True)
    rec = net.layers[tl]
    lat, ps = rec["lat"].clone(), rec["pstar"].clone()
    for _ in range(3):
        rec["lat"].copy_(lat)
        rec["pstar"].copy_(ps)
        spk.inhibit(rec["lat"], rec["pstar"], net.T)
        spk.wta(rec["lat"], rec["pstar"], net.T, net.k, rec["L"]["wta"]["radius"], win=net.win, nwin=net.nwin)
torch.cuda.synchronize()
print("done", stage)
