"""Per-layer conv timing (median of 7, no profiling) of the C2 network — A/B aid.

SPK_LIB_OVERRIDE selects the library; prints one line `tag conv0 conv1 conv2` in ms."""
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
import synth
from paper_2301_13659_b200.network import Network
cfg = synth.load_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
tag = sys.argv[2] if len(sys.argv) > 2 else os.environ.get("SPK_LIB_OVERRIDE", "base")
B = cfg["batch"]
net = Network(cfg, B, prec=os.environ.get("SPK_PREC", "exact"))
net.img.copy_(torch.from_numpy(synth.images(cfg, 0, B)))
net.set_weights([torch.from_numpy(w) for w in synth.layer_weights(cfg)])
net.front()
out = []
for li in range(len(net.layers)):
    ts = []
    for rep in range(8):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); net.layer(li, pstar=(li == cfg.get("train_layer"))); e1.record(); torch.cuda.synchronize()
        if rep: ts.append(e0.elapsed_time(e1))
    out.append(float(np.median(ts)))
print(tag, " ".join(f"{t:.3f}" for t in out))
