"""Front end, then every conv layer of a config once (one launch per layer) — for ncu --set full captures.

    SPK_PREC=auto ncu --set full -k regex:"conv_(tc|event)_kernel" -c 3 python scripts/conv_once.py c2
"""
import os, sys
sys.path.insert(0, ".")
import torch
import synth
from paper_2301_13659_b200.network import Network

cfg = synth.load_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
B = int(sys.argv[2]) if len(sys.argv) > 2 else cfg["batch"]
net = Network(cfg, B, prec=os.environ.get("SPK_PREC", "auto"))
net.img.copy_(torch.from_numpy(synth.images_parallel(cfg, 0, B)))
net.set_weights([torch.from_numpy(w) for w in synth.layer_weights(cfg)])
net.front()
for li in range(len(net.layers)):
    net.layer(li, pstar=(li == cfg.get("train_layer")))
torch.cuda.synchronize()
print("layers", [r["prec"] for r in net.layers])
