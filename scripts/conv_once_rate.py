"""C6 (rate-coded, T' = 1) front end, then every conv layer once — for ncu --set full captures of the
TP = 1 tcgen05 path:  ncu --set full -k regex:conv_tc_kernel -c 1 python scripts/conv_once_rate.py [B]"""
import sys
sys.path.insert(0, ".")
import torch
import synth
from paper_2301_13659_b200.network import RateNetwork

cfg = synth.load_config("c6")
B = int(sys.argv[1]) if len(sys.argv) > 1 else cfg["batch"]
net = RateNetwork(cfg, B, prec="auto")
net.img.copy_(torch.from_numpy(synth.images(cfg, 0, B)))
net.set_weights([torch.from_numpy(w) for w in synth.layer_weights(cfg)])
net.front()
for li in range(len(net.layers)):
    net.layer(li)
torch.cuda.synchronize()
print("layers", [r["prec"] for r in net.layers])
