"""Small end-to-end runs through every kernel family for compute-sanitizer:
C1 train step on both conv engines (conv_tc_kernel, conv_event_kernel, inhibit, WTA cluster,
STDP), a C2 train step at batch 4 (event conv0, tcgen05 conv1/conv2 with P*, small-map
inhibition, one-warp WTA), a C4-shaped large-map WTA/inhibit, rate coding + rate pooling
(C6 at batch 1), FC + fcwta, ZCA.  One compute-sanitizer tool per invocation:

    compute-sanitizer --tool racecheck python scripts/sanitize_once.py
"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import synth
from paper_2301_13659_b200 import spk
from paper_2301_13659_b200.network import Network, RateNetwork

torch.cuda.set_device(0)


def run(name, B, prec):
    cfg = synth.load_config(name)
    net = Network(cfg, B, prec=prec)
    net.img.copy_(torch.from_numpy(synth.images(cfg, 0, B)))
    net.labels.copy_(torch.from_numpy(synth.labels(cfg, 0, B)))
    net.set_weights([torch.from_numpy(w) for w in synth.layer_weights(cfg)])
    net.train_step()
    torch.cuda.synchronize()
    print(name, prec, "winners", int(net.nwin.sum()), flush=True)


run("c1", 1, "exact")
run("c1", 1, "event")
run("c2", 4, "auto")
run("c2q", 2, "auto")
# large maps: wide inhibition and an 8-CTA WTA cluster with the per-pixel top-k pre-reduction
rng = np.random.default_rng(0)
lat = torch.from_numpy(rng.integers(0, 16, (2, 40, 60, 70)).astype(np.uint8)).cuda()
ps = torch.from_numpy(rng.uniform(1, 2, (2, 40, 60, 70)).astype(np.float32)).cuda()
spk.inhibit(lat, ps, 15)
spk.wta(lat, ps, 15, 5, 3)
# NEXT-3: rate coding, per-step conv/fire, rate pooling (C6, batch 1)
cfg = synth.load_config("c6")
rn = RateNetwork(cfg, 1, prec="auto")
rn.img.copy_(torch.from_numpy(synth.images(cfg, 0, 1)))
rn.set_weights([torch.from_numpy(w) for w in synth.layer_weights(cfg)])
rn.infer()
# NEXT-4: FC + fcwta, ZCA
lat = torch.from_numpy(rng.integers(0, 16, (3, 300)).astype(np.uint8)).cuda()
w = torch.from_numpy(rng.uniform(0, 1, (40, 300)).astype(np.float32)).cuda()
l2, p2 = spk.fc(lat, w, 15, prec="exact", epi="fire", theta=50.0)
spk.fcwta(l2, p2, 15, 3, 1)
x = torch.from_numpy(rng.normal(0, 1, (64, 48)).astype(np.float32)).cuda()
m, wz = spk.zca_fit(x, 0.1)
spk.zca_apply(x, m, wz)
torch.cuda.synchronize()
print("sanitize_once done", flush=True)
