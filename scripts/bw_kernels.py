"""Bandwidth-bound kernels at the large shapes of SURVEY §8(d)-2, timed alone (CUDA events,
median of 5 after 2 warm-ups, L2 flushed before each run): algorithmic bytes / time against the
measured HBM copy peak.  One JSON line per kernel.  For the ncu DRAM counters run it under
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,...`.

    python scripts/bw_kernels.py [--quick]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import synth
from paper_2301_13659_b200 import spk

PEAK = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
quick = "--quick" in sys.argv


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def report(name, shape, nbytes, ms, note):
    gbs = nbytes / (ms * 1e-3) / 1e9
    print(json.dumps({"kernel": name, "shape": shape, "algorithmic_bytes": nbytes, "ms": ms, "GBps": gbs,
                      "hbm_frac": gbs / PEAK, "peak_GBps": PEAK, "note": note}), flush=True)


g = torch.Generator(device=dev).manual_seed(0)

# rank coding at C5 (4096 x 6 x 224 x 224 synthetic DoG responses): 4 B in + 1 B out per value
cfg = synth.load_config("c5")
B5 = 512 if quick else 4096
img = torch.from_numpy(synth.images_parallel(cfg, 0, 64)).to(dev).repeat((B5 // 64, 1, 1, 1))
y = spk.dog(img, cfg["front"]["pairs"], cfg["front"]["radius"], cfg["front"]["pad"])
lat = torch.empty(y.shape, dtype=torch.uint8, device=dev)
N = y[0].numel()
ms = timeit(lambda: spk.rank_code(y, 15, 0.01, True, out=lat))
report("rank_code (sort, C5)", [B5, N], 5 * y.numel(), ms, "4 B in + 1 B out per value")
ms = timeit(lambda: spk.dog(img, cfg["front"]["pairs"], cfg["front"]["radius"], cfg["front"]["pad"], out=y))
report("filter DoG (C5, FP32-issue bound)", list(y.shape), img.numel() + 4 * y.numel(), ms, "1 B in per pixel + 4 B out per value")
del y

# fire on materialised potentials, C4 conv1 16-image chunk [16][30][64][160][250] f32
P = torch.cumsum(torch.rand((16, 30, 64, 160, 250), device=dev, generator=g), dim=1)
fl = torch.empty((16, 64, 160, 250), dtype=torch.uint8, device=dev)
fp = torch.empty((16, 64, 160, 250), dtype=torch.float32, device=dev)
ms = timeit(lambda: spk.fire(P, 20.0, out=fl, pstar=fp))
report("fire (C4 conv1, 16-image chunk)", list(P.shape), P.numel() * 4 + fl.numel() * 5, ms, "4 T B in + 1 + 4 B out per neuron")
del P

# pooling, C5 conv1 unpooled latencies of a 512-image shard [512][128][224][224] -> 2x2
L = torch.randint(0, 16, (128 if quick else 512, 128, 224, 224), dtype=torch.uint8, device=dev, generator=g)
Lp = torch.empty((L.shape[0], 128, 112, 112), dtype=torch.uint8, device=dev)
ms = timeit(lambda: spk.pool(L, 15, 2, 2, 0, out=Lp))
report("pool 2x2 (C5 conv1, shard)", list(L.shape), L.numel() + Lp.numel(), ms, "1 B in + 1 B out (pooled)")
del L, Lp

# inhibition and k-WTA on C4 conv2 records [256][128][80][125]
lat = torch.randint(0, 31, (256, 128, 80, 125), dtype=torch.uint8, device=dev, generator=g)
lat[torch.rand(lat.shape, device=dev, generator=g) < 0.8] = 30
ps = torch.rand(lat.shape, device=dev, generator=g) + 1.0
l2, p2 = lat.clone(), ps.clone()
n = lat.numel()
ms = timeit(lambda: (l2.copy_(lat), p2.copy_(ps)))
ms_inh = timeit(lambda: (l2.copy_(lat), p2.copy_(ps), spk.inhibit(l2, p2, 30))) - ms
report("inhibit (C4 conv2 records)", list(lat.shape), 10 * n, ms_inh, "5 B in + 5 B out per neuron (copy-back time subtracted)")
ms = timeit(lambda: spk.wta(lat, ps, 30, 8, 1))
report("wta (C4 conv2 records, k=8 r=1)", list(lat.shape), 5 * n, ms, "5 B in per neuron")
ms = timeit(lambda: spk.inhibit_wta(lat, ps, 30, 8, 1))
report("inhibit_wta fused (C4 conv2 records)", list(lat.shape), 5 * n, ms, "5 B in per neuron (inhibited map not written)")
del lat, ps, l2, p2

# gather, C5 features [4096][512][28][28]
L = torch.randint(0, 16, (B5, 512, 28, 28), dtype=torch.uint8, device=dev, generator=g)
F = torch.empty(L.shape, dtype=torch.float32, device=dev)
ms = timeit(lambda: spk.gather(L, 15, out=F))
report("gather (C5 features)", list(L.shape), 5 * L.numel(), ms, "1 B in + 4 B out per neuron")
del L, F

# rate coding, C6 (256 x 6 x 28 x 28, T = 300): 4 B in + T B out per value
cfg6 = synth.load_config("c6")
img = torch.from_numpy(synth.images(cfg6, 0, 256)).to(dev)
y = spk.log(img, cfg6["front"]["stds"], 3, 3)
st = torch.empty((256, 300) + tuple(y.shape[1:]), dtype=torch.uint8, device=dev)
ms = timeit(lambda: spk.rate_code(y, 300, 0.01, 60606, out=st))
report("rate_code (C6, T=300)", [256, y[0].numel(), 300], 4 * y.numel() + st.numel(), ms,
       "4 B in + T B out per value; one splitmix64 draw per (step, neuron)")
r = torch.empty((256,) + tuple(y.shape[1:]), dtype=torch.float32, device=dev)
ms = timeit(lambda: spk.rate_gather(st, out=r))
report("rate_gather (C6 step maps)", list(st.shape), st.numel() + 4 * r.numel(), ms, "T B in + 4 B out per neuron")
