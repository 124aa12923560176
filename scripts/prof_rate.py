"""Per-role cycle accounting of the tcgen05 conv on the rate-coded C6 layers (T' = 1, TP = 1 path);
debug aid: needs a libspk built with -DSPK_CONV_PROF_BUILD (SPK_LIB_OVERRIDE) and SPK_CONV_PROF=1."""
import ctypes, os, sys
os.environ["SPK_CONV_PROF"] = "1"
sys.path.insert(0, ".")
import numpy as np, torch
import synth
from paper_2301_13659_b200 import spk
from paper_2301_13659_b200.network import RateNetwork
cfg = synth.load_config("c6")
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
net = RateNetwork(cfg, B, prec="exact")
net.img.copy_(torch.from_numpy(synth.images(cfg, 0, B)))
net.set_weights([torch.from_numpy(w) for w in synth.layer_weights(cfg)])
net.front()
L = spk.lib()
buf = np.zeros((1024, 25, 2), np.uint64)
names = ["producer", "epilogue", "mma", "bload", "band"]
for li in range(len(net.layers)):
    for rep in range(2):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); net.layer(li); e1.record(); torch.cuda.synchronize()
    L.spk_debug_conv_prof(buf.ctypes.data_as(ctypes.c_void_p))
    ms = e0.elapsed_time(e1)
    tot = buf[:148, :, 0].astype(float); wt = buf[:148, :, 1].astype(float)
    print(f"layer {li}: {ms:.3f} ms (incl. rates/pool) " + "  ".join(f"{n}: busy {np.mean(tot[:, i]-wt[:, i])/1e3:.0f}k wait {np.mean(wt[:, i])/1e3:.0f}k" for i, n in enumerate(names))
          + f"  | mma fence {np.mean(tot[:, 5])/1e3:.0f}k issue {np.mean(tot[:, 6])/1e3:.0f}k commit {np.mean(tot[:, 7])/1e3:.0f}k"
          + "  | T=1 prod region/gather/slot-wait/store " + " ".join(f"{np.mean(tot[:, 8 + q])/1e3:.0f}k" for q in range(4))
          + "  | epi lead wait/barsync/work/tail " + " ".join(f"{np.mean(tot[:, 17 + q])/1e3:.0f}k" for q in range(4))
          + "  warp5 sync+wait/work " + " ".join(f"{np.mean(tot[:, 21 + q])/1e3:.0f}k" for q in range(2)))
