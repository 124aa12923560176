"""Freeze the per-step IF thresholds of a rate-coded config (configs/c6.json) — oracle only.

Reading R-THETA-CAL-RATE: with rate coding the potential of step t is the
convolution of that step's spikes (Eq. 2 per step), and the weights are quantized to {0, 1}
(Listing 4), so per-step potentials are small integers.  theta_l = the 90th percentile of the
POSITIVE per-step potentials of layer l over global images 0..7 (earlier layers at their frozen
thresholds, rate pooling as configured), rounded to 3 significant figures — about a tenth of the
active (neuron, step) pairs fire.  Calls only oracle/ and synth/.
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle  # noqa: E402
from oracle import pipeline  # noqa: E402
import synth  # noqa: E402


def calibrate(name: str, n_images: int = 8, pct: float = 90.0) -> dict:
    cfg = synth.load_config(name)
    Ws = pipeline.quantized_weights(cfg, synth.layer_weights(cfg))
    for li, L in enumerate(cfg["layers"]):
        if L["theta"] is not None:
            continue
        vals = []
        for q in range(n_images):
            S = pipeline.rate_front_end(cfg, synth.images(cfg, q, 1), q)
            for lj in range(li + 1):
                Lj = cfg["layers"][lj]
                P = oracle.conv(S, Ws[lj], (Lj["stride"],) * 2, (Lj["pad"],) * 2)
                if lj == li:
                    vals.append(P[P > 0].ravel())
                    break
                S = oracle.fire(P, Lj["theta"])
                p = Lj["pool"]
                if p:
                    r = oracle.gather(S)
                    S = oracle.pool_rates(S, r, (p["kernel"],) * 2, (p["stride"],) * 2, (p["pad"],) * 2)
        v = np.concatenate(vals)
        L["theta"] = pipeline.sig3(float(np.percentile(v, pct)))
        print(f"{name} layer {li}: theta = {L['theta']} (positive per-step potentials: n={v.size}, "
              f"median {np.median(v)}, max {v.max()})", flush=True)
    path = synth.CONFIG_DIR / f"{name.lower()}.json"
    raw = json.loads(path.read_text())
    for li, L in enumerate(cfg["layers"]):
        raw["layers"][li]["theta"] = L["theta"]
    path.write_text(json.dumps(raw, indent=2) + "\n")
    return cfg


if __name__ == "__main__":
    for n in sys.argv[1:] or ["c6"]:
        calibrate(n)
