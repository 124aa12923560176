"""Freeze the calibrated IF thresholds of configs whose layers say "theta": null.

Reading R-THETA-CAL: the paper and BASELINE.json give no threshold
for these layers, so theta_l = the 80th percentile of the final-step potentials
P[T-1] of layer l over global images 0..15 of the config's seed (earlier layers
at their own thresholds), rounded to 3 significant figures, then written into
configs/<name>.json.  Calls only oracle/ (the CPU oracle) and synth/; images are
processed one at a time so the fp64 potentials of big layers fit in memory.
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle  # noqa: E402
from oracle import pipeline  # noqa: E402
import synth  # noqa: E402


def calibrate(name: str, n_images: int = 16) -> dict:
    cfg = synth.load_config(name)
    Ws = pipeline.quantized_weights(cfg, synth.layer_weights(cfg))  # Listing 4 layers quantized
    T = cfg["T"]
    nl = len(cfg["layers"])
    for li in range(nl):
        L = cfg["layers"][li]
        if L["theta"] is not None:
            continue
        finals = []
        for q in range(n_images):
            img = synth.images(cfg, q, 1)
            _, lat = pipeline.front_end(cfg, img)
            for lj in range(li + 1):
                Lj = cfg["layers"][lj]
                P = oracle.conv_event(lat, T, Ws[lj], (Lj["stride"],) * 2, (Lj["pad"],) * 2)
                if lj == li:
                    finals.append(P[:, T - 1].ravel())
                    break
                S = oracle.fire(P, Lj["theta"])
                del P
                if Lj["pool"]:
                    p = Lj["pool"]
                    S = oracle.pool(S, (p["kernel"],) * 2, (p["stride"],) * 2, (p["pad"],) * 2)
                lat = oracle.dense_to_lat(S)
        L["theta"] = pipeline.sig3(float(np.percentile(np.concatenate(finals), 80)))
        print(f"{name} layer {li}: theta = {L['theta']}", flush=True)
    path = synth.CONFIG_DIR / f"{name.lower()}.json"
    raw = json.loads(path.read_text())
    for li, L in enumerate(cfg["layers"]):
        raw["layers"][li]["theta"] = L["theta"]
    path.write_text(json.dumps(raw, indent=2) + "\n")
    return cfg


if __name__ == "__main__":
    for n in sys.argv[1:] or ["c2", "c3"]:
        calibrate(n)
