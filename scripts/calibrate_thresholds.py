"""Freeze the calibrated IF thresholds of configs whose layers say "theta": null.

Reading R-THETA-CAL: the paper and BASELINE.json give no threshold
for these layers, so theta_l = the 80th percentile of the final-step potentials
P[T-1] of layer l over global images 0..15 of the config's seed (earlier layers
at their own thresholds), rounded to 3 significant figures, then written into
configs/<name>.json.  Calls only oracle/ (the CPU oracle) and synth/.
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
    imgs = synth.images(cfg, 0, n_images)
    Ws = synth.layer_weights(cfg)
    T = cfg["T"]
    _, lat0 = pipeline.front_end(cfg, imgs)
    S = oracle.lat_to_dense(lat0, T)
    for li, L in enumerate(cfg["layers"]):
        P = oracle.conv_event(oracle.dense_to_lat(S), T, Ws[li], (L["stride"],) * 2, (L["pad"],) * 2)
        if L["theta"] is None:
            L["theta"] = pipeline.sig3(float(np.percentile(P[:, T - 1], 80)))
            print(f"{name} layer {li}: theta = {L['theta']}")
        S = oracle.pool(oracle.fire(P, L["theta"]), (L["pool"]["kernel"],) * 2,
                        (L["pool"]["stride"],) * 2, (L["pool"]["pad"],) * 2) if L["pool"] else oracle.fire(P, L["theta"])
    path = synth.CONFIG_DIR / f"{name.lower()}.json"
    raw = json.loads(path.read_text())
    for li, L in enumerate(cfg["layers"]):
        raw["layers"][li]["theta"] = L["theta"]
    path.write_text(json.dumps(raw, indent=2) + "\n")
    return cfg


if __name__ == "__main__":
    for n in sys.argv[1:] or ["c2", "c3"]:
        calibrate(n)
