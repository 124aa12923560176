"""Freeze the FC workload's IF threshold (configs/fc.json) — oracle only (reading R-THETA-CAL):
the 80th percentile of the final-step FC potentials over rows 0..15, 3 significant figures."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle  # noqa: E402
from oracle import pipeline  # noqa: E402
import synth  # noqa: E402

cfg = synth.load_config("fc")
lat = synth.latencies(cfg, 0, 16, cfg["I"], cfg["T"], cfg["p_fire"])
P = oracle.fc(oracle.lat_to_dense(lat, cfg["T"]), synth.fc_weights(cfg))
path = synth.CONFIG_DIR / "fc.json"
raw = json.loads(path.read_text())
raw["theta"] = pipeline.sig3(float(np.percentile(P[:, -1], 80)))
path.write_text(json.dumps(raw, indent=2) + "\n")
print("fc theta", raw["theta"])
