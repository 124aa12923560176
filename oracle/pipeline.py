"""Oracle network steps — TEST INFRASTRUCTURE ONLY.

Composes the oracle's per-op definitions in exactly the order of the paper's
listings on dense BTCHW arrays:

* front end — Listing 1: filter -> threshold(0.01) -> code(T);
* inference — Listing 5: conv -> fire(theta) -> pool ... -> gather;
* training of layer L — Listing 3: forward to layer L's input,
  conv_L -> threshold(theta_L) -> inhibit -> convwta -> fire -> conv_L.stdp;
* R-STDP: winners routed to reward/punish configs by label.
"""
from __future__ import annotations

import numpy as np

from . import (conv, conv_event, dog_bank, filter_apply, fire, gabor_bank, gather, inhibit,
               lat_to_dense, log_kernels, pool, rank_code, rstdp_route, stdp, threshold, wta)


def filter_bank(cfg: dict) -> np.ndarray:
    fr = cfg["front"]
    r = fr["radius"]
    if fr["kind"] == "dog":
        return dog_bank(fr["pairs"], r)
    if fr["kind"] == "log":
        return log_kernels(fr["stds"], r)
    if fr["kind"] == "gabor":
        return gabor_bank(fr["params"], r)
    raise ValueError(fr["kind"])


def front_end(cfg: dict, imgs: np.ndarray):
    """Listing 1: -> (filter response fp32 [B][C][H][W], latency u8 [B][C][H][W])."""
    fr = cfg["front"]
    y = filter_apply(imgs, filter_bank(cfg), fr["pad"])
    lat = rank_code(y, cfg["T"], fr["thresh"], fr["sort"])
    return y, lat


def _conv(S, W, L, event: bool, T: int):
    st, pd = (L["stride"],) * 2, (L["pad"],) * 2
    if event:
        from . import dense_to_lat
        return conv_event(dense_to_lat(S), T, W, st, pd)
    return conv(S, W, st, pd)


def _pool(S, L):
    p = L["pool"]
    if not p:
        return S
    return pool(S, (p["kernel"],) * 2, (p["stride"],) * 2, (p["pad"],) * 2)


def forward(cfg: dict, imgs: np.ndarray, weights, upto: int | None = None, event: bool = False):
    """Dense input trains of every layer up to `upto` (exclusive end = input of layer upto).

    Returns (y, lat0, inputs) where inputs[l] is the dense BTCHW train fed to layer l;
    if upto is None the list also holds the output train of the last layer (pooled)."""
    T = cfg["T"]
    weights = quantized_weights(cfg, weights)
    y, lat0 = front_end(cfg, imgs)
    S = lat_to_dense(lat0, T)
    inputs = [S]
    n = len(cfg["layers"]) if upto is None else upto
    for li in range(n):
        L = cfg["layers"][li]
        P = _conv(S, weights[li], L, event, T)
        S = _pool(fire(P, L["theta"]), L)
        inputs.append(S)
    return y, lat0, inputs


def train_step(cfg: dict, imgs: np.ndarray, weights, labels=None, event: bool = False):
    """One training step of layer cfg['train_layer'] (Listing 3; R-STDP for cfg['learning']=='rstdp').

    Returns a dict with every intermediate the GPU path is compared against."""
    li = cfg["train_layer"]
    L = cfg["layers"][li]
    T = cfg["T"]
    weights = quantized_weights(cfg, weights)  # Listing 4: layers quantized after their training
    y, lat0, inputs = forward(cfg, imgs, weights, upto=li, event=event)
    S_in = inputs[li]
    P = _conv(S_in, weights[li], L, event, T)
    Q = threshold(P, L["theta"])
    Qi = inhibit(Q)
    win, nwin = wta(Qi, L["wta"]["count"], L["wta"]["radius"])
    if cfg["learning"] == "rstdp":
        win = rstdp_route(win, nwin, labels, cfg["maps_per_class"])
    cfgs = [tuple(c) for c in cfg["stdp"]]
    W_new = stdp(weights[li], S_in, win, nwin, cfgs, (L["stride"],) * 2, (L["pad"],) * 2)
    return dict(y=y, lat0=lat0, inputs=inputs, S_in=S_in, P=P, Q=Q, Qi=Qi, win=win, nwin=nwin,
                W_new=W_new, spikes=fire(Qi, 0.0))


def infer(cfg: dict, imgs: np.ndarray, weights, event: bool = False):
    """Listing 5: forward through every layer then gather -> features [B][C][H][W]."""
    _, _, inputs = forward(cfg, imgs, weights, event=event)
    return gather(inputs[-1])


def sig3(x: float) -> float:
    """Round to 3 significant figures (calibrated thresholds, reading R-THETA-CAL)."""
    return float(f"{x:.3g}") if x > 0 else 0.0


# ------------------------------------------------------------------ NEXT-3 rate-coded inference
def quantized_weights(cfg: dict, weights):
    """Listing 4: layers with a "quantize" entry (lower, mid, upper) use
    quantize(kernel, lower, mid, upper) of their weights."""
    from . import quantize

    out = []
    for L, W in zip(cfg["layers"], weights):
        q = L.get("quantize")
        out.append(quantize(W, *q) if q else W)
    return out


def rate_front_end(cfg: dict, imgs: np.ndarray, start: int = 0):
    """Listing 1 with rate coding: filter -> threshold -> rate code.
    Returns the dense non-cumulative train [B][T][C][H][W].  `start` = global index of imgs[0]
    (the generator's counter runs over the global sample index)."""
    from . import rate_code

    fr = cfg["front"]
    y = threshold(filter_apply(imgs, filter_bank(cfg), fr["pad"]), fr["thresh"])
    return rate_code(y, cfg["T"], cfg["rate_seed"], start)


def rate_infer(cfg: dict, imgs: np.ndarray, weights, start: int = 0):
    """Rate-coded inference: per layer conv (per step, Eq. 2) -> fire (per step,
    P:L125) -> pool by rates or per-step max; features = firing rates.
    Returns dict(S0, steps=[layer output trains], pooled=[...], rates=[...], features)."""
    from . import gather, pool_rates

    T = cfg["T"]
    Ws = quantized_weights(cfg, weights)
    S = rate_front_end(cfg, imgs, start)
    out = dict(S0=S, steps=[], pooled=[], rates=[])
    for li, L in enumerate(cfg["layers"]):
        P = _conv(S, Ws[li], L, False, T)
        Sl = fire(P, L["theta"])
        del P
        out["steps"].append(Sl)
        p = L["pool"]
        if p:
            r = gather(Sl)
            out["rates"].append(r)
            if L.get("pool_rates"):
                Sl = pool_rates(Sl, r, (p["kernel"],) * 2, (p["stride"],) * 2, (p["pad"],) * 2)
            else:
                Sl = pool(Sl, (p["kernel"],) * 2, (p["stride"],) * 2, (p["pad"],) * 2)
        out["pooled"].append(Sl)
        S = Sl
    out["features"] = gather(S)
    return out
