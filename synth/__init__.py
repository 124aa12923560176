"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds no arithmetic of the method: it only draws images, labels
and initial weights (the random numbers the method is given as inputs,
P:L127 "synaptic weights are initialized randomly with a normal
distribution").  Every array is a function of (seed, global index) only, so a
shard of a batch generated on any rank is bit-identical to the same rows of
the whole batch.
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

CONFIG_DIR = Path(__file__).resolve().parent.parent / "configs"


def load_config(name: str) -> dict:
    """configs/<name>.json — every constant of one workload (C1..C5)."""
    return json.loads((CONFIG_DIR / f"{name.lower()}.json").read_text())


def _rng(seed: int, *key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), *map(int, key)])))


# ----------------------------------------------------------------- images
def _seg_dist(yy, xx, y0, x0, y1, x1):
    dy, dx = y1 - y0, x1 - x0
    L2 = dy * dy + dx * dx + 1e-12
    u = np.clip(((yy - y0) * dy + (xx - x0) * dx) / L2, 0.0, 1.0)
    return np.hypot(yy - (y0 + u * dy), xx - (x0 + u * dx))


def mnist_like(seed: int, index: int, H: int = 28, W: int = 28) -> np.ndarray:
    """One 28x28 u8 digit-like image: black background, 4-7 anti-aliased strokes
    (width 2-3 px) forming a connected glyph in the central 20x20 box, the way
    MNIST digits are centred.  Returns [1][H][W] u8."""
    g = _rng(seed, 0x4D4E, index)
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    ink = np.zeros((H, W))
    n = int(g.integers(4, 8))  # strokes
    py, px = g.uniform(6, H - 6), g.uniform(6, W - 6)
    for _ in range(n):
        qy = float(np.clip(py + g.normal(0, 7), 4, H - 5))
        qx = float(np.clip(px + g.normal(0, 6), 4, W - 5))
        w = g.uniform(1.2, 1.8)  # half width -> 2-3 px strokes (+AA rim)
        d = _seg_dist(yy, xx, py, px, qy, qx)
        ink = np.maximum(ink, np.clip(w + 0.5 - d, 0.0, 1.0))
        py, px = qy, qx
    return np.round(ink * 255.0).astype(np.uint8)[None]


def caltech_like(seed: int, index: int, H: int = 160, W: int = 250) -> np.ndarray:
    """Full-frame grey scene: a random gradient plus 20-40 filled ellipses and
    rectangles of random grey levels, plus Gaussian noise sigma=4.  [1][H][W] u8."""
    g = _rng(seed, 0xCA17, index)
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float32)
    a, b, c = g.uniform(-0.4, 0.4), g.uniform(-0.4, 0.4), g.uniform(60, 190)
    img = c + a * (yy - H / 2) + b * (xx - W / 2)
    for _ in range(int(g.integers(20, 41))):
        cy, cx = g.uniform(0, H), g.uniform(0, W)
        ry, rx = g.uniform(4, H / 4), g.uniform(4, W / 4)
        lvl = g.uniform(0, 255)
        if g.random() < 0.5:
            m = ((yy - cy) / ry) ** 2 + ((xx - cx) / rx) ** 2 <= 1.0
        else:
            m = (np.abs(yy - cy) <= ry) & (np.abs(xx - cx) <= rx)
        img = np.where(m, lvl, img)
    img = img + g.normal(0, 4.0, size=img.shape)
    return np.clip(np.round(img), 0, 255).astype(np.uint8)[None]


def imagenet_like(seed: int, index: int, H: int = 224, W: int = 224) -> np.ndarray:
    """Full-frame colour scene: shared luminance (gradient + 15-30 shapes) with a
    small per-channel chroma offset per shape, plus noise.  [3][H][W] u8."""
    g = _rng(seed, 0x1A6E, index)
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float32)
    base = g.uniform(60, 190) + g.uniform(-0.3, 0.3) * (yy - H / 2) + g.uniform(-0.3, 0.3) * (xx - W / 2)
    img = np.stack([base, base, base])
    for _ in range(int(g.integers(15, 31))):
        cy, cx = g.uniform(0, H), g.uniform(0, W)
        ry, rx = g.uniform(6, H / 4), g.uniform(6, W / 4)
        m = ((yy - cy) / ry) ** 2 + ((xx - cx) / rx) ** 2 <= 1.0
        lvl = g.uniform(0, 255) + g.uniform(-25, 25, size=3)
        for ch in range(3):
            img[ch] = np.where(m, lvl[ch], img[ch])
    img = img + g.normal(0, 4.0, size=img.shape)
    return np.clip(np.round(img), 0, 255).astype(np.uint8)


_KINDS = {"mnist": mnist_like, "caltech": caltech_like, "imagenet": imagenet_like}


def images(cfg: dict, start: int, count: int) -> np.ndarray:
    """Global images [start, start+count) of config `cfg` -> u8 [count][C][H][W]."""
    im = cfg["image"]
    fn = _KINDS[im["kind"]]
    out = np.empty((count, im["C"], im["H"], im["W"]), np.uint8)
    for q in range(count):
        out[q] = fn(cfg["seed"], start + q, im["H"], im["W"])
    return out


def _images_chunk(args):
    cfg, start, count = args
    return images(cfg, start, count)


def images_parallel(cfg: dict, start: int, count: int, workers: int | None = None) -> np.ndarray:
    """images() spread over host processes (bit-identical: each image depends only on its index)."""
    import os
    from concurrent.futures import ProcessPoolExecutor

    workers = workers or min(16, os.cpu_count() or 1)
    if count < 64 or workers <= 1:
        return images(cfg, start, count)
    step = (count + workers - 1) // workers
    jobs = [(cfg, start + q, min(step, count - q)) for q in range(0, count, step)]
    with ProcessPoolExecutor(workers) as ex:
        return np.concatenate(list(ex.map(_images_chunk, jobs)))


def labels(cfg: dict, start: int, count: int, classes: int = 10) -> np.ndarray:
    """Labels uniform over 0..classes-1, one draw per global index (C3)."""
    return np.array([int(_rng(cfg["seed"], 0x1AB, start + q).integers(0, classes)) for q in range(count)],
                    np.int32)


# ----------------------------------------------------------------- weights
def weights(cfg: dict, layer: int, shape, mean: float, std: float, lower: float = 0.0,
            upper: float = 1.0, fp16: bool = False) -> np.ndarray:
    """N(mean, std) initial kernel [Co][Ci][Kh][Kw] fp32, clipped to
    [lower, upper] (reading R-INIT-CLIP); optionally rounded to fp16-representable
    values (reading R-FP16-WEIGHTS, C5)."""
    g = _rng(cfg["seed"], 0x3E16, layer)
    w = g.normal(mean, std, size=shape)
    w = np.clip(w, lower, upper).astype(np.float32)
    if fp16:
        w = w.astype(np.float16).astype(np.float32)
    return np.ascontiguousarray(w)


def layer_weights(cfg: dict) -> list[np.ndarray]:
    """Initial weights of every conv layer of config `cfg`."""
    out = []
    ci = cfg["image"]["C"] * cfg["front"]["n_kernels"]
    for li, L in enumerate(cfg["layers"]):
        init = L["init"]
        out.append(weights(cfg, li, (L["Co"], ci, L["K"], L["K"]), init["mean"], init["std"],
                           init.get("lower", 0.0), init.get("upper", 1.0), init.get("fp16", False)))
        ci = L["Co"]
    return out


def latencies(cfg: dict, start: int, count: int, n: int, T: int, p_fire: float) -> np.ndarray:
    """Synthetic first-spike latency maps u8 [count][n] (an input to the FC workload): each input
    fires with probability p_fire at a uniform step 0..T-1, else never (T).  One draw per global row."""
    out = np.empty((count, n), np.uint8)
    for q in range(count):
        g = _rng(cfg["seed"], 0x1A7, start + q)
        lat = g.integers(0, T, n)
        lat[g.random(n) >= p_fire] = T
        out[q] = lat.astype(np.uint8)
    return out


def fc_weights(cfg: dict) -> np.ndarray:
    """FC kernel in the paper's I x O layout, N(mean, std) clipped to [0, 1]."""
    g = _rng(cfg["seed"], 0xFC, 0)
    w = np.clip(g.normal(cfg["init"]["mean"], cfg["init"]["std"], (cfg["I"], cfg["O"])), 0.0, 1.0)
    return np.ascontiguousarray(w.astype(np.float32))
