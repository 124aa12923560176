"""Comparison rules of the parity protocol, shared by the GPU tests.

* spike times / latencies / winners / indices: bit-exact, except neurons whose
  oracle potential lies within REL_THR * theta of the threshold at some step
  (counted and reported: float rounding may legitimately decide them either way);
* potentials: |gpu - oracle| <= RTOL * |oracle| + ATOL;
* weights after STDP: bit-exact.
"""
import numpy as np

REL_THR = 1e-4   # north_star: "except where a potential lies within 1e-4 relative of threshold"
RTOL = 1e-5      # north_star: "fp32 potentials within 1e-5"
ATOL = 1e-6
TIE_REL = 1e-5   # WTA / inhibition near-ties in P*


def near_threshold(P: np.ndarray, theta: float) -> np.ndarray:
    """[B][T][C][H][W] oracle potentials -> [B][C][H][W] neurons with any step within REL_THR*theta."""
    return (np.abs(P - theta) <= REL_THR * max(abs(theta), 1e-30)).any(axis=1)


def assert_potentials(gpu: np.ndarray, ref: np.ndarray, rtol=RTOL, atol=ATOL):
    err = np.abs(gpu.astype(np.float64) - ref)
    tol = rtol * np.abs(ref) + atol
    bad = err > tol
    assert not bad.any(), (f"{bad.sum()} potentials out of tolerance; max rel err "
                           f"{(err / np.maximum(np.abs(ref), 1e-30)).max():.3e}")
    return float((err / np.maximum(np.abs(ref), 1e-12)).max())


def compare_latency(gpu_lat: np.ndarray, ref_lat: np.ndarray, excluded: np.ndarray | None = None):
    """Exact equality outside the excluded set; returns (#mismatch inside excluded, #excluded)."""
    diff = gpu_lat != ref_lat
    if excluded is None:
        assert not diff.any(), f"{diff.sum()} latency mismatches (no exclusions allowed)"
        return 0, 0
    unexplained = diff & ~excluded
    assert not unexplained.any(), (f"{unexplained.sum()} latency mismatches outside the near-threshold set "
                                   f"(first at {np.argwhere(unexplained)[:3].tolist()})")
    return int((diff & excluded).sum()), int(excluded.sum())


def lat_and_pstar(P: np.ndarray, theta: float):
    """Oracle (double) potentials -> first crossing latency and potential at it."""
    fired = P > theta
    T = P.shape[1]
    any_ = fired.any(axis=1)
    lat = np.where(any_, fired.argmax(axis=1), T).astype(np.uint8)
    ps = np.take_along_axis(P, np.minimum(lat, T - 1)[:, None].astype(np.int64), axis=1)[:, 0]
    ps = np.where(any_, ps, 0.0)
    return lat, ps
