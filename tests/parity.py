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


# ---------------------------------------------------------------------------------------
# Parity report (SURVEY §8(c) protocol items 2 and 5; north_star "such cases are counted and
# reported"): every GPU parity test that compares a stage adds its counts here, and the session
# writes them to $SPK_PARITY_REPORT (default profiles/parity_report.json) — see conftest.py.
# ---------------------------------------------------------------------------------------
class ParityReport:
    entries: dict = {}
    _errs: dict = {}
    CAP = 4_000_000  # relative errors kept per entry for the percentile (uniform subsample)

    @classmethod
    def _e(cls, key):
        return cls.entries.setdefault(key, dict(neurons=0, near_threshold=0, mismatch_in_near_threshold=0,
                                                mismatch_outside=0, near_ties=0, tie_decisions=0,
                                                samples_excluded=0, potentials=0, max_abs_err=0.0,
                                                max_rel_err=0.0, p9999_rel_err=None))

    @classmethod
    def latency(cls, key, gpu_lat, ref_lat, excluded):
        e = cls._e(key)
        diff = gpu_lat != ref_lat
        e["neurons"] += int(diff.size)
        e["near_threshold"] += int(excluded.sum()) if excluded is not None else 0
        if excluded is not None:
            e["mismatch_in_near_threshold"] += int((diff & excluded).sum())
            e["mismatch_outside"] += int((diff & ~excluded).sum())
        else:
            e["mismatch_outside"] += int(diff.sum())

    @classmethod
    def potentials(cls, key, gpu, ref):
        e = cls._e(key)
        ref = np.asarray(ref, np.float64).ravel()
        err = np.abs(np.asarray(gpu, np.float64).ravel() - ref)
        if err.size == 0:
            return
        e["potentials"] += int(err.size)
        e["max_abs_err"] = max(e["max_abs_err"], float(err.max()))
        # relative errors over potentials of at least 1e-3 (a weight sum; smaller ones are
        # covered by the absolute term ATOL of the protocol)
        big = np.abs(ref) >= 1e-3
        rel = err[big] / np.abs(ref[big])
        if rel.size == 0:
            return
        e["max_rel_err"] = max(e["max_rel_err"], float(rel.max()))
        if rel.size > cls.CAP:
            rel = np.random.default_rng(0).choice(rel, cls.CAP, replace=False)
        errs = cls._errs.setdefault(key, [])
        errs.append(rel)
        allr = np.concatenate(errs)
        e["p9999_rel_err"] = float(np.quantile(allr, 0.9999))
        if allr.size > cls.CAP:
            cls._errs[key] = [np.random.default_rng(1).choice(allr, cls.CAP, replace=False)]

    @classmethod
    def ties(cls, key, n_near, n_decisions):
        e = cls._e(key)
        e["near_ties"] += int(n_near)
        e["tie_decisions"] += int(n_decisions)

    @classmethod
    def excluded_samples(cls, key, n):
        cls._e(key)["samples_excluded"] += int(n)

    @classmethod
    def dump(cls, path):
        import json
        import time
        if not cls.entries:
            return None
        out = {"protocol": {"REL_THR": REL_THR, "RTOL": RTOL, "ATOL": ATOL, "TIE_REL": TIE_REL,
                            "note": "near_threshold = neurons whose oracle potential lies within REL_THR*theta of "
                                    "theta at some step (spike-time mismatches there are counted, not failed); "
                                    "near_ties = inhibition/WTA decisions whose two best P* (same step) lie within "
                                    "TIE_REL relative; mismatch_outside must be 0 (the tests assert it)"},
               "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
               "entries": {" / ".join(k) if isinstance(k, tuple) else k: v for k, v in sorted(cls.entries.items())}}
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
        return path


def _keys(Q: np.ndarray):
    """Oracle thresholded potentials [T][C][H][W] of one sample -> (lat, P*) per neuron."""
    T = Q.shape[0]
    fired = Q > 0
    anyf = fired.any(0)
    lat = np.where(anyf, fired.argmax(0), T)
    ps = np.take_along_axis(Q, np.minimum(lat, T - 1)[None], 0)[0]
    return lat, np.where(anyf, ps, 0.0)


def near_ties_inhibit(Q: np.ndarray):
    """Inhibition decisions (locations with >= 2 firing channels) whose winner's P* is within
    TIE_REL of another channel firing at the same step -> (near ties, decisions)."""
    near = dec = 0
    for b in range(Q.shape[0]):
        lat, ps = _keys(Q[b])
        T = Q.shape[1]
        nf = (lat < T).sum(0)
        m = lat.min(0)
        for y, x in zip(*np.nonzero(nf >= 2)):
            dec += 1
            cand = np.sort(ps[lat[:, y, x] == m[y, x], y, x])[::-1]
            if cand.size >= 2 and abs(cand[0] - cand[1]) <= TIE_REL * abs(cand[0]):
                near += 1
    return near, dec


def near_ties_wta(Qi: np.ndarray, count: int, radius: int):
    """k-WTA picks (R-WTA-FOOTPRINT scan, written independently of the oracle) whose P* lies
    within TIE_REL of another live neuron of the same step -> (near ties, picks)."""
    near = picks = 0
    B, T, C, H, W = Qi.shape
    for b in range(B):
        lat, ps = _keys(Qi[b])
        live = lat < T
        for _ in range(count):
            if not live.any():
                break
            m = lat[live].min()
            cand = live & (lat == m)
            best = ps[cand].max()
            picks += 1
            if (np.abs(ps[cand] - best) <= TIE_REL * abs(best)).sum() >= 2:
                near += 1
            # the oracle's pick (lowest flat index among the max-P* neurons of step m)
            idx = np.flatnonzero((cand & (ps == best)).ravel())[0]
            c, y, x = idx // (H * W), (idx // W) % H, idx % W
            live[c] = False
            live[:, max(0, y - radius):y + radius + 1, max(0, x - radius):x + radius + 1] = False
    return near, picks
