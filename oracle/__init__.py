"""CPU oracle for the Spyker SDNN hot path — TEST INFRASTRUCTURE ONLY.

Plain, slow, single-threaded definitions from the paper (arXiv 2301.13659,
/root/reference/PAPER.md, cited P:Lnn), implemented in ``oracle.c`` on dense
BTCHW arrays and wrapped here with ctypes + numpy.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (``cpu_baseline`` leg and
``--impl reference``) may import this package.  It shares no code with the CUDA
path (``paper_2301_13659_b200``); inputs come from ``synth``.

Every wrapper names the oracle.c function (and so the passage) it calls.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_DIR = Path(__file__).resolve().parent
_SRC = _DIR / "oracle.c"
_LIB = _DIR / "liboracle.so"
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-shared", "-fPIC"]


def build(force: bool = False) -> Path:
    """Compile oracle.c with gcc (no FMA contraction, no fast-math)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".so.{os.getpid()}")
        subprocess.check_call(["gcc", *CFLAGS, str(_SRC), "-o", str(tmp), "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(str(build()))
        _declare(_lib)
    return _lib


P = ctypes.c_void_p
I = ctypes.c_int
D = ctypes.c_double
F = ctypes.c_float
SZ = ctypes.c_size_t


def _declare(L):
    sig = {
        "oracle_dog_kernel": [D, D, I, P],
        "oracle_gabor_kernel": [D, D, D, D, D, I, P],
        "oracle_log_kernels": [P, I, I, P],
        "oracle_filter": [P, I, I, I, I, P, I, I, I, P],
        "oracle_threshold_f32": [P, SZ, F],
        "oracle_threshold_f64": [P, SZ, D],
        "oracle_rank_code": [P, I, I, I, F, I, P],
        "oracle_lat_to_dense": [P, I, I, SZ, P],
        "oracle_dense_to_lat": [P, I, I, SZ, P],
        "oracle_conv": [P, I, I, I, I, I, P, I, I, I, I, I, I, I, P],
        "oracle_conv_event": [P, I, I, I, I, I, P, I, I, I, I, I, I, I, P],
        "oracle_fire": [P, SZ, D, P],
        "oracle_pool": [P, I, I, I, I, I, I, I, I, I, I, I, P],
        "oracle_inhibit": [P, I, I, I, I, I],
        "oracle_wta": [P, I, I, I, I, I, I, I, P, P],
        "oracle_stdp": [P, I, I, I, I, I, I, I, I, P, I, I, I, I, P, P, I, P, P, I],
        "oracle_rstdp_route": [P, P, I, I, P, I],
        "oracle_gather": [P, I, I, SZ, P],
        "oracle_rate_code": [P, I, I, I, ctypes.c_uint64, ctypes.c_uint64, P],
        "oracle_pool_rates": [P, P, I, I, I, I, I, I, I, I, I, I, I, P],
        "oracle_quantize": [P, SZ, F, F, F],
        "oracle_fc": [P, I, I, I, P, I, P],
        "oracle_fc_stdp": [P, I, I, P, I, I, P, P, I, P, P, I],
        "oracle_fcwta": [P, I, I, I, I, I, P, P],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = None
    L.oracle_splitmix64.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    L.oracle_splitmix64.restype = ctypes.c_uint64


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------- filters (O2)
def dog_kernel(sigma1: float, sigma2: float, r: int) -> np.ndarray:
    """DoG = unit-sum G(sigma1) - G(sigma2) on [-r, r]^2."""
    out = np.empty((2 * r + 1, 2 * r + 1), np.float32)
    lib().oracle_dog_kernel(sigma1, sigma2, r, _p(out))
    return out


def gabor_kernel(sigma, theta, gamma, lam, psi, r: int) -> np.ndarray:
    """Standard unnormalised Gabor."""
    out = np.empty((2 * r + 1, 2 * r + 1), np.float32)
    lib().oracle_gabor_kernel(sigma, theta, gamma, lam, psi, r, _p(out))
    return out


def log_kernels(stds, r: int) -> np.ndarray:
    """LoG(s) -> [DoG(s*sqrt2, s/sqrt2), DoG(s/sqrt2, s*sqrt2)] per std."""
    s = _c(stds, np.float64)
    out = np.empty((2 * len(s), 2 * r + 1, 2 * r + 1), np.float32)
    lib().oracle_log_kernels(_p(s), len(s), r, _p(out))
    return out


def dog_bank(pairs, r: int) -> np.ndarray:
    return np.stack([dog_kernel(a, b, r) for a, b in pairs]).astype(np.float32)


def gabor_bank(params, r: int) -> np.ndarray:
    return np.stack([gabor_kernel(*p, r) for p in params]).astype(np.float32)


def filter_apply(img: np.ndarray, kern: np.ndarray, pad: int) -> np.ndarray:
    """Depthwise filter bank on u8 images [B][C][H][W] -> fp32 [B][C*K][Ho][Wo] (Eq. 1)."""
    img = _c(img, np.uint8)
    kern = _c(kern, np.float32)
    B, C, H, W = img.shape
    K, e, _ = kern.shape
    r = (e - 1) // 2
    Ho, Wo = H + 2 * pad - e + 1, W + 2 * pad - e + 1
    out = np.empty((B, C * K, Ho, Wo), np.float32)
    lib().oracle_filter(_p(img), B, C, H, W, _p(kern), K, r, pad, _p(out))
    return out


# ----------------------------------------------------------------- coding (O4, O5)
def threshold(x: np.ndarray, theta: float) -> np.ndarray:
    """x if x > theta else 0."""
    x = np.array(x, copy=True, order="C")
    if x.dtype == np.float32:
        lib().oracle_threshold_f32(_p(x), x.size, theta)
    else:
        x = x.astype(np.float64)
        lib().oracle_threshold_f64(_p(x), x.size, theta)
    return x


def rank_code(y: np.ndarray, T: int, thresh: float, sort: bool = True) -> np.ndarray:
    """Threshold + rank-order code each sample -> u8 first-spike latency, T = never."""
    y = _c(y, np.float32)
    B = y.shape[0]
    N = int(np.prod(y.shape[1:]))
    lat = np.empty(y.shape, np.uint8)
    lib().oracle_rank_code(_p(y), B, N, T, thresh, int(bool(sort)), _p(lat))
    return lat


def lat_to_dense(lat: np.ndarray, T: int) -> np.ndarray:
    """[B][...] latencies -> cumulative dense train [B][T][...]."""
    lat = _c(lat, np.uint8)
    B = lat.shape[0]
    N = int(np.prod(lat.shape[1:]))
    S = np.empty((B, T) + lat.shape[1:], np.uint8)
    lib().oracle_lat_to_dense(_p(lat), B, T, N, _p(S))
    return S


def dense_to_lat(S: np.ndarray) -> np.ndarray:
    S = _c(S, np.uint8)
    B, T = S.shape[:2]
    N = int(np.prod(S.shape[2:]))
    lat = np.empty((B,) + S.shape[2:], np.uint8)
    lib().oracle_dense_to_lat(_p(S), B, T, N, _p(lat))
    return lat


# ------------------------------------------------------------------- conv (O6)
def conv_out_hw(Hi, Wi, Kh, Kw, Sh, Sw, Ph, Pw):
    return (Hi + 2 * Ph - Kh) // Sh + 1, (Wi + 2 * Pw - Kw) // Sw + 1


def conv(S: np.ndarray, W: np.ndarray, stride=(1, 1), pad=(0, 0)) -> np.ndarray:
    """Direct Eq. 2 on a dense BTCHW train -> fp64 potentials BTCHW."""
    S = _c(S, np.uint8)
    W = _c(W, np.float32)
    B, T, Ci, Hi, Wi = S.shape
    Co, Ci2, Kh, Kw = W.shape
    assert Ci == Ci2
    Ho, Wo = conv_out_hw(Hi, Wi, Kh, Kw, *stride, *pad)
    P = np.empty((B, T, Co, Ho, Wo), np.float64)
    lib().oracle_conv(_p(S), B, T, Ci, Hi, Wi, _p(W), Co, Kh, Kw, *stride, *pad, _p(P))
    return P


def conv_event(lat: np.ndarray, T: int, W: np.ndarray, stride=(1, 1), pad=(0, 0)) -> np.ndarray:
    """Event form of Eq. 2 from a latency map [B][Ci][Hi][Wi] -> fp64 BTCHW potentials."""
    lat = _c(lat, np.uint8)
    W = _c(W, np.float32)
    B, Ci, Hi, Wi = lat.shape
    Co, _, Kh, Kw = W.shape
    Ho, Wo = conv_out_hw(Hi, Wi, Kh, Kw, *stride, *pad)
    P = np.empty((B, T, Co, Ho, Wo), np.float64)
    lib().oracle_conv_event(_p(lat), B, T, Ci, Hi, Wi, _p(W), Co, Kh, Kw, *stride, *pad, _p(P))
    return P


# ---------------------------------------------------------- fire / pool (O7, O8)
def fire(P: np.ndarray, theta: float) -> np.ndarray:
    P = _c(P, np.float64)
    S = np.empty(P.shape, np.uint8)
    lib().oracle_fire(_p(P), P.size, theta, _p(S))
    return S


def pool(S: np.ndarray, kernel, stride=None, pad=(0, 0)) -> np.ndarray:
    S = _c(S, np.uint8)
    B, T, C, H, W = S.shape
    Lh, Lw = kernel
    Sh, Sw = stride if stride is not None else kernel
    Ph, Pw = pad
    Ho, Wo = (H + 2 * Ph - Lh) // Sh + 1, (W + 2 * Pw - Lw) // Sw + 1
    out = np.empty((B, T, C, Ho, Wo), np.uint8)
    lib().oracle_pool(_p(S), B, T, C, H, W, Lh, Lw, Sh, Sw, Ph, Pw, _p(out))
    return out


# ------------------------------------------------------ inhibit / wta (O9, O10)
def inhibit(Q: np.ndarray) -> np.ndarray:
    Q = np.array(Q, dtype=np.float64, order="C", copy=True)
    B, T, C, H, W = Q.shape
    lib().oracle_inhibit(_p(Q), B, T, C, H, W)
    return Q


def wta(Q: np.ndarray, count: int, radius: int):
    """-> (win int32 [B][count][6] = {b, t, c, y, x, cfg}, nwin int32 [B])."""
    Q = _c(Q, np.float64)
    B, T, C, H, W = Q.shape
    win = np.full((B, count, 6), -1, np.int32)
    nwin = np.zeros(B, np.int32)
    lib().oracle_wta(_p(Q), B, T, C, H, W, count, radius, _p(win), _p(nwin))
    return win, nwin


# ------------------------------------------------------- stdp / rstdp (O11, O12)
def stdp(W: np.ndarray, S_in: np.ndarray, win, nwin, cfgs, stride=(1, 1), pad=(0, 0)) -> np.ndarray:
    """cfgs: list of (A+, A-, L, U, stabilize).  Returns updated copy of W (fp32)."""
    W = np.array(W, dtype=np.float32, order="C", copy=True)
    S_in = _c(S_in, np.uint8)
    win = _c(win, np.int32)
    nwin = _c(nwin, np.int32)
    Co, Ci, Kh, Kw = W.shape
    B, T, Ci2, Hi, Wi = S_in.shape
    assert Ci2 == Ci
    assert win.shape[0] == B and nwin.shape[0] == B and win.shape[2] == 6, "winners must cover every sample"
    cfg = _c([[c[0], c[1], c[2], c[3]] for c in cfgs], np.float32)
    stab = _c([int(bool(c[4])) for c in cfgs], np.int32)
    lib().oracle_stdp(_p(W), Co, Ci, Kh, Kw, *stride, *pad, _p(S_in), B, T, Hi, Wi, _p(win),
                      _p(nwin), win.shape[1], _p(cfg), _p(stab), len(cfgs))
    return W


def rstdp_route(win, nwin, labels, maps_per_class: int):
    win = np.array(win, dtype=np.int32, order="C", copy=True)
    nwin = _c(nwin, np.int32)
    labels = _c(labels, np.int32)
    lib().oracle_rstdp_route(_p(win), _p(nwin), win.shape[0], win.shape[1], _p(labels), maps_per_class)
    return win


# ----------------------------------------------------------------- gather (O13)
def gather(S: np.ndarray) -> np.ndarray:
    S = _c(S, np.uint8)
    B, T = S.shape[:2]
    N = int(np.prod(S.shape[2:]))
    f = np.empty((B,) + S.shape[2:], np.float32)
    lib().oracle_gather(_p(S), B, T, N, _p(f))
    return f


# ------------------------------------------------- NEXT-3: rate coding (O14-O16)
def splitmix64(seed: int, counter: int) -> int:
    """Value `counter` of the counter-based stream `seed` (O14)."""
    return int(lib().oracle_splitmix64(seed, counter))


def rate_code(y: np.ndarray, T: int, seed: int, b0: int = 0) -> np.ndarray:
    """Per-step Bernoulli(v / vmax) spikes of thresholded responses [B][...] -> dense
    non-cumulative train [B][T][...]; b0 = global index of row 0."""
    y = _c(y, np.float32)
    B = y.shape[0]
    N = int(np.prod(y.shape[1:]))
    S = np.empty((B, T) + y.shape[1:], np.uint8)
    lib().oracle_rate_code(_p(y), B, N, T, seed, b0, _p(S))
    return S


def pool_rates(S: np.ndarray, rates: np.ndarray, kernel, stride=None, pad=(0, 0)) -> np.ndarray:
    """Rate-based max pooling: the window's highest-rate cell's whole train."""
    S = _c(S, np.uint8)
    rates = _c(rates, np.float32)
    B, T, C, H, W = S.shape
    assert rates.shape == (B, C, H, W)
    Lh, Lw = kernel
    Sh, Sw = stride if stride is not None else kernel
    Ph, Pw = pad
    Ho, Wo = (H + 2 * Ph - Lh) // Sh + 1, (W + 2 * Pw - Lw) // Sw + 1
    out = np.empty((B, T, C, Ho, Wo), np.uint8)
    lib().oracle_pool_rates(_p(S), _p(rates), B, T, C, H, W, Lh, Lw, Sh, Sw, Ph, Pw, _p(out))
    return out


# ------------------------------------------- NEXT-4: quantize, FC, fcwta (O17-O19)
def quantize(w: np.ndarray, lower: float, mid: float, upper: float) -> np.ndarray:
    """Listing 4 quantize(kernel, lower, mid, upper) on a copy."""
    w = np.array(w, dtype=np.float32, order="C", copy=True)
    lib().oracle_quantize(_p(w), w.size, lower, mid, upper)
    return w


def fc(S: np.ndarray, W: np.ndarray) -> np.ndarray:
    """Fully connected potentials: dense train [B][T][I] x W[I][O] -> fp64 [B][T][O]."""
    S = _c(S, np.uint8)
    W = _c(W, np.float32)
    B, T, I_ = S.shape
    I2, O = W.shape
    assert I_ == I2
    P_ = np.empty((B, T, O), np.float64)
    lib().oracle_fc(_p(S), B, T, I_, _p(W), O, _p(P_))
    return P_


def fc_stdp(W: np.ndarray, S_in: np.ndarray, win, nwin, cfgs) -> np.ndarray:
    """STDP of an FC layer (weights I x O), winners {b, t, o, 0, 0, cfg}; returns a copy."""
    W = np.array(W, dtype=np.float32, order="C", copy=True)
    S_in = _c(S_in, np.uint8)
    win = _c(win, np.int32)
    nwin = _c(nwin, np.int32)
    I_, O = W.shape
    B, T, I2 = S_in.shape
    assert I2 == I_
    assert win.shape[0] == B and nwin.shape[0] == B and win.shape[2] == 6, "winners must cover every sample"
    cfg = _c([[c[0], c[1], c[2], c[3]] for c in cfgs], np.float32)
    stab = _c([int(bool(c[4])) for c in cfgs], np.int32)
    lib().oracle_fc_stdp(_p(W), I_, O, _p(S_in), B, T, _p(win), _p(nwin), win.shape[1], _p(cfg), _p(stab),
                         len(cfgs))
    return W


def fcwta(Q: np.ndarray, count: int, radius: int):
    """FC winner-take-all on thresholded potentials [B][T][O] -> (win [B][count][6], nwin [B])."""
    Q = _c(Q, np.float64)
    B, T, O = Q.shape
    win = np.full((B, count, 6), -1, np.int32)
    nwin = np.zeros(B, np.int32)
    lib().oracle_fcwta(_p(Q), B, T, O, count, radius, _p(win), _p(nwin))
    return win, nwin
