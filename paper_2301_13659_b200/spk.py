"""ctypes binding of libspk.so (include/spk.h) — argument marshalling only.

Every function passes torch CUDA tensors' device pointers and the current
torch stream to the C ABI of the same name; every step of the hot path runs in
the library's CUDA kernels.  There is no fallback: if libspk.so is missing or a
call fails, SpkError is raised.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

_LIB_PATH = Path(os.environ.get("SPK_LIB_OVERRIDE", Path(__file__).resolve().parent / "libspk.so"))
_lib = None

SPK_PREC = {"fp32": 0, "exact": 1, "event": 2}
SPK_EPI = {"potential": 0, "fire": 1}


class SpkError(RuntimeError):
    pass


class ConvGeom(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("B", "T", "Ci", "Hi", "Wi", "Co", "Kh", "Kw", "Sh", "Sw", "Ph", "Pw")]


class PoolGeom(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("Lh", "Lw", "Sh", "Sw", "Ph", "Pw")]


class StdpConfig(ctypes.Structure):
    _fields_ = [("a_plus", ctypes.c_float), ("a_minus", ctypes.c_float), ("lower", ctypes.c_float),
                ("upper", ctypes.c_float), ("stabilize", ctypes.c_int32)]


EXPORTS = [
    "spk_last_error", "spk_abi_version", "spk_last_kernel", "spk_launch_count", "spk_dog", "spk_gabor",
    "spk_rank_code_workspace", "spk_rank_code", "spk_conv_workspace", "spk_conv", "spk_fire", "spk_pool",
    "spk_inhibit", "spk_wta", "spk_stdp_workspace", "spk_stdp", "spk_rstdp_route", "spk_winners_rebase", "spk_gather",
    "spk_lat_to_dense", "spk_dense_to_lat", "spk_conv_status", "spk_conv_fire_pool_supported", "spk_conv_fire_pool",
    "spk_rate_code_workspace", "spk_rate_code", "spk_rate_gather", "spk_pool_rates", "spk_quantize", "spk_fc_workspace",
    "spk_fc", "spk_fcwta", "spk_zca_fit_workspace", "spk_zca_fit", "spk_zca_apply", "spk_conv_prepack",
    "spk_stdp_status", "spk_inhibit_wta", "spk_log",
]


def lib():
    """Load libspk.so (built by paper_2301_13659_b200.build); raise if it is absent."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise SpkError(f"{_LIB_PATH} is missing: run `python -m paper_2301_13659_b200.build` "
                           "(there is no CPU fallback)")
        L = ctypes.CDLL(str(_LIB_PATH))
        V, I, F, Z, U64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_size_t, ctypes.c_uint64
        sig = {
            "spk_last_error": ([], ctypes.c_char_p),
            "spk_last_kernel": ([], ctypes.c_char_p),
            "spk_abi_version": ([], I),
            "spk_launch_count": ([], U64),
            "spk_dog": ([V, I, I, I, I, V, I, I, I, V, V], I),
            "spk_gabor": ([V, I, I, I, I, V, I, I, I, V, V], I),
            "spk_rank_code_workspace": ([I, I, I, I], Z),
            "spk_rank_code": ([V, I, I, I, F, I, V, V, Z, V], I),
            "spk_conv_workspace": ([ctypes.POINTER(ConvGeom), I], Z),
            "spk_conv": ([V, V, ctypes.POINTER(ConvGeom), I, I, F, F, V, V, V, Z, V], I),
            "spk_fire": ([V, I, I, I, I, I, F, V, V, V], I),
            "spk_pool": ([V, I, I, I, I, I, ctypes.POINTER(PoolGeom), V, V], I),
            "spk_inhibit": ([V, V, I, I, I, I, I, V], I),
            "spk_wta": ([V, V, I, I, I, I, I, I, I, V, V, V], I),
            "spk_stdp_workspace": ([ctypes.POINTER(ConvGeom), I], Z),
            "spk_stdp": ([V, ctypes.POINTER(ConvGeom), V, V, V, I, ctypes.POINTER(StdpConfig), I, V, Z, V], I),
            "spk_rstdp_route": ([V, V, I, I, V, I, V], I),
            "spk_winners_rebase": ([V, V, I, I, I, V], I),
            "spk_gather": ([V, Z, I, V, V], I),
            "spk_lat_to_dense": ([V, I, I, Z, V, V], I),
            "spk_dense_to_lat": ([V, I, I, Z, V, V, V], I),
            "spk_conv_status": ([V, ctypes.POINTER(I), V], I),
            "spk_conv_fire_pool_supported": ([ctypes.POINTER(ConvGeom), I, ctypes.POINTER(PoolGeom)], I),
            "spk_conv_fire_pool": ([V, V, ctypes.POINTER(ConvGeom), I, F, F, ctypes.POINTER(PoolGeom), V, V, Z, V], I),
            "spk_rate_code_workspace": ([I, I, I], Z),
            "spk_rate_code": ([V, I, I, I, F, U64, U64, V, V, Z, V], I),
            "spk_rate_gather": ([V, I, I, Z, V, V], I),
            "spk_pool_rates": ([V, V, I, I, I, I, I, ctypes.POINTER(PoolGeom), V, V], I),
            "spk_quantize": ([V, Z, F, F, F, V], I),
            "spk_fc_workspace": ([I, I, I, I, I], Z),
            "spk_fc": ([V, V, I, I, I, I, I, I, F, F, V, V, V, Z, V], I),
            "spk_fcwta": ([V, V, I, I, I, I, I, V, V, V], I),
            "spk_zca_fit_workspace": ([I, I], Z),
            "spk_zca_fit": ([V, I, I, ctypes.c_double, V, V, V, Z, V], I),
            "spk_zca_apply": ([V, I, I, V, V, V, V], I),
            "spk_conv_prepack": ([V, ctypes.POINTER(ConvGeom), I, F, V, Z, V], I),
            "spk_stdp_status": ([V, ctypes.POINTER(ConvGeom), I, ctypes.POINTER(ctypes.c_int32), V], I),
            "spk_inhibit_wta": ([V, V, I, I, I, I, I, I, I, V, V, V], I),
            "spk_log": ([V, I, I, I, I, V, I, I, I, V, V], I),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _check(name: str, st: int):
    if st != 0:
        raise SpkError(f"{name} -> status {st}: {lib().spk_last_error().decode()}")


def _p(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise SpkError("libspk takes CUDA tensors only")
    if not t.is_contiguous():
        raise SpkError("libspk takes contiguous tensors only")
    return ctypes.c_void_p(t.data_ptr())


def _s():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def launch_count() -> int:
    return int(lib().spk_launch_count())


def last_kernel() -> str:
    return lib().spk_last_kernel().decode()


# ---------------------------------------------------------------- a1 filters
def dog(img: torch.Tensor, sigmas, radius: int, pad: int, out: torch.Tensor | None = None) -> torch.Tensor:
    B, C, H, W = img.shape
    sig = (ctypes.c_double * (2 * len(sigmas)))(*[float(v) for pr in sigmas for v in pr])
    e = 2 * radius + 1
    if out is None:
        out = torch.empty((B, C * len(sigmas), H + 2 * pad - e + 1, W + 2 * pad - e + 1), dtype=torch.float32,
                          device=img.device)
    _check("spk_dog", lib().spk_dog(_p(img), B, C, H, W, sig, len(sigmas), radius, pad, _p(out), _s()))
    return out


def log(img: torch.Tensor, stds, radius: int, pad: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """LoG bank: 2 channels (a DoG pair) per std, expanded behind the ABI (spk_log)."""
    B, C, H, W = img.shape
    st = (ctypes.c_double * len(stds))(*[float(v) for v in stds])
    e = 2 * radius + 1
    if out is None:
        out = torch.empty((B, C * 2 * len(stds), H + 2 * pad - e + 1, W + 2 * pad - e + 1), dtype=torch.float32,
                          device=img.device)
    _check("spk_log", lib().spk_log(_p(img), B, C, H, W, st, len(stds), radius, pad, _p(out), _s()))
    return out


def log_pairs(stds):
    """The DoG sigma pairs spk_log expands a LoG bank into (for inspection; spk_log does it)."""
    r2 = 2.0 ** 0.5
    out = []
    for s in stds:
        out += [(s * r2, s / r2), (s / r2, s * r2)]
    return out


def gabor(img: torch.Tensor, params, radius: int, pad: int, out: torch.Tensor | None = None) -> torch.Tensor:
    B, C, H, W = img.shape
    par = (ctypes.c_double * (5 * len(params)))(*[float(v) for pr in params for v in pr])
    e = 2 * radius + 1
    if out is None:
        out = torch.empty((B, C * len(params), H + 2 * pad - e + 1, W + 2 * pad - e + 1), dtype=torch.float32,
                          device=img.device)
    _check("spk_gabor", lib().spk_gabor(_p(img), B, C, H, W, par, len(params), radius, pad, _p(out), _s()))
    return out


# ---------------------------------------------------------------- a2 coding
def rank_code(y: torch.Tensor, T: int, thresh: float, sort: bool = True,
              out: torch.Tensor | None = None) -> torch.Tensor:
    B = y.shape[0]
    N = y[0].numel()
    if out is None:
        out = torch.empty(y.shape, dtype=torch.uint8, device=y.device)
    _check("spk_rank_code", lib().spk_rank_code(_p(y), B, N, T, float(thresh), int(bool(sort)), _p(out), None, 0,
                                                _s()))
    return out


# ---------------------------------------------------------------- a3/a4 conv + fire
def conv_geom(lat_in: torch.Tensor, w: torch.Tensor, T: int, stride=1, pad=0) -> ConvGeom:
    B, Ci, Hi, Wi = lat_in.shape
    Co, Ci2, Kh, Kw = w.shape
    if Ci != Ci2:
        raise SpkError(f"channel mismatch {Ci} vs {Ci2}")
    s = stride if isinstance(stride, (tuple, list)) else (stride, stride)
    p = pad if isinstance(pad, (tuple, list)) else (pad, pad)
    return ConvGeom(B, T, Ci, Hi, Wi, Co, Kh, Kw, s[0], s[1], p[0], p[1])


def conv_out_hw(g: ConvGeom):
    return (g.Hi + 2 * g.Ph - g.Kh) // g.Sh + 1, (g.Wi + 2 * g.Pw - g.Kw) // g.Sw + 1


def conv_workspace(g: ConvGeom, prec: str = "exact") -> int:
    return int(lib().spk_conv_workspace(ctypes.byref(g), SPK_PREC[prec]))


def conv(lat_in: torch.Tensor, w: torch.Tensor, T: int, stride=1, pad=0, prec: str = "exact",
         epi: str = "fire", theta: float = 0.0, w_max: float = 1.0, out0=None, out1=None, ws=None,
         want_pstar: bool = True, prepacked: bool = False):
    """Eq. 2 potentials (epi='potential' -> f32 [B][T][Co][Ho][Wo]) or IF fire
    (epi='fire' -> (lat u8 [B][Co][Ho][Wo], P* f32 or None)).  prepacked: ws holds w packed by
    conv_prepack (w only gives the shape)."""
    g = conv_geom(lat_in, w, T, stride, pad)
    Ho, Wo = conv_out_hw(g)
    dev = lat_in.device
    if out0 is None:
        out0 = (torch.empty((g.B, T, g.Co, Ho, Wo), dtype=torch.float32, device=dev) if epi == "potential"
                else torch.empty((g.B, g.Co, Ho, Wo), dtype=torch.uint8, device=dev))
    if epi == "fire" and want_pstar and out1 is None:
        out1 = torch.empty((g.B, g.Co, Ho, Wo), dtype=torch.float32, device=dev)
    need = conv_workspace(g, prec)
    if ws is None and need:
        ws = torch.empty(need, dtype=torch.uint8, device=dev)
    nbytes = ws.numel() if ws is not None else 0
    _check("spk_conv", lib().spk_conv(_p(lat_in), None if prepacked else _p(w), ctypes.byref(g), SPK_PREC[prec],
                                      SPK_EPI[epi],
                                      float(theta), float(w_max), _p(out0), _p(out1), _p(ws), nbytes, _s()))
    return out0 if epi == "potential" else (out0, out1)


def conv_prepack(w: torch.Tensor, g: ConvGeom, prec: str, w_max: float, ws: torch.Tensor):
    """Pack a layer's weights into ws once; later conv()/conv_fire_pool() calls pass w=None."""
    _check("spk_conv_prepack", lib().spk_conv_prepack(_p(w), ctypes.byref(g), SPK_PREC[prec], float(w_max), _p(ws),
                                                      ws.numel(), _s()))
    return ws


def conv_clamp_flag(ws: torch.Tensor) -> int:
    v = ctypes.c_int(0)
    _check("spk_conv_status", lib().spk_conv_status(_p(ws), ctypes.byref(v), _s()))
    return v.value


def fire(pot: torch.Tensor, theta: float, out=None, pstar=None, want_pstar: bool = True):
    B, T, C, H, W = pot.shape
    if out is None:
        out = torch.empty((B, C, H, W), dtype=torch.uint8, device=pot.device)
    if want_pstar and pstar is None:
        pstar = torch.empty((B, C, H, W), dtype=torch.float32, device=pot.device)
    _check("spk_fire", lib().spk_fire(_p(pot), B, T, C, H, W, float(theta), _p(out), _p(pstar), _s()))
    return out, pstar


# ---------------------------------------------------------------- a5 pool
def pool(lat: torch.Tensor, T: int, kernel, stride=None, pad=0, out=None) -> torch.Tensor:
    B, C, H, W = lat.shape
    k = kernel if isinstance(kernel, (tuple, list)) else (kernel, kernel)
    s = stride if stride is not None else k
    s = s if isinstance(s, (tuple, list)) else (s, s)
    p = pad if isinstance(pad, (tuple, list)) else (pad, pad)
    geom = PoolGeom(k[0], k[1], s[0], s[1], p[0], p[1])
    Ho, Wo = (H + 2 * p[0] - k[0]) // s[0] + 1, (W + 2 * p[1] - k[1]) // s[1] + 1
    if out is None:
        out = torch.empty((B, C, Ho, Wo), dtype=torch.uint8, device=lat.device)
    _check("spk_pool", lib().spk_pool(_p(lat), B, C, H, W, T, ctypes.byref(geom), _p(out), _s()))
    return out


def _pool_geom(kernel, stride=None, pad=0):
    k = kernel if isinstance(kernel, (tuple, list)) else (kernel, kernel)
    s = stride if stride is not None else k
    s = s if isinstance(s, (tuple, list)) else (s, s)
    p = pad if isinstance(pad, (tuple, list)) else (pad, pad)
    return PoolGeom(k[0], k[1], s[0], s[1], p[0], p[1])


def conv_fire_pool_supported(g: ConvGeom, prec: str, kernel, stride=None, pad=0) -> bool:
    return bool(lib().spk_conv_fire_pool_supported(ctypes.byref(g), SPK_PREC[prec],
                                                   ctypes.byref(_pool_geom(kernel, stride, pad))))


def conv_fire_pool(lat_in: torch.Tensor, w: torch.Tensor, T: int, stride=1, pad=0, prec: str = "event",
                   theta: float = 0.0, w_max: float = 1.0, pool_kernel=2, pool_stride=None, pool_pad=0,
                   out=None, ws=None, prepacked: bool = False) -> torch.Tensor:
    """spk_conv(FIRE) + spk_pool fused: pooled latencies [B][Co][Hp][Wp]."""
    g = conv_geom(lat_in, w, T, stride, pad)
    Ho, Wo = conv_out_hw(g)
    pg = _pool_geom(pool_kernel, pool_stride, pool_pad)
    Hp, Wp = (Ho + 2 * pg.Ph - pg.Lh) // pg.Sh + 1, (Wo + 2 * pg.Pw - pg.Lw) // pg.Sw + 1
    if out is None:
        out = torch.empty((g.B, g.Co, Hp, Wp), dtype=torch.uint8, device=lat_in.device)
    need = conv_workspace(g, prec)
    if ws is None and need:
        ws = torch.empty(need, dtype=torch.uint8, device=lat_in.device)
    nbytes = ws.numel() if ws is not None else 0
    _check("spk_conv_fire_pool", lib().spk_conv_fire_pool(_p(lat_in), None if prepacked else _p(w), ctypes.byref(g),
                                                          SPK_PREC[prec],
                                                          float(theta), float(w_max), ctypes.byref(pg), _p(out),
                                                          _p(ws), nbytes, _s()))
    return out


# ---------------------------------------------------------------- a6 inhibit, a7 wta
def inhibit(lat: torch.Tensor, pstar: torch.Tensor, T: int):
    B, C, H, W = lat.shape
    _check("spk_inhibit", lib().spk_inhibit(_p(lat), _p(pstar), B, C, H, W, T, _s()))
    return lat, pstar


def wta(lat: torch.Tensor, pstar: torch.Tensor, T: int, k: int, radius: int, win=None, nwin=None):
    B, C, H, W = lat.shape
    if win is None:
        win = torch.empty((B, k, 6), dtype=torch.int32, device=lat.device)
    if nwin is None:
        nwin = torch.empty((B,), dtype=torch.int32, device=lat.device)
    _check("spk_wta", lib().spk_wta(_p(lat), _p(pstar), B, C, H, W, T, k, radius, _p(win), _p(nwin), _s()))
    return win, nwin


def inhibit_wta(lat: torch.Tensor, pstar: torch.Tensor, T: int, k: int, radius: int, win=None, nwin=None):
    """spk_inhibit + spk_wta fused: winners of the inhibited records (records not modified)."""
    B, C, H, W = lat.shape
    if win is None:
        win = torch.empty((B, k, 6), dtype=torch.int32, device=lat.device)
    if nwin is None:
        nwin = torch.empty((B,), dtype=torch.int32, device=lat.device)
    _check("spk_inhibit_wta", lib().spk_inhibit_wta(_p(lat), _p(pstar), B, C, H, W, T, k, radius, _p(win), _p(nwin),
                                                    _s()))
    return win, nwin


# ---------------------------------------------------------------- a8 stdp
def stdp_configs(cfgs):
    arr = (StdpConfig * len(cfgs))()
    for i, c in enumerate(cfgs):
        arr[i] = StdpConfig(float(c[0]), float(c[1]), float(c[2]), float(c[3]), int(bool(c[4])))
    return arr


def stdp_workspace(g: ConvGeom, k: int) -> int:
    return int(lib().spk_stdp_workspace(ctypes.byref(g), k))


def stdp(w: torch.Tensor, lat_in: torch.Tensor, win: torch.Tensor, nwin: torch.Tensor, cfgs, T: int, stride=1,
         pad=0, ws=None, cfg_arr=None):
    """In-place STDP of conv weights w from winners (Listing 3 conv.stdp)."""
    g = conv_geom(lat_in, w, T, stride, pad)
    k = win.shape[1]
    need = stdp_workspace(g, k)
    if ws is None:
        ws = torch.empty(need, dtype=torch.uint8, device=w.device)
    arr = cfg_arr if cfg_arr is not None else stdp_configs(cfgs)
    _check("spk_stdp", lib().spk_stdp(_p(w), ctypes.byref(g), _p(lat_in), _p(win), _p(nwin), k, arr, len(arr),
                                      _p(ws), ws.numel(), _s()))
    return w


def stdp_invalid(ws: torch.Tensor, lat_in: torch.Tensor, w: torch.Tensor, T: int, k: int, stride=1, pad=0) -> int:
    """Winners the last stdp() on ws skipped (out-of-range coordinate or config)."""
    g = conv_geom(lat_in, w, T, stride, pad)
    v = ctypes.c_int32(0)
    _check("spk_stdp_status", lib().spk_stdp_status(_p(ws), ctypes.byref(g), k, ctypes.byref(v), _s()))
    return v.value


def rstdp_route(win: torch.Tensor, nwin: torch.Tensor, labels: torch.Tensor, maps_per_class: int):
    B, k, _ = win.shape
    _check("spk_rstdp_route", lib().spk_rstdp_route(_p(win), _p(nwin), B, k, _p(labels), maps_per_class, _s()))
    return win


def winners_rebase(win: torch.Tensor, nwin: torch.Tensor, b0: int):
    """Local -> global sample index of every valid winner (data-parallel mini-batch STDP)."""
    B, k, _ = win.shape
    _check("spk_winners_rebase", lib().spk_winners_rebase(_p(win), _p(nwin), B, k, int(b0), _s()))
    return win


# ---------------------------------------------------------------- a9 gather + boundary
def gather(lat: torch.Tensor, T: int, out=None) -> torch.Tensor:
    if out is None:
        out = torch.empty(lat.shape, dtype=torch.float32, device=lat.device)
    _check("spk_gather", lib().spk_gather(_p(lat), lat.numel(), T, _p(out), _s()))
    return out


def lat_to_dense(lat: torch.Tensor, T: int) -> torch.Tensor:
    B = lat.shape[0]
    N = lat[0].numel()
    out = torch.empty((B, T) + tuple(lat.shape[1:]), dtype=torch.uint8, device=lat.device)
    _check("spk_lat_to_dense", lib().spk_lat_to_dense(_p(lat), B, T, N, _p(out), _s()))
    return out


def dense_to_lat(dense: torch.Tensor):
    B, T = dense.shape[:2]
    N = dense[0, 0].numel()
    lat = torch.empty((B,) + tuple(dense.shape[2:]), dtype=torch.uint8, device=dense.device)
    bad = torch.empty((1,), dtype=torch.int32, device=dense.device)
    _check("spk_dense_to_lat", lib().spk_dense_to_lat(_p(dense), B, T, N, _p(lat), _p(bad), _s()))
    return lat, bad


# ---------------------------------------------------------------- NEXT-3 rate coding
def rate_code(y: torch.Tensor, T: int, thresh: float, seed: int, b0: int = 0, out=None, ws=None) -> torch.Tensor:
    """Per-step Bernoulli rate coding -> step map u8 [B][T][...] (0 = spike at that step); b0 = global
    index of sample 0 (the random stream runs over global sample indices)."""
    B = y.shape[0]
    N = y[0].numel()
    if out is None:
        out = torch.empty((B, T) + tuple(y.shape[1:]), dtype=torch.uint8, device=y.device)
    if ws is None:
        ws = torch.empty(int(lib().spk_rate_code_workspace(B, N, T)), dtype=torch.uint8, device=y.device)
    _check("spk_rate_code", lib().spk_rate_code(_p(y), B, N, T, float(thresh), int(seed) & (2 ** 64 - 1), int(b0), _p(out),
                                                _p(ws), ws.numel(), _s()))
    return out


def rate_gather(step: torch.Tensor, out=None) -> torch.Tensor:
    """Firing rate (spikes / T) of a step map [B][T][...] -> f32 [B][...]."""
    B, T = step.shape[:2]
    N = step[0, 0].numel()
    if out is None:
        out = torch.empty((B,) + tuple(step.shape[2:]), dtype=torch.float32, device=step.device)
    _check("spk_rate_gather", lib().spk_rate_gather(_p(step), B, T, N, _p(out), _s()))
    return out


def pool_rates(step: torch.Tensor, rate: torch.Tensor, kernel, stride=None, pad=0, out=None) -> torch.Tensor:
    """Rate-based max pooling of a step map [B][T][C][H][W] with rates [B][C][H][W]."""
    B, T, C, H, W = step.shape
    pg = _pool_geom(kernel, stride, pad)
    Ho, Wo = (H + 2 * pg.Ph - pg.Lh) // pg.Sh + 1, (W + 2 * pg.Pw - pg.Lw) // pg.Sw + 1
    if out is None:
        out = torch.empty((B, T, C, Ho, Wo), dtype=torch.uint8, device=step.device)
    _check("spk_pool_rates", lib().spk_pool_rates(_p(step), _p(rate), B, T, C, H, W, ctypes.byref(pg), _p(out), _s()))
    return out


# ---------------------------------------------------------------- NEXT-4 quantize, FC, fcwta, ZCA
def quantize(w: torch.Tensor, lower: float, mid: float, upper: float) -> torch.Tensor:
    """Listing 4 quantize(kernel, lower, mid, upper), in place."""
    _check("spk_quantize", lib().spk_quantize(_p(w), w.numel(), float(lower), float(mid), float(upper), _s()))
    return w


def fc_workspace(B: int, T: int, I: int, O: int, prec: str = "exact") -> int:
    return int(lib().spk_fc_workspace(B, T, I, O, SPK_PREC[prec]))


def fc(lat_in: torch.Tensor, w: torch.Tensor, T: int, prec: str = "exact", epi: str = "fire", theta: float = 0.0,
       w_max: float = 1.0, out0=None, out1=None, ws=None, want_pstar: bool = True):
    """FC IF layer: lat_in u8 [B][I], w f32 [O][I] (the paper's I x O kernel, output-major)."""
    B, I = lat_in.shape
    O, I2 = w.shape
    if I != I2:
        raise SpkError(f"FC input size mismatch {I} vs {I2}")
    dev = lat_in.device
    if out0 is None:
        out0 = (torch.empty((B, T, O), dtype=torch.float32, device=dev) if epi == "potential"
                else torch.empty((B, O), dtype=torch.uint8, device=dev))
    if epi == "fire" and want_pstar and out1 is None:
        out1 = torch.empty((B, O), dtype=torch.float32, device=dev)
    need = fc_workspace(B, T, I, O, prec)
    if ws is None and need:
        ws = torch.empty(need, dtype=torch.uint8, device=dev)
    nbytes = ws.numel() if ws is not None else 0
    _check("spk_fc", lib().spk_fc(_p(lat_in), _p(w), B, T, I, O, SPK_PREC[prec], SPK_EPI[epi], float(theta),
                                  float(w_max), _p(out0), _p(out1), _p(ws), nbytes, _s()))
    return out0 if epi == "potential" else (out0, out1)


def fcwta(lat: torch.Tensor, pstar: torch.Tensor, T: int, k: int, radius: int, win=None, nwin=None):
    B, O = lat.shape
    if win is None:
        win = torch.empty((B, k, 6), dtype=torch.int32, device=lat.device)
    if nwin is None:
        nwin = torch.empty((B,), dtype=torch.int32, device=lat.device)
    _check("spk_fcwta", lib().spk_fcwta(_p(lat), _p(pstar), B, O, T, k, radius, _p(win), _p(nwin), _s()))
    return win, nwin


def fc_stdp(w: torch.Tensor, lat_in: torch.Tensor, win: torch.Tensor, nwin: torch.Tensor, cfgs, T: int, ws=None,
            cfg_arr=None):
    """STDP of an FC layer (w [O][I]) = spk_stdp on the 1x1 geometry."""
    B, I = lat_in.shape
    return stdp(w.view(w.shape[0], I, 1, 1), lat_in.view(B, I, 1, 1), win, nwin, cfgs, T, 1, 0, ws=ws,
                cfg_arr=cfg_arr)


def zca_fit(x: torch.Tensor, eps: float):
    """ZCA fit (synchronous): x f32 [B][F] -> (mean [F], Wz [F][F])."""
    B, F = x.shape
    mean = torch.empty((F,), dtype=torch.float32, device=x.device)
    wz = torch.empty((F, F), dtype=torch.float32, device=x.device)
    ws = torch.empty(int(lib().spk_zca_fit_workspace(B, F)), dtype=torch.uint8, device=x.device)
    _check("spk_zca_fit", lib().spk_zca_fit(_p(x), B, F, float(eps), _p(mean), _p(wz), _p(ws), ws.numel(), _s()))
    return mean, wz


def zca_apply(x: torch.Tensor, mean: torch.Tensor, wz: torch.Tensor, out=None) -> torch.Tensor:
    B, F = x.shape
    if out is None:
        out = torch.empty_like(x)
    _check("spk_zca_apply", lib().spk_zca_apply(_p(x), B, F, _p(mean), _p(wz), _p(out), _s()))
    return out
