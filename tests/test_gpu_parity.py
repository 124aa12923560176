"""GPU parity: every libspk stage against the CPU oracle on the same seeded inputs.

Stage-wise tests are teacher-forced (the GPU stage gets the oracle's input to
that stage); pipeline tests run end to end.  Comparison rules: tests/parity.py.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import pipeline as opipe
from parity import (ParityReport, assert_potentials, compare_latency, lat_and_pstar, near_threshold,
                    near_ties_inhibit, near_ties_wta)

pytestmark = pytest.mark.gpu
RNG = np.random.default_rng(2024)


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


# ------------------------------------------------------------------------- a1 filters
@pytest.mark.parametrize("name", ["c1", "c2", "c4", "c5"])
def test_filter_bit_identical(spk, name):
    cfg = synth.load_config(name)
    imgs = synth.images(cfg, 0, 3)
    fr = cfg["front"]
    ref = oracle.filter_apply(imgs, opipe.filter_bank(cfg), fr["pad"])
    if fr["kind"] == "dog":
        got = spk.dog(cu(imgs), fr["pairs"], fr["radius"], fr["pad"])
    elif fr["kind"] == "log":
        got = spk.log(cu(imgs), fr["stds"], fr["radius"], fr["pad"])  # pairs expanded behind the ABI
    else:
        got = spk.gabor(cu(imgs), fr["params"], fr["radius"], fr["pad"])
    # bit for bit, including the sign of zeros (on/off pairs are computed as 0 - acc)
    np.testing.assert_array_equal(host(got).view(np.uint32), ref.astype(np.float32).view(np.uint32))


def test_filter_odd_geometry(spk):
    imgs = RNG.integers(0, 256, (2, 3, 37, 45), dtype=np.uint8)
    for r, pad in [(2, 0), (3, 1), (1, 4), (0, 0)]:
        pairs = [(0.8, 1.7), (2.2, 1.1)]
        ref = oracle.filter_apply(imgs, oracle.dog_bank(pairs, r), pad)
        np.testing.assert_array_equal(host(spk.dog(cu(imgs), pairs, r, pad)).view(np.uint32),
                                      ref.astype(np.float32).view(np.uint32))
        onoff = [(1.0, 2.0), (2.0, 1.0), (0.7, 1.5), (1.5, 0.7)]  # exact negation pairs
        ref = oracle.filter_apply(imgs, oracle.dog_bank(onoff, r), pad)
        np.testing.assert_array_equal(host(spk.dog(cu(imgs), onoff, r, pad)).view(np.uint32),
                                      ref.astype(np.float32).view(np.uint32))
        gab = [(2.0, 0.3, 0.6, 4.0, 0.5)]
        ref = oracle.filter_apply(imgs, oracle.gabor_bank(gab, r), pad)
        np.testing.assert_array_equal(host(spk.gabor(cu(imgs), gab, r, pad)), ref)


# ---------------------------------------------------------------------- a2 rank coding
@pytest.mark.parametrize("T", [1, 4, 15, 30, 100, 254])
@pytest.mark.parametrize("sort", [True, False])
def test_rank_code_exact(spk, T, sort):
    cfg = synth.load_config("c2")
    imgs = synth.images(cfg, 0, 6)
    y = oracle.filter_apply(imgs, opipe.filter_bank(cfg), 3)
    y[1] = np.round(y[1] * 8) / 8          # many ties
    y[2] = 0.0                             # nothing fires
    y[3] = -1.0
    y[3, 0, 5, 5] = 0.5                    # a single positive
    y[4, :, :14] = y[4, :, 14:]            # exact duplicate halves
    ref = oracle.rank_code(y, T, 0.01, sort)
    got = host(spk.rank_code(cu(y), T, 0.01, sort))
    np.testing.assert_array_equal(got, ref)


def test_rank_code_large_sample_global_path(spk):
    y = RNG.normal(0, 1, (3, 50_000)).astype(np.float32)  # > staged limit -> global-memory path
    y[0, ::7] = np.round(y[0, ::7], 1)
    for T, sort in [(15, True), (30, True), (15, False)]:
        np.testing.assert_array_equal(host(spk.rank_code(cu(y), T, 0.01, sort)), oracle.rank_code(y, T, 0.01, sort))


@pytest.mark.parametrize("T", [1, 15, 30, 254])
def test_rank_code_large_sample_histogram_path(spk, T):
    """N > 8192, sort on: bucket histogram + boundary-bucket sort, and its radix-select
    fallback when a boundary bucket holds more exact ties than shared memory."""
    cfg = synth.load_config("c4")
    imgs = synth.images(cfg, 0, 2)
    y = oracle.filter_apply(imgs, opipe.filter_bank(cfg), 3)   # C4-shaped Gabor responses
    y = np.concatenate([y.reshape(2, -1), RNG.normal(0, 1, (4, y[0].size)).astype(np.float32)])
    y[2, : y.shape[1] // 2] = 0.5                              # 80,000 exact ties -> fallback
    y[3] = np.round(y[3], 2)                                   # ties across many buckets
    y[4] = -1.0
    y[4, 12345] = 3.0                                          # a single positive
    y[5, 1::3] = np.float32(2.0) ** RNG.integers(-6, 6, y[5, 1::3].shape)  # bucket edges
    y = np.concatenate([y, np.full((1, y.shape[1]), -1.0, np.float32)])  # nothing fires
    np.testing.assert_array_equal(host(spk.rank_code(cu(y), T, 0.01, True)), oracle.rank_code(y, T, 0.01, True))


@pytest.mark.parametrize("N", [65_536, 301_056, 400_004])
def test_rank_code_c5_sized_samples(spk, N):
    """Large samples, sort on (C5: 301,056 values per sample): ties across buckets, N/2 exact
    ties in the middle of the sample (radix-select fallback), an empty sample, every value twice."""
    y = RNG.normal(0, 1, (5, N)).astype(np.float32)
    y[1] = np.round(y[1], 2)                      # ties across buckets and across the CTA parts
    y[2, N // 4: 3 * N // 4] = 0.75               # N/2 exact ties straddling the parts -> fallback
    y[3] = -1.0                                   # nothing fires
    y[4, : N // 2] = y[4, N // 2:]                # every value twice, once in each half
    for T in (1, 15, 30):
        np.testing.assert_array_equal(host(spk.rank_code(cu(y), T, 0.01, True)), oracle.rank_code(y, T, 0.01, True))


@pytest.mark.parametrize("N", [1, 3, 4705, 8192, 8193, 50_001])
@pytest.mark.parametrize("T", [1, 15, 30])
def test_rank_code_odd_sizes(spk, N, T):
    """Sample sizes around every dispatch edge (small staged histogram <= 8192 < large
    histogram), N % 4 != 0 (scalar paths), a single value, heavy ties."""
    y = RNG.normal(0, 1, (3, N)).astype(np.float32)
    y[1] = np.round(y[1], 1)
    y[2, : N // 2] = 0.25
    for sort in (True, False):
        np.testing.assert_array_equal(host(spk.rank_code(cu(y), T, 0.01, sort)), oracle.rank_code(y, T, 0.01, sort))


# ------------------------------------------------------------------------- a3 conv
CONV_CASES = [
    # B, T, Ci, Hi, Wi, Co, K, stride, pad
    (2, 15, 6, 28, 28, 30, 5, 1, 2),      # C2 conv1
    (2, 15, 30, 14, 14, 250, 3, 1, 1),    # C2 conv2 (2 N tiles)
    (3, 15, 250, 4, 4, 200, 5, 1, 2),     # C2 conv3 (K = 6250, 98 stages)
    (1, 30, 4, 20, 23, 64, 5, 1, 2),      # C4 conv1 shape class, T = 30
    (2, 30, 64, 9, 11, 128, 3, 1, 1),     # C4 conv2 shape class
    (3, 7, 3, 9, 11, 20, 3, 2, 0),        # strided, ragged tiles
    (1, 16, 5, 6, 5, 17, 4, 3, 1),        # T = TP, odd Co
    (2, 1, 2, 5, 7, 8, 2, 1, 0),          # T = 1
    (160, 15, 2, 12, 12, 8, 5, 1, 2),     # grid >= 148 CTAs: whole sample per event CTA
    # T = 1 (one time step per row; kernel rows of 3..7 synapses padded to 8 in K, read as words)
    (3, 1, 6, 13, 17, 20, 5, 1, 2),       # C6 conv0 shape class, ragged 128-pixel tiles
    (2, 1, 25, 14, 14, 50, 3, 1, 1),      # C6 conv1 shape class, 2 N tiles
    (2, 1, 3, 11, 9, 12, 7, 2, 3),        # 7-wide rows, stride 2, pad 3 (rows end in the sentinel)
    (1, 1, 40, 9, 10, 33, 5, 1, 0),       # K' = 1600 over many stages, Co = 33
]


def _conv_inputs(B, T, Ci, Hi, Wi, Co, K, dens=0.5):
    lat = RNG.integers(0, T, (B, Ci, Hi, Wi)).astype(np.uint8)
    lat[RNG.random(lat.shape) > dens] = T  # never fires
    w = RNG.uniform(0.0, 1.0, (Co, Ci, K, K)).astype(np.float32)
    return lat, w


def _skip_unsupported(spk, lat, w, T, s, p, prec):
    if prec == "event" and spk.conv_workspace(spk.conv_geom(cu(lat), cu(w), T, s, p), "event") == 0:
        pytest.skip("event path: weight block does not fit shared memory")


@pytest.mark.parametrize("case", CONV_CASES)
@pytest.mark.parametrize("prec", ["exact", "fp32", "event"])
def test_conv_potentials(spk, case, prec):
    B, T, Ci, Hi, Wi, Co, K, s, p = case
    lat, w = _conv_inputs(B, T, Ci, Hi, Wi, Co, K)
    _skip_unsupported(spk, lat, w, T, s, p, prec)
    ref = oracle.conv_event(lat, T, w, (s, s), (p, p))
    got = host(spk.conv(cu(lat), cu(w), T, s, p, prec=prec, epi="potential"))
    ParityReport.potentials(("conv potentials (CONV_CASES)", prec), got, ref)
    assert_potentials(got, ref)


@pytest.mark.parametrize("case", CONV_CASES)
@pytest.mark.parametrize("prec", ["exact", "fp32", "event"])
def test_conv_fire_epilogue(spk, case, prec):
    B, T, Ci, Hi, Wi, Co, K, s, p = case
    lat, w = _conv_inputs(B, T, Ci, Hi, Wi, Co, K)
    _skip_unsupported(spk, lat, w, T, s, p, prec)
    P = oracle.conv_event(lat, T, w, (s, s), (p, p))
    theta = float(np.percentile(P[:, -1], 60)) + 0.123  # fire for roughly 40 % of neurons
    ref_lat, ref_ps = lat_and_pstar(P, theta)
    glat, gps = spk.conv(cu(lat), cu(w), T, s, p, prec=prec, epi="fire", theta=theta)
    glat, gps = host(glat), host(gps)
    excl = near_threshold(P, theta)
    ParityReport.latency(("conv fire (CONV_CASES)", prec), glat, ref_lat, excl)
    compare_latency(glat, ref_lat, excl)
    ok = (glat == ref_lat) & (ref_lat < T)
    ParityReport.potentials(("conv fire P* (CONV_CASES)", prec), gps[ok], ref_ps[ok])
    assert_potentials(gps[ok], ref_ps[ok])
    assert (gps[glat == T] == 0).all()


@pytest.mark.parametrize("case", CONV_CASES)
@pytest.mark.parametrize("dens", [0.05, 0.5, 1.0])
def test_conv_event_equals_exact_bitwise(spk, case, dens):
    """The event (latency-histogram) form sums the same fixed-point weights exactly, so its
    latencies and P* equal the tensor-core path's bit for bit (any density, any T)."""
    B, T, Ci, Hi, Wi, Co, K, s, p = case
    lat, w = _conv_inputs(B, T, Ci, Hi, Wi, Co, K, dens)
    _skip_unsupported(spk, lat, w, T, s, p, "event")
    P = oracle.conv_event(lat, T, w, (s, s), (p, p))
    theta = float(np.percentile(P[:, -1], 60)) + 0.123
    el, ep = spk.conv(cu(lat), cu(w), T, s, p, prec="event", epi="fire", theta=theta)
    xl, xp = spk.conv(cu(lat), cu(w), T, s, p, prec="exact", epi="fire", theta=theta)
    np.testing.assert_array_equal(host(el), host(xl))
    np.testing.assert_array_equal(host(ep), host(xp))
    np.testing.assert_array_equal(host(spk.conv(cu(lat), cu(w), T, s, p, prec="event", epi="potential")),
                                  host(spk.conv(cu(lat), cu(w), T, s, p, prec="exact", epi="potential")))


def test_conv_quantised_weights_exact_integers(spk):
    # binary weights (Listing 4 quantize) make potentials exact integers on every path
    lat, _ = _conv_inputs(2, 15, 30, 14, 14, 250, 3)
    w = RNG.integers(0, 2, (250, 30, 3, 3)).astype(np.float32)
    ref = oracle.conv_event(lat, 15, w, (1, 1), (1, 1))
    for prec in ("exact", "fp32", "event"):
        np.testing.assert_array_equal(host(spk.conv(cu(lat), cu(w), 15, 1, 1, prec=prec, epi="potential")), ref)


def test_conv_weight_scale_and_clamp_flag(spk):
    lat, w = _conv_inputs(1, 15, 4, 8, 8, 16, 3)
    w2 = w * 3.0  # w_max = 3 -> scale 4
    ref = oracle.conv_event(lat, 15, w2, (1, 1), (1, 1))
    g = spk.conv_geom(cu(lat), cu(w2), 15, 1, 1)
    ws = torch.empty(spk.conv_workspace(g), dtype=torch.uint8, device="cuda")
    got = spk.conv(cu(lat), cu(w2), 15, 1, 1, epi="potential", w_max=3.0, ws=ws)
    assert_potentials(host(got), ref)
    assert spk.conv_clamp_flag(ws) == 0
    spk.conv(cu(lat), cu(w2), 15, 1, 1, epi="potential", w_max=1.0, ws=ws)  # weights above the scale
    assert spk.conv_clamp_flag(ws) == 1


def test_conv_matches_dense_definition(spk):
    # the direct BTCHW definition of Eq. 2 (not only the event form)
    lat, w = _conv_inputs(2, 6, 3, 7, 9, 12, 3)
    ref = oracle.conv(oracle.lat_to_dense(lat, 6), w, (1, 1), (1, 1))
    assert_potentials(host(spk.conv(cu(lat), cu(w), 6, 1, 1, epi="potential")), ref)


# ------------------------------------------------------------------------- a4 fire
def test_fire_exact(spk):
    P = np.cumsum(RNG.uniform(0, 2, (3, 15, 5, 7, 9)), axis=1).astype(np.float32)
    theta = 9.5
    lat, ps = spk.fire(cu(P), theta)
    S = oracle.fire(P.astype(np.float64), theta)
    np.testing.assert_array_equal(host(lat), oracle.dense_to_lat(S))
    rl, rp = lat_and_pstar(P.astype(np.float64), theta)
    np.testing.assert_array_equal(host(ps), rp.astype(np.float32))


@pytest.mark.parametrize("T", [1, 7, 15, 30])
@pytest.mark.parametrize("monotone", [True, False])
def test_fire_vectorised_exact(spk, T, monotone):
    """The 4-neurons-per-thread kernel (N % 4 == 0): first strict crossing and P*, including
    non-monotone potentials (the first crossing, not the last) and never-firing neurons."""
    P = RNG.uniform(0, 2, (3, T, 8, 9, 12))
    if monotone:
        P = np.cumsum(P, axis=1)
    P = P.astype(np.float32)
    theta = float(np.percentile(P, 60))
    lat, ps = spk.fire(cu(P), theta)
    rl, rp = lat_and_pstar(P.astype(np.float64), theta)
    np.testing.assert_array_equal(host(lat), rl)
    np.testing.assert_array_equal(host(ps), rp.astype(np.float32))


# ------------------------------------------------------------------------- a5 pool
@pytest.mark.parametrize("L,s,p", [(2, 2, 0), (3, 3, 0), (3, 2, 1), (2, 1, 1), (4, 4, 2)])
def test_pool_exact(spk, L, s, p):
    T = 15
    lat = RNG.integers(0, T + 1, (2, 5, 14, 13)).astype(np.uint8)
    ref = oracle.dense_to_lat(oracle.pool(oracle.lat_to_dense(lat, T), (L, L), (s, s), (p, p)))
    np.testing.assert_array_equal(host(spk.pool(cu(lat), T, L, s, p)), ref)


# plane shapes of the large configs: C5 conv1 (16-byte rows: streaming 2x2 kernel; an odd item
# count), C4 conv1 (2-byte rows),
# many small planes per CTA, a plane too large for shared memory (global path), and
# narrow output rows (Wo < 16: one output per thread from shared memory)
@pytest.mark.parametrize("shape,L,s,p", [((2, 3, 224, 224), 2, 2, 0), ((3, 7, 64, 48), 2, 2, 0),
                                          ((1, 5, 160, 250), 2, 2, 0),
                                          ((3, 250, 14, 14), 3, 3, 0), ((1, 1, 300, 330), 2, 2, 1),
                                          ((2, 4, 50, 45), 3, 2, 1), ((2, 3, 64, 64), 8, 8, 0),
                                          ((2, 3, 61, 47), 5, 4, 2)])
def test_pool_exact_large_planes(spk, shape, L, s, p):
    T = 15
    lat = RNG.integers(0, T + 1, shape).astype(np.uint8)
    ref = oracle.dense_to_lat(oracle.pool(oracle.lat_to_dense(lat, T), (L, L), (s, s), (p, p)))
    np.testing.assert_array_equal(host(spk.pool(cu(lat), T, L, s, p)), ref)


# ----------------------------------------------------------------- a6 inhibit, a7 wta
def _records(B, T, C, H, W, dens=0.4, ties=False):
    P = np.cumsum(RNG.uniform(0, 1, (B, T, C, H, W)) * (RNG.random((B, 1, C, H, W)) < dens), axis=1)
    if ties:
        P = np.round(P * 4) / 4
    P = P.astype(np.float32).astype(np.float64)  # values representable in fp32: no rounding ambiguity
    Q = oracle.threshold(P, 1.2)
    lat, ps = lat_and_pstar(P, 1.2)
    return Q, lat, ps


@pytest.mark.parametrize("ties", [False, True])
def test_inhibit_exact(spk, ties):
    T = 10
    Q, lat, ps = _records(3, T, 6, 7, 8, 0.6, ties)
    ref = oracle.inhibit(Q)
    rlat, rps = lat_and_pstar(ref, 0.0)
    glat, gps = spk.inhibit(cu(lat), cu(ps.astype(np.float32)), T)
    np.testing.assert_array_equal(host(glat), rlat)
    np.testing.assert_array_equal(host(gps), rps.astype(np.float32))


@pytest.mark.parametrize("shape", [(4, 200, 4, 4), (2, 50, 5, 6), (3, 7, 1, 1)])
@pytest.mark.parametrize("ties", [False, True])
def test_inhibit_and_wta_small_maps(spk, shape, ties):
    """HW <= 32 (C2 layer 3: 200 maps of 4 x 4): the per-sample register inhibition kernel, and
    the one-warp WTA rounds on its <= HW surviving keys."""
    B, C, H, W = shape
    T = 15
    Q, lat, ps = _records(B, T, C, H, W, 0.5, ties)
    ref = oracle.inhibit(Q)
    rlat, rps = lat_and_pstar(ref, 0.0)
    glat, gps = spk.inhibit(cu(lat), cu(ps.astype(np.float32)), T)
    np.testing.assert_array_equal(host(glat), rlat)
    np.testing.assert_array_equal(host(gps), rps.astype(np.float32))
    for k, r in [(8, 1), (5, 3), (20, 0)]:
        win, nwin = oracle.wta(ref, k, r)
        gw, gn = spk.wta(glat, gps, T, k, r)
        gw, gn = host(gw), host(gn)
        np.testing.assert_array_equal(gn, nwin)
        for b in range(B):
            np.testing.assert_array_equal(gw[b, :nwin[b]], win[b, :nwin[b]])
            assert (gw[b, nwin[b]:] == -1).all()


# one C1-shaped sample (the small-grid rule: a few pixels per inhibition CTA, an 8-CTA WTA
# cluster) and a batch large enough to keep 256 pixels per CTA and the 16K-neuron clusters
@pytest.mark.parametrize("shape", [(1, 32, 28, 28), (2, 30, 28, 28), (160, 6, 20, 20)])
@pytest.mark.parametrize("ties", [False, True])
def test_inhibit_and_wta_grid_sizing(spk, shape, ties):
    B, C, H, W = shape
    T = 15
    Q, lat, ps = _records(B, T, C, H, W, 0.5, ties)
    ref = oracle.inhibit(Q)
    rlat, rps = lat_and_pstar(ref, 0.0)
    glat, gps = spk.inhibit(cu(lat), cu(ps.astype(np.float32)), T)
    np.testing.assert_array_equal(host(glat), rlat)
    np.testing.assert_array_equal(host(gps), rps.astype(np.float32))
    for k, r in [(5, 3), (8, 1)]:
        win, nwin = oracle.wta(ref, k, r)
        gw, gn = spk.wta(glat, gps, T, k, r)
        gw, gn = host(gw), host(gn)
        np.testing.assert_array_equal(gn, nwin)
        for b in range(B):
            np.testing.assert_array_equal(gw[b, :nwin[b]], win[b, :nwin[b]])


@pytest.mark.parametrize("ties", [False, True])
def test_inhibit_exact_large_maps(spk, ties):
    """HW >= 4096: the 4-pixels-per-thread register kernel (C4 shapes)."""
    T = 10
    Q, lat, ps = _records(2, T, 9, 64, 80, 0.5, ties)
    ref = oracle.inhibit(Q)
    rlat, rps = lat_and_pstar(ref, 0.0)
    glat, gps = spk.inhibit(cu(lat), cu(ps.astype(np.float32)), T)
    np.testing.assert_array_equal(host(glat), rlat)
    np.testing.assert_array_equal(host(gps), rps.astype(np.float32))


@pytest.mark.parametrize("k,r", [(5, 3), (8, 1), (1, 0), (3, 10), (20, 0)])
@pytest.mark.parametrize("ties", [False, True])
def test_wta_exact(spk, k, r, ties):
    T = 12
    Q, lat, ps = _records(4, T, 7, 9, 8, 0.5, ties)
    win, nwin = oracle.wta(Q, k, r)
    gw, gn = spk.wta(cu(lat), cu(ps.astype(np.float32)), T, k, r)
    gw, gn = host(gw), host(gn)
    np.testing.assert_array_equal(gn, nwin)
    for b in range(4):
        np.testing.assert_array_equal(gw[b, :nwin[b]], win[b, :nwin[b]])
        assert (gw[b, nwin[b]:] == -1).all()


# (C, H, W, k, r): a 2-CTA cluster keeping every live key; 8-CTA clusters with the
# per-pixel top-k pre-reduction (k=5 -> 8 kept, k=8 with a C4-like slice); a slice
# that overflows shared memory and re-reads its records every round (k=20)
@pytest.mark.parametrize("C,H,W,k,r", [(8, 50, 50, 5, 3), (40, 60, 70, 5, 3), (128, 40, 50, 8, 1),
                                       (40, 60, 70, 20, 2)])
@pytest.mark.parametrize("ties", [False, True])
def test_wta_exact_large_samples(spk, C, H, W, k, r, ties):
    T = 15
    Q, lat, ps = _records(2, T, C, H, W, 0.3, ties)
    win, nwin = oracle.wta(Q, k, r)
    gw, gn = spk.wta(cu(lat), cu(ps.astype(np.float32)), T, k, r)
    gw, gn = host(gw), host(gn)
    np.testing.assert_array_equal(gn, nwin)
    for b in range(2):
        np.testing.assert_array_equal(gw[b, :nwin[b]], win[b, :nwin[b]])


@pytest.mark.parametrize("C,H,W,k,r", [(1, 1, 1, 3, 0), (1000, 2, 2, 4, 1), (3, 1, 9000, 6, 2), (64, 3, 5, 64, 0)])
def test_wta_degenerate_shapes(spk, C, H, W, k, r):
    """Single neuron, many channels on a tiny map, one long row (8-CTA cluster with thin
    slices), k larger than the live count."""
    T = 9
    Q, lat, ps = _records(2, T, C, H, W, 0.4, True)
    win, nwin = oracle.wta(Q, k, r)
    gw, gn = spk.wta(cu(lat), cu(ps.astype(np.float32)), T, k, r)
    gw, gn = host(gw), host(gn)
    np.testing.assert_array_equal(gn, nwin)
    for b in range(2):
        np.testing.assert_array_equal(gw[b, :nwin[b]], win[b, :nwin[b]])
        assert (gw[b, nwin[b]:] == -1).all()


# ------------------------------------------------------------------------- a8 stdp
@pytest.mark.parametrize("stab", [1, 0])
def test_stdp_bit_exact(spk, stab):
    T, B, k = 15, 6, 4
    lat_in = RNG.integers(0, T + 1, (B, 5, 9, 8)).astype(np.uint8)
    W0 = RNG.uniform(0.0, 1.0, (7, 5, 3, 3)).astype(np.float32)
    W0[0, 0, 0, :] = [0.0, 1.0, 0.5]
    win = np.full((B, k, 6), -1, np.int32)
    nwin = RNG.integers(0, k + 1, B).astype(np.int32)
    for b in range(B):
        for q in range(nwin[b]):
            win[b, q] = [b, RNG.integers(0, T), RNG.integers(0, 7), RNG.integers(0, 9), RNG.integers(0, 8),
                         RNG.integers(0, 2)]
    cfgs = [(0.004, -0.003, 0.0, 1.0, stab), (-0.004, 0.003, 0.0, 1.0, stab)]
    ref = oracle.stdp(W0, oracle.lat_to_dense(lat_in, T), win, nwin, cfgs, (1, 1), (1, 1))
    w = cu(W0)
    spk.stdp(w, cu(lat_in), cu(win), cu(nwin), cfgs, T, 1, 1)
    np.testing.assert_array_equal(host(w), ref)


def test_rstdp_route_exact(spk):
    B, k = 9, 3
    win = np.full((B, k, 6), -1, np.int32)
    nwin = RNG.integers(0, k + 1, B).astype(np.int32)
    for b in range(B):
        for q in range(nwin[b]):
            win[b, q] = [b, 3, RNG.integers(0, 200), 1, 1, 0]
    labels = RNG.integers(0, 10, B).astype(np.int32)
    ref = oracle.rstdp_route(win, nwin, labels, 20)
    gw = cu(win)
    spk.rstdp_route(gw, cu(nwin), cu(labels), 20)
    np.testing.assert_array_equal(host(gw), ref)


# ---------------------------------------------------------------- a9 gather, boundary
def test_gather_and_conversions(spk):
    T = 15
    lat = RNG.integers(0, T + 1, (3, 4, 5, 6)).astype(np.uint8)
    S = oracle.lat_to_dense(lat, T)
    np.testing.assert_array_equal(host(spk.gather(cu(lat), T)), oracle.gather(S))
    np.testing.assert_array_equal(host(spk.lat_to_dense(cu(lat), T)), S)
    glat, bad = spk.dense_to_lat(cu(S))
    np.testing.assert_array_equal(host(glat), lat)
    assert int(host(bad)[0]) == -1
    S2 = S.copy()
    S2[1, 7, 2, 3, 4] = 0  # break the cumulative train of neuron (1, 2, 3, 4)
    S2[1, 8, 2, 3, 4] = 1
    if S2[1, 6, 2, 3, 4] == 0:
        S2[1, 6, 2, 3, 4] = 1
    _, bad = spk.dense_to_lat(cu(S2))
    assert int(host(bad)[0]) == 1 * 120 + 2 * 30 + 3 * 6 + 4


@pytest.mark.parametrize("T", [1, 15, 30, 254])
def test_gather_vectorised(spk, T):
    """16-byte path (n % 16 == 0, aligned): every latency 0..T and out-of-range values."""
    lat = RNG.integers(0, 256, (5, 8, 28, 28)).astype(np.uint8)
    lat[0, 0, 0, :T + 1] = np.arange(T + 1) if T < 28 else lat[0, 0, 0, :T + 1]
    ref = oracle.gather(oracle.lat_to_dense(np.minimum(lat, T), T))
    np.testing.assert_array_equal(host(spk.gather(cu(lat), T)), ref)


# ------------------------------------------------------------------ pipelines end to end
def _gpu_train(cfg, imgs, Ws, labels=None, prec="exact", fuse=True):
    from paper_2301_13659_b200.network import Network

    net = Network(cfg, imgs.shape[0], prec=prec, fuse_inhibit=fuse)
    net.img.copy_(cu(imgs))
    if labels is not None:
        net.labels.copy_(cu(labels))
    net.set_weights([cu(w) for w in Ws])
    net.train_step()
    torch.cuda.synchronize()
    return net


def _layer_out_diff(rec, L, rlat, excl, excluded, T, key=None):
    """GPU output of a non-trained layer vs the oracle's latencies: the latency map itself,
    or — when the layer's conv and pool run fused — the pooled map, a pooled neuron being
    excluded when a near-threshold neuron lies in its window (Eq. 3)."""
    if rec.get("fused_pool"):
        p = L["pool"]
        k, st, pd = (p["kernel"],) * 2, (p["stride"],) * 2, (p["pad"],) * 2
        rlat = oracle.dense_to_lat(oracle.pool(oracle.lat_to_dense(rlat, T), k, st, pd))
        excl = oracle.pool(excl[:, None].astype(np.uint8), k, st, pd)[:, 0].astype(bool)
        glat = host(rec["pooled"])
    else:
        glat = host(rec["lat"])
    if key is not None:
        keep = ~excluded
        ParityReport.latency(key, glat[keep], rlat[keep], excl[keep])
    diff = (glat != rlat) & ~excluded[:, None, None, None]
    assert not (diff & ~excl).any(), "unexplained latency mismatches"
    return diff.any(axis=(1, 2, 3))


def _check_pipeline(cfg, n, labels=False, prec="exact", fuse=True):
    name = f"{cfg['name']} train step, batch {n}, prec={prec}" + ("" if fuse else ", unfused inhibit")
    imgs = synth.images(cfg, 0, n)
    lab = synth.labels(cfg, 0, n) if labels else None
    Ws = synth.layer_weights(cfg)
    ref = opipe.train_step(cfg, imgs, Ws, lab, event=True)
    net = _gpu_train(cfg, imgs, Ws, lab, prec, fuse)
    T = cfg["T"]
    np.testing.assert_array_equal(host(net.lat0), ref["lat0"])
    tl = cfg["train_layer"]
    # layer inputs (teacher-free: whole chain on the GPU)
    excluded_samples = np.zeros(n, bool)
    for li in range(tl):
        L = cfg["layers"][li]
        P = oracle.conv_event(oracle.dense_to_lat(ref["inputs"][li]), T, Ws[li], (L["stride"],) * 2, (L["pad"],) * 2)
        excl = near_threshold(P, L["theta"])
        rlat, _ = lat_and_pstar(P, L["theta"])
        excluded_samples |= _layer_out_diff(net.layers[li], L, rlat, excl, excluded_samples, T,
                                            key=(name, f"conv{li} fire"))
    # trained layer: (lat, P*) after inhibition, winners, weights
    L = cfg["layers"][tl]
    excl = near_threshold(ref["P"], L["theta"])
    # fused inhibition+WTA leaves the fire record un-inhibited (only the winners carry it)
    rlat, rps = lat_and_pstar(ref["Q"] if net.fused_inhibit else ref["Qi"], 0.0)
    glat = host(net.layers[tl]["lat"])
    keep = ~excluded_samples
    ParityReport.latency((name, f"conv{tl} fire" + ("" if net.fused_inhibit else " + inhibit")), glat[keep], rlat[keep],
                         excl[keep])
    ParityReport.ties((name, f"conv{tl} inhibit"), *near_ties_inhibit(ref["Q"]))
    ParityReport.ties((name, f"conv{tl} wta"), *near_ties_wta(ref["Qi"], L["wta"]["count"], L["wta"]["radius"]))
    gps = host(net.layers[tl]["pstar"])
    okp = (glat == rlat) & (rlat < T) & keep[:, None, None, None]
    ParityReport.potentials((name, f"conv{tl} P*"), gps[okp], rps[okp])
    diff = (glat != rlat) & ~excluded_samples[:, None, None, None]
    assert not (diff & ~excl).any(), "trained layer: unexplained mismatches after inhibition"
    excluded_samples |= diff.any(axis=(1, 2, 3))
    gw, gn = host(net.win), host(net.nwin)
    for b in range(n):
        if excluded_samples[b]:
            continue
        assert gn[b] == ref["nwin"][b]
        np.testing.assert_array_equal(gw[b, :gn[b]], ref["win"][b, :gn[b]])
    ParityReport.excluded_samples((name, "samples"), int(excluded_samples.sum()))
    if not excluded_samples.any():
        np.testing.assert_array_equal(host(net.weights[tl]), ref["W_new"])
    else:
        # teacher-forced STDP with the GPU's own winners: still bit-exact
        S_in = oracle.lat_to_dense(host(net.input_of(tl)), T)
        W = oracle.stdp(Ws[tl], S_in, gw, gn, [tuple(c) for c in cfg["stdp"]], (L["stride"],) * 2, (L["pad"],) * 2)
        np.testing.assert_array_equal(host(net.weights[tl]), W)
    return int(excluded_samples.sum())


def test_pipeline_c1(spk):
    assert _check_pipeline(synth.load_config("c1"), 1) == 0


@pytest.mark.parametrize("prec", ["exact", "fp32", "auto", "event"])
def test_pipeline_c2_small_batch(spk, prec):
    assert _check_pipeline(synth.load_config("c2"), 12, prec=prec) <= 1


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_pipeline_unfused_inhibit(spk, name):
    """The unfused trained-layer path (spk_inhibit writes the inhibited record, then spk_wta)."""
    cfg = synth.load_config(name)
    assert _check_pipeline(cfg, 1 if name == "c1" else 12, labels=name == "c3", fuse=False) <= 1


def test_pipeline_c3_rstdp(spk):
    assert _check_pipeline(synth.load_config("c3"), 12, labels=True) <= 1


# a 64-image parity subset of the full C2 / C3 batch, spread over the batch
PARITY_ROWS_64 = [int(r) for r in np.linspace(0, 1023, 64)]


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_full_batch_sampled_64(spk, name):
    """BASELINE configs[1] (C2) and configs[2] (C3, R-STDP) at full size (batch 1024), launched
    exactly as bench.py does (auto engines, CUDA graph replay): 64 sampled images checked
    against the oracle stage by stage (front end bit-exact; every layer, inhibition and the
    winners outside the near-threshold set), and the STDP update of the whole batch checked
    bit-exactly with the GPU's winners teacher-forced."""
    from paper_2301_13659_b200.network import Network

    cfg = synth.load_config(name)
    B, T, tl = cfg["batch"], cfg["T"], cfg["train_layer"]
    imgs = synth.images_parallel(cfg, 0, B)
    lab = synth.labels(cfg, 0, B)
    Ws = synth.layer_weights(cfg)
    net = Network(cfg, B, prec="auto")
    net.img.copy_(cu(imgs))
    net.labels.copy_(cu(lab))
    net.set_weights([cu(w) for w in Ws])
    net.capture(warmup=1)
    net.set_weights([cu(w) for w in Ws])  # the capture warm-up ran one training step
    net.replay()
    torch.cuda.synchronize()
    assert _check_rows_train(cfg, net, imgs, PARITY_ROWS_64, Ws, labels=lab) <= 1
    gw, gn = host(net.win), host(net.nwin)
    L = cfg["layers"][tl]
    S_in = oracle.lat_to_dense(host(net.input_of(tl)), T)
    W = oracle.stdp(Ws[tl], S_in, gw, gn, [tuple(c) for c in cfg["stdp"]], (L["stride"],) * 2, (L["pad"],) * 2)
    np.testing.assert_array_equal(host(net.weights[tl]), W)


def _check_rows_train(cfg, net, imgs, rows, Ws, labels=None):
    """Rows of a full-batch GPU training step against the oracle, stage by stage and
    teacher-forced (every layer is per sample): the front end must be bit-exact; each
    layer's output must equal the oracle applied to the GPU's own input of that layer
    outside the near-threshold set; the trained layer's inhibited record and winners must
    equal the oracle's threshold -> inhibit -> convwta on the GPU's input (samples with an
    explained near-threshold mismatch in that layer are counted, not compared)."""
    T, tl = cfg["T"], cfg["train_layer"]
    name = f"{cfg['name']} full batch {net.B} (bench launch), {len(rows)} sampled rows"
    lat0, gw, gn = host(net.lat0), host(net.win), host(net.nwin)
    excluded = 0
    for b in rows:
        _, rl0 = opipe.front_end(cfg, imgs[b:b + 1])
        np.testing.assert_array_equal(lat0[b:b + 1], rl0)
        for li in range(tl):
            L = cfg["layers"][li]
            P = oracle.conv_event(host(net.input_of(li)[b:b + 1]), T, Ws[li], (L["stride"],) * 2, (L["pad"],) * 2)
            rlat, _ = lat_and_pstar(P, L["theta"])
            rec = dict(net.layers[li])
            for key in ("lat", "pooled"):
                if rec.get(key) is not None:
                    rec[key] = rec[key][b:b + 1]
            _layer_out_diff(rec, L, rlat, near_threshold(P, L["theta"]), np.zeros(1, bool), T,
                            key=(name, f"conv{li} fire"))
        L = cfg["layers"][tl]
        P = oracle.conv_event(host(net.input_of(tl)[b:b + 1]), T, Ws[tl], (L["stride"],) * 2, (L["pad"],) * 2)
        Q = oracle.threshold(P, L["theta"])
        Qi = oracle.inhibit(Q)
        win, nwin = oracle.wta(Qi, L["wta"]["count"], L["wta"]["radius"])
        if cfg["learning"] == "rstdp":
            win = oracle.rstdp_route(win, nwin, labels[b:b + 1], cfg["maps_per_class"])
        rlat, rps = lat_and_pstar(Q if net.fused_inhibit else Qi, 0.0)
        glat_b = host(net.layers[tl]["lat"][b:b + 1])
        diff = glat_b != rlat
        excl_b = near_threshold(P, L["theta"])
        ParityReport.latency((name, f"conv{tl} fire" + ("" if net.fused_inhibit else " + inhibit")), glat_b, rlat,
                             excl_b)
        ParityReport.ties((name, f"conv{tl} inhibit"), *near_ties_inhibit(Q))
        ParityReport.ties((name, f"conv{tl} wta"), *near_ties_wta(Qi, L["wta"]["count"], L["wta"]["radius"]))
        gps_b = host(net.layers[tl]["pstar"][b:b + 1])
        okp = (glat_b == rlat) & (rlat < T)
        ParityReport.potentials((name, f"conv{tl} P*"), gps_b[okp], rps[okp])
        assert not (diff & ~excl_b).any(), "trained layer: unexplained mismatches"
        del P, Q, Qi
        if diff.any():
            excluded += 1
            ParityReport.excluded_samples((name, "samples"), 1)
            continue
        assert gn[b] == nwin[0]
        got = gw[b, :gn[b]].copy()
        got[:, 0] = 0
        np.testing.assert_array_equal(got, win[0, :gn[b]])
    return excluded


def test_c4_full_batch_sampled(spk):
    """BASELINE configs[3] (C4) at full size — batch 256, T = 30 — launched as bench.py does
    (auto engines, CUDA graph replay); sampled images checked against the oracle one by one."""
    from paper_2301_13659_b200.network import Network

    cfg = synth.load_config("c4")
    B = cfg["batch"]
    imgs = synth.images_parallel(cfg, 0, B)
    Ws = synth.layer_weights(cfg)
    net = Network(cfg, B, prec="auto")
    net.img.copy_(cu(imgs))
    net.set_weights([cu(w) for w in Ws])
    net.capture(warmup=1)
    net.set_weights([cu(w) for w in Ws])  # the capture warm-up ran one training step
    net.replay()
    torch.cuda.synchronize()
    assert _check_rows_train(cfg, net, imgs, [0, 137, B - 1], Ws) <= 1


@pytest.mark.slow
def test_c5_full_batch_sampled(spk):
    """BASELINE configs[4] (C5) at full size — batch 4096 forward, as bench.py runs it at N = 1 —
    with the first and last image checked against the oracle (features bit-exact outside the
    near-threshold set)."""
    from paper_2301_13659_b200.network import Network

    cfg = synth.load_config("c5")
    B, T = cfg["batch"], cfg["T"]
    Ws = synth.layer_weights(cfg)
    net = Network(cfg, B, prec="auto")
    net.img.copy_(cu(synth.images_parallel(cfg, 0, B)))
    net.set_weights([cu(w) for w in Ws])
    net.capture(warmup=1)
    net.replay()
    torch.cuda.synchronize()
    for b in [0, B - 1]:
        img = synth.images(cfg, b, 1)
        _, lat = opipe.front_end(cfg, img)
        np.testing.assert_array_equal(host(net.lat0[b:b + 1]), lat)
        excluded = np.zeros(1, bool)
        for li, L in enumerate(cfg["layers"]):
            P = oracle.conv_event(lat, T, Ws[li], (L["stride"],) * 2, (L["pad"],) * 2)
            rlat, _ = lat_and_pstar(P, L["theta"])
            excl = near_threshold(P, L["theta"])
            del P
            rec = dict(net.layers[li])
            for key in ("lat", "pooled"):
                if rec.get(key) is not None:
                    rec[key] = rec[key][b:b + 1]
            excluded |= _layer_out_diff(rec, L, rlat, excl, excluded, T)
            p = L["pool"]
            lat = oracle.dense_to_lat(oracle.pool(oracle.lat_to_dense(rlat, T), (p["kernel"],) * 2,
                                                  (p["stride"],) * 2, (p["pad"],) * 2))
        if not excluded[0]:
            feats = oracle.gather(oracle.lat_to_dense(lat, T))
            np.testing.assert_array_equal(host(net.features[b:b + 1]), feats)


def test_pipeline_c4_train_t30(spk):
    """Caltech-shaped C4 (Gabor front end, T = 30 -> 32-row time tiles), layer-2 training step on
    2 images: end to end, then stage by stage with each layer teacher-forced on the GPU's own
    input (so a near-threshold flip in conv0 does not hide the trained layer from the check)."""
    from paper_2301_13659_b200.network import Network
    cfg = synth.load_config("c4")
    assert _check_pipeline(cfg, 2) <= 2
    imgs = synth.images(cfg, 0, 2)
    Ws = synth.layer_weights(cfg)
    net = Network(cfg, 2, prec="exact")
    net.img.copy_(cu(imgs))
    net.set_weights([cu(w) for w in Ws])
    net.train_step()
    torch.cuda.synchronize()
    assert _check_rows_train(cfg, net, imgs, [0, 1], Ws) <= 1


def _check_forward(cfg, n, prec="exact"):
    from paper_2301_13659_b200.network import Network

    imgs = synth.images(cfg, 0, n)
    Ws = synth.layer_weights(cfg)
    T = cfg["T"]
    net = Network(cfg, n, prec=prec)
    net.img.copy_(cu(imgs))
    net.set_weights([cu(w) for w in Ws])
    net.infer()
    torch.cuda.synchronize()
    name = f"{cfg['name']} forward, batch {n}, prec={prec}"
    _, lat0 = opipe.front_end(cfg, imgs)
    np.testing.assert_array_equal(host(net.lat0), lat0)
    lat = lat0
    excluded = np.zeros(n, bool)
    for li, L in enumerate(cfg["layers"]):
        P = oracle.conv_event(lat, T, Ws[li], (L["stride"],) * 2, (L["pad"],) * 2)
        rlat, _ = lat_and_pstar(P, L["theta"])
        excl = near_threshold(P, L["theta"])
        del P
        excluded |= _layer_out_diff(net.layers[li], L, rlat, excl, excluded, T, key=(name, f"conv{li} fire"))
        if L["pool"]:
            p = L["pool"]
            lat = oracle.dense_to_lat(oracle.pool(oracle.lat_to_dense(rlat, T), (p["kernel"],) * 2,
                                                  (p["stride"],) * 2, (p["pad"],) * 2))
            np.testing.assert_array_equal(host(net.layers[li]["pooled"])[~excluded], lat[~excluded])
        else:
            lat = rlat
    feats = oracle.gather(oracle.lat_to_dense(lat, T))
    np.testing.assert_array_equal(host(net.features)[~excluded], feats[~excluded])
    ParityReport.excluded_samples((name, "samples"), int(excluded.sum()))
    return int(excluded.sum())


@pytest.mark.slow
def test_pipeline_c5_forward(spk):
    """ImageNet-shaped C5 forward (3 conv layers of 128/256/512 maps, fp16-representable weights) + gather."""
    assert _check_forward(synth.load_config("c5"), 1) == 0


@pytest.mark.parametrize("prec", ["exact", "auto"])
def test_forward_c2_all_layers(spk, prec):
    assert _check_forward(synth.load_config("c2"), 6, prec) <= 1


# whole samples per CTA (overlapping and padded windows), and row chunks of a large map
# (fused when no window straddles a chunk)
@pytest.mark.parametrize("case", [(3, 15, 6, 28, 28, 30, 5, 1, 2, 2, 2, 0), (2, 15, 6, 28, 28, 30, 5, 1, 2, 3, 2, 1),
                                  (2, 30, 4, 20, 23, 40, 5, 1, 2, 2, 2, 0), (2, 7, 3, 9, 11, 20, 3, 2, 0, 3, 3, 0),
                                  (5, 15, 6, 27, 27, 30, 5, 1, 2, 2, 2, 0), (2, 30, 4, 160, 250, 64, 5, 1, 2, 2, 2, 0)])
def test_conv_fire_pool_fused(spk, case):
    """spk_conv_fire_pool == spk_pool(spk_conv(FIRE)) bit for bit (EVENT engine)."""
    B, T, Ci, Hi, Wi, Co, K, s, p, L, ps, pp = case
    lat, w = _conv_inputs(B, T, Ci, Hi, Wi, Co, K, 0.3)
    g = spk.conv_geom(cu(lat), cu(w), T, s, p)
    if not spk.conv_fire_pool_supported(g, "event", L, ps, pp):
        pytest.skip("fused fire+pool not supported for this geometry")
    P = oracle.conv_event(lat[:2], T, w, (s, s), (p, p))
    theta = float(np.percentile(P[:, -1], 60)) + 0.123
    flat, _ = spk.conv(cu(lat), cu(w), T, s, p, prec="event", epi="fire", theta=theta)
    ref = spk.pool(flat, T, L, ps, pp)
    got = spk.conv_fire_pool(cu(lat), cu(w), T, s, p, prec="event", theta=theta, pool_kernel=L, pool_stride=ps,
                             pool_pad=pp)
    np.testing.assert_array_equal(host(got), host(ref))


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_data_parallel_stdp_shards_equal_whole_batch(spk, name):
    """NEXT-2 on one GPU: two shards forwarded separately with the pre-batch weights, winners
    rebased to global sample indices (spk_winners_rebase) and concatenated in shard order,
    then one STDP over the global batch == the whole-batch train step, bit for bit (R-BATCH);
    and Network.enable_dp's exchange path (identity gather at world size 1) == train_step."""
    from paper_2301_13659_b200.network import Network
    cfg = synth.load_config(name)
    tl = cfg["train_layer"]
    n, half = 64, 32
    imgs, lab = synth.images(cfg, 0, n), synth.labels(cfg, 0, n)
    Ws = [torch.from_numpy(w) for w in synth.layer_weights(cfg)]

    def make(lo, hi):
        net = Network(cfg, hi - lo, prec="auto")
        net.img.copy_(torch.from_numpy(imgs[lo:hi]))
        net.labels.copy_(torch.from_numpy(lab[lo:hi]))
        net.set_weights(Ws)
        return net
    whole = make(0, n)
    whole.train_step()
    shards = [make(0, half), make(half, n)]
    for s, net in enumerate(shards):
        net.train_forward()
        spk.winners_rebase(net.win, net.nwin, s * half)
    g_win = torch.cat([net.win for net in shards])
    g_nwin = torch.cat([net.nwin for net in shards])
    g_lat = torch.cat([net.input_of(tl) for net in shards])
    L = cfg["layers"][tl]
    W = Ws[tl].clone().cuda()
    spk.stdp(W, g_lat, g_win, g_nwin, None, cfg["T"], L["stride"], L["pad"], cfg_arr=spk.stdp_configs(cfg["stdp"]))
    np.testing.assert_array_equal(host(W), host(whole.weights[tl]))
    assert int(host(g_nwin).sum()) == int(host(whole.nwin).sum()) > 0
    dp = make(0, n)
    dp.enable_dp(0, n, lambda dst, src: dst.copy_(src))
    dp.train_step()
    np.testing.assert_array_equal(host(dp.weights[tl]), host(whole.weights[tl]))


def test_data_parallel_stdp_matches_oracle_global_batch(spk):
    """NEXT-2 (R-BATCH) against the ORACLE: two replicas forward their shards, exchange
    winners + trained-layer inputs (Network.enable_dp with an in-process all-gather standing in
    for NCCL), and apply one sequential update; the result equals oracle.stdp applied with the
    oracle's own global-batch winners (bit-exact), or — when a near-threshold neuron changed a
    sample's winners — the oracle's update with the GPU winners teacher-forced."""
    from paper_2301_13659_b200.network import Network
    cfg = synth.load_config("c2")
    tl, T = cfg["train_layer"], cfg["T"]
    L = cfg["layers"][tl]
    n, half = 32, 16
    imgs = synth.images(cfg, 0, n)
    Ws = synth.layer_weights(cfg)
    ref = opipe.train_step(cfg, imgs, Ws, None, event=True)
    nets = []
    for s in range(2):
        net = Network(cfg, half, prec="auto")
        net.img.copy_(cu(imgs[s * half:(s + 1) * half]))
        net.set_weights([cu(w) for w in Ws])
        nets.append(net)
    # forward both shards with the pre-batch weights; the rank-ordered concatenation of the
    # shards' winners and trained-layer inputs is what NCCL's all-gather hands every replica
    for s, net in enumerate(nets):
        net.enable_dp(s * half, n, None)
        net.train_forward()
        spk.winners_rebase(net.win, net.nwin, s * half)
    g_win = torch.cat([net.win for net in nets])
    g_nwin = torch.cat([net.nwin for net in nets])
    g_lat = torch.cat([net.input_of(tl) for net in nets])
    for net in nets:
        spk.stdp(net.weights[tl], g_lat, g_win, g_nwin, None, T, L["stride"], L["pad"], ws=net.stdp_ws,
                 cfg_arr=net.stdp_cfg)
    w0, w1 = host(nets[0].weights[tl]), host(nets[1].weights[tl])
    np.testing.assert_array_equal(w0, w1)  # replicas stay bit-identical with no broadcast
    gw, gn = host(g_win), host(g_nwin)
    bad = [b for b in range(n) if gn[b] != ref["nwin"][b] or not (gw[b, :gn[b]] == ref["win"][b, :gn[b]]).all()]
    ParityReport.excluded_samples(("C2 data-parallel STDP (2 replicas x 16)", "samples"), len(bad))
    assert len(bad) <= 1, f"winners differ from the oracle's global batch in samples {bad}"
    if not bad:
        np.testing.assert_array_equal(w0, ref["W_new"])
    else:
        S_in = oracle.lat_to_dense(host(g_lat), T)
        W = oracle.stdp(Ws[tl], S_in, gw, gn, [tuple(c) for c in cfg["stdp"]], (L["stride"],) * 2, (L["pad"],) * 2)
        np.testing.assert_array_equal(w0, W)


def _train_outputs(net):
    torch.cuda.synchronize()
    outs = [host(net.lat0), host(net.win), host(net.nwin)] + [host(w) for w in net.weights]
    for rec in net.layers:
        for key in ("lat", "pstar", "pooled"):
            if rec.get(key) is not None:
                outs.append(host(rec[key]))
    return outs


@pytest.mark.parametrize("name,batch", [("c2", 1024), ("c3", 1024), ("c4", 8)])
def test_run_twice_bitwise_deterministic(spk, name, batch):
    """SURVEY §4.2 T4 / §8(b) "Determinism": the same step run twice from the same state (CUDA
    graph replay, bench engines) gives bit-identical latencies, P*, winners and weights."""
    from paper_2301_13659_b200.network import Network
    cfg = synth.load_config(name)
    imgs = synth.images_parallel(cfg, 0, batch)
    Ws = [cu(w) for w in synth.layer_weights(cfg)]
    net = Network(cfg, batch, prec="auto")
    net.img.copy_(cu(imgs))
    net.labels.copy_(cu(synth.labels(cfg, 0, batch)))
    net.capture(warmup=1)
    runs = []
    for _ in range(2):
        net.set_weights(Ws)
        net.replay()
        runs.append(_train_outputs(net))
    for a, b in zip(*runs):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("name,batch", [("c2", 32), ("c3", 16), ("c1", 1)])
def test_host_io_graph_equals_copies_around_step(spk, name, batch):
    """Network.capture_io (the host-to-host step bench.py's e2e times: copies in, the step, copies
    out as one CUDA graph) gives the same winners and weights as explicit copies around step()."""
    import torch
    from paper_2301_13659_b200.network import Network
    cfg = synth.load_config(name)
    h_img = torch.from_numpy(synth.images_parallel(cfg, 0, batch)).pin_memory()
    h_lab = torch.from_numpy(synth.labels(cfg, 0, batch)).pin_memory()
    Ws = [cu(w) for w in synth.layer_weights(cfg)]
    outs = []
    for use_io in (False, True):
        net = Network(cfg, batch, prec="auto")
        net.set_weights(Ws)
        h_win = torch.empty(net.win.shape, dtype=torch.int32).pin_memory()
        h_nwin = torch.empty(net.nwin.shape, dtype=torch.int32).pin_memory()
        io_in, io_out = [(net.img, h_img), (net.labels, h_lab)], [(h_win, net.win), (h_nwin, net.nwin)]
        if use_io:
            net.capture_io(io_in, io_out)
            net.set_weights(Ws)  # the capture ran no step: weights are still the initial ones
            net.replay_io()
        else:
            for dst, src in io_in:
                dst.copy_(src, non_blocking=True)
            net.step()
            for dst, src in io_out:
                dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        tl = cfg["train_layer"]
        outs.append((h_win.numpy().copy(), h_nwin.numpy().copy(), host(net.weights[tl])))
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("name,batch,shards", [("c5", 8, 2), ("c5", 12, 4), ("c2", 64, 2), ("c4", 6, 3)])
def test_sharded_forward_bitwise_equals_whole_batch(spk, name, batch, shards):
    """SURVEY §8(e) test: the batched forward split into contiguous image shards (rank g gets
    parallel.shard_range) — each shard generated from its global indices and forwarded
    separately — concatenates to exactly the whole-batch output, bit for bit."""
    from paper_2301_13659_b200 import parallel
    from paper_2301_13659_b200.network import Network
    cfg = synth.load_config(name)
    Ws = [cu(w) for w in synth.layer_weights(cfg)]

    def run(start, n):
        net = Network(cfg, n, prec="auto")
        net.img.copy_(cu(synth.images_parallel(cfg, start, n)))
        net.set_weights(Ws)
        net.infer()
        torch.cuda.synchronize()
        return host(net.features), host(net.lat0)

    whole_f, whole_l = run(0, batch)
    parts = [run(*parallel.shard_range(batch, shards, g)) for g in range(shards)]
    np.testing.assert_array_equal(np.concatenate([p[1] for p in parts]), whole_l)
    np.testing.assert_array_equal(np.concatenate([p[0] for p in parts]), whole_f)


@pytest.mark.parametrize("case", CONV_CASES)
@pytest.mark.parametrize("wkind", ["fp16", "binary", "zero", "digit0_only"])
def test_conv_live_digit_planes(spk, case, wkind):
    """The tcgen05 conv issues MMAs only for digit planes with a non-zero digit (fp16-representable
    weights: planes 1-2; binary {0,1}: plane 2; all-zero weights; weights with only the lowest
    digit): potentials and fire records equal the event form (which has no planes) bit for bit and
    the oracle within the fp32 protocol; prepacked weights give the same outputs."""
    B, T, Ci, Hi, Wi, Co, K, s, p = case
    lat, w = _conv_inputs(B, T, Ci, Hi, Wi, Co, K)
    if wkind == "fp16":
        w = w.astype(np.float16).astype(np.float32)
    elif wkind == "binary":
        w = oracle.quantize(w, 0, 0.5, 1)
    elif wkind == "zero":
        w[:] = 0
    else:
        w = (np.floor(w * 255) * 2.0 ** -23).astype(np.float32)  # q = 0..255: only digit 0
    ref = oracle.conv_event(lat, T, w, (s, s), (p, p))
    got = host(spk.conv(cu(lat), cu(w), T, s, p, prec="exact", epi="potential"))
    assert_potentials(got, ref)
    theta = float(np.percentile(ref[:, -1], 60)) + 1e-7
    xl, xp = spk.conv(cu(lat), cu(w), T, s, p, prec="exact", epi="fire", theta=theta)
    g = spk.conv_geom(cu(lat), cu(w), T, s, p)
    ws = torch.empty(spk.conv_workspace(g, "exact"), dtype=torch.uint8, device="cuda")
    spk.conv_prepack(cu(w), g, "exact", 1.0, ws)
    pl, pp = spk.conv(cu(lat), cu(w) * 0 + 7, T, s, p, prec="exact", epi="fire", theta=theta, ws=ws, prepacked=True)
    np.testing.assert_array_equal(host(pl), host(xl))
    np.testing.assert_array_equal(host(pp), host(xp))
    if spk.conv_workspace(g, "event") > 0:
        el, ep = spk.conv(cu(lat), cu(w), T, s, p, prec="event", epi="fire", theta=theta)
        np.testing.assert_array_equal(host(el), host(xl))
        np.testing.assert_array_equal(host(ep), host(xp))


@pytest.mark.parametrize("shape,k,r", [((4, 200, 4, 4), 8, 1), ((2, 30, 28, 28), 5, 3), ((1, 32, 28, 28), 5, 3),
                                       ((2, 128, 80, 125), 8, 1), ((3, 7, 1, 1), 3, 0), ((2, 64, 30, 40), 20, 2),
                                       ((2, 20, 33, 35), 6, 2)])
@pytest.mark.parametrize("ties", [False, True])
def test_inhibit_wta_fused_exact(spk, shape, k, r, ties):
    """spk_inhibit_wta == oracle inhibit -> wta (winners bit-exact), records left untouched."""
    B, C, H, W = shape
    T = 15
    Q, lat, ps = _records(B, T, C, H, W, 0.4, ties)
    win, nwin = oracle.wta(oracle.inhibit(Q), k, r)
    glat, gps = cu(lat), cu(ps.astype(np.float32))
    gw, gn = spk.inhibit_wta(glat, gps, T, k, r)
    gw, gn = host(gw), host(gn)
    np.testing.assert_array_equal(gn, nwin)
    for b in range(B):
        np.testing.assert_array_equal(gw[b, :nwin[b]], win[b, :nwin[b]])
        assert (gw[b, nwin[b]:] == -1).all()
    np.testing.assert_array_equal(host(glat), lat)


def test_stdp_invalid_winners_counted(spk):
    """Out-of-range winners (coordinate or cfg) are skipped and counted (spk_stdp_status)."""
    T, B, k = 15, 2, 3
    lat_in = RNG.integers(0, T + 1, (B, 2, 6, 6)).astype(np.uint8)
    W0 = RNG.uniform(0.1, 0.9, (4, 2, 3, 3)).astype(np.float32)
    win = np.full((B, k, 6), -1, np.int32)
    win[0, 0] = [0, 3, 1, 2, 2, 0]     # valid
    win[0, 1] = [0, 3, 9, 2, 2, 0]     # map out of range
    win[1, 0] = [1, 3, 1, 2, 2, 5]     # cfg out of range
    win[1, 1] = [1, 3, 1, 2, 7, 0]     # x out of range
    nwin = np.array([2, 2], np.int32)
    cfgs = [(0.004, -0.003, 0.0, 1.0, 1)]
    # the only valid winner is (sample 0, pick 0): the oracle applies just that one
    ref = oracle.stdp(W0, oracle.lat_to_dense(lat_in[:1], T), win[:1, :1], np.ones(1, np.int32), cfgs, (1, 1), (1, 1))
    w = cu(W0)
    g = spk.conv_geom(cu(lat_in), w, T, 1, 1)
    ws = torch.empty(spk.stdp_workspace(g, k), dtype=torch.uint8, device="cuda")
    spk.stdp(w, cu(lat_in), cu(win), cu(nwin), cfgs, T, 1, 1, ws=ws)
    assert spk.stdp_invalid(ws, cu(lat_in), w, T, k, 1, 1) == 3
    np.testing.assert_array_equal(host(w), ref)
