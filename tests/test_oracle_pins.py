"""Pins for the CPU oracle against what the paper and mathematics fix (no GPU).

Each test names the passage (P:Lnn of /root/reference/PAPER.md) or the closed
form it checks.  None of these re-types the oracle's formula: they check
closed forms, invariants, hand-worked numbers, library special cases, or an
independently written brute force on tiny inputs.
"""
import math

import numpy as np
import pytest
from scipy import signal

import oracle
import synth
from oracle import pipeline

RNG = np.random.default_rng(1234)


# ------------------------------------------------------------------ filters (O2, O3)
@pytest.mark.parametrize("s1,s2", [(1.0, 2.0), (2.0, 1.0), (0.471 * 2 ** .5, 0.471 / 2 ** .5), (1.5, 3.0)])
def test_dog_zero_sum_and_antisymmetry(s1, s2):
    # P:L72 DoG of unit-sum Gaussians sums to 0; swapping the sigmas negates.
    k = oracle.dog_kernel(s1, s2, 3).astype(np.float64)
    assert abs(k.sum()) < 1e-6
    np.testing.assert_array_equal(oracle.dog_kernel(s2, s1, 3), -oracle.dog_kernel(s1, s2, 3))
    # centre-surround: on-centre iff sigma1 < sigma2
    assert (k[3, 3] > 0) == (s1 < s2)
    # isotropy: the kernel is invariant under the 8 symmetries of the square
    for kk in (k.T, k[::-1], k[:, ::-1], np.rot90(k)):
        np.testing.assert_allclose(kk, k, atol=1e-9)


def test_gaussian_ratio_closed_form():
    # G(1,0)/G(0,0) = exp(-1/(2 sigma^2)) for a Gaussian; read it off DoG(s, big) where the
    # big-sigma term is almost flat: DoG(s, inf) -> G_s - 1/49.  Use the exact difference
    # of two kernels with a shared second sigma instead: D1 - D2 = G_a - G_b.
    a, b, c = 1.3, 0.9, 2.5
    g_diff = oracle.dog_kernel(a, c, 3).astype(np.float64) - oracle.dog_kernel(b, c, 3).astype(np.float64)
    ys, xs = np.mgrid[-3:4, -3:4]

    def unit_gauss(s):
        g = np.exp(-(xs ** 2 + ys ** 2) / (2 * s * s))
        return g / g.sum()

    np.testing.assert_allclose(g_diff, unit_gauss(a) - unit_gauss(b), atol=2e-7)


def test_gabor_closed_forms():
    # P:L76 Gabor: centre = cos(psi); theta and theta+pi agree for psi=0; psi=theta=0 is y-symmetric.
    for psi in (0.0, 0.3, 1.0, math.pi / 2):
        g = oracle.gabor_kernel(2.8, 0.7, 0.5, 5.0, psi, 3)
        assert g[3, 3] == np.float32(math.cos(psi))
    np.testing.assert_allclose(oracle.gabor_kernel(2.8, 0.4, 0.5, 5.0, 0.0, 3),
                               oracle.gabor_kernel(2.8, 0.4 + math.pi, 0.5, 5.0, 0.0, 3), atol=1e-6)
    g0 = oracle.gabor_kernel(2.8, 0.0, 0.5, 5.0, 0.0, 3)
    np.testing.assert_array_equal(g0, g0[::-1, :])
    # theta = 0: along the x axis (y = 0) the envelope is exp(-x^2/2s^2) and the carrier cos(2 pi x/lam)
    x = np.arange(-3, 4)
    np.testing.assert_allclose(g0[3], np.exp(-x ** 2 / (2 * 2.8 ** 2)) * np.cos(2 * np.pi * x / 5.0), atol=1e-6)
    # theta = pi/2 rotates the kernel by 90 degrees
    g90 = oracle.gabor_kernel(2.8, math.pi / 2, 0.5, 5.0, 0.0, 3)
    np.testing.assert_allclose(g90, g0.T, atol=1e-6)


@pytest.mark.parametrize("gamma", [0.5, 1.0, 2.0])
@pytest.mark.parametrize("psi", [0.0, 0.4])
def test_gabor_gamma_off_axis_closed_form(gamma, psi):
    # at theta = 0, x' = x and y' = y, so on the column x = 0 the carrier is
    # cos(psi) and the envelope exp(-gamma^2 y^2 / (2 sigma^2)).  This fixes gamma SQUARED on
    # the y' term (gamma = 0.5 and 2 separate gamma from gamma^2; gamma = 1 checks the sigma),
    # and that y runs along the kernel rows (index r + y).
    sigma, r = 2.8, 3
    g = oracle.gabor_kernel(sigma, 0.0, gamma, 5.0, psi, r).astype(np.float64)
    for y in range(-r, r + 1):
        expect = math.exp(-(gamma ** 2) * y * y / (2 * sigma ** 2)) * math.cos(psi)
        assert abs(g[r + y, r] - expect) < 1e-6, (gamma, y)
    # rotating by theta = pi/2 moves that column onto the row y = 0: g(x, 0) = exp(-gamma^2 x^2/2s^2) cos(psi)
    g90 = oracle.gabor_kernel(sigma, math.pi / 2, gamma, 5.0, psi, r).astype(np.float64)
    for x in range(-r, r + 1):
        expect = math.exp(-(gamma ** 2) * x * x / (2 * sigma ** 2)) * math.cos(psi)
        assert abs(g90[r, r + x] - expect) < 1e-6, (gamma, x)


def test_log_pair_order():
    # LoG(sigma) = (DoG(sigma*sqrt2, sigma/sqrt2), DoG(sigma/sqrt2, sigma*sqrt2)) in this
    # order.  The first DoG subtracts the narrower Gaussian (sigma2 = sigma/sqrt2 < sigma1), so its
    # centre is NEGATIVE (off-centre) and the second's positive (centre > 0 iff s1 < s2).
    for s in (0.471, 1.099, 2.042):
        k = oracle.log_kernels([s], 3)
        assert k[0, 3, 3] < 0 < k[1, 3, 3], s
        # the centre is the extreme of each kernel: the most negative / most positive tap
        assert k[0, 3, 3] == k[0].min() and k[1, 3, 3] == k[1].max()
    # list order is kept: stds [a, b] -> [pair(a), pair(b)] (R-CHORDER)
    ka, kb = oracle.log_kernels([0.471], 3), oracle.log_kernels([2.042], 3)
    np.testing.assert_array_equal(oracle.log_kernels([0.471, 2.042], 3), np.concatenate([ka, kb]))


def test_log_six_channels_pairs_negate():
    # Listing 1: 3 LoG stds -> 6 channels; each pair is an exact negation.
    k = oracle.log_kernels([0.471, 1.099, 2.042], 3)
    assert k.shape == (6, 7, 7)
    for q in range(3):
        np.testing.assert_array_equal(k[2 * q], -k[2 * q + 1])
    img = RNG.integers(0, 256, (2, 1, 28, 28), dtype=np.uint8)
    assert oracle.filter_apply(img, k, 3).shape == (2, 6, 28, 28)


def test_filter_delta_kernel_is_crop():
    img = RNG.integers(0, 256, (1, 2, 9, 11), dtype=np.uint8)
    k = np.zeros((1, 5, 5), np.float32)
    k[0, 2, 2] = 1.0
    out = oracle.filter_apply(img, k, 0)  # Eq. 1: 9+0-5+1 = 5, 11-4 = 7
    assert out.shape == (1, 2, 5, 7)
    np.testing.assert_array_equal(out, (img[:, :, 2:7, 2:9].astype(np.float32) / np.float32(255)))


def test_filter_matches_library_correlation():
    # Eq. 1 depthwise filtering == scipy correlate2d (zero fill) per channel and kernel.
    img = RNG.integers(0, 256, (2, 3, 13, 10), dtype=np.uint8)
    k = RNG.normal(0, 1, (4, 7, 7)).astype(np.float32)
    for pad in (0, 2, 3):
        out = oracle.filter_apply(img, k, pad)
        for b in range(2):
            for c in range(3):
                x = np.pad(img[b, c].astype(np.float64) / 255.0, pad)
                for q in range(4):
                    ref = signal.correlate2d(x, k[q].astype(np.float64), mode="valid")
                    np.testing.assert_allclose(out[b, c * 4 + q], ref, rtol=1e-5, atol=1e-5)


def test_eq1_shape_law_random():
    for _ in range(40):
        H, W, r = int(RNG.integers(1, 12)), int(RNG.integers(1, 12)), int(RNG.integers(0, 3))
        pad = int(RNG.integers(0, 4))
        if H + 2 * pad < 2 * r + 1 or W + 2 * pad < 2 * r + 1:
            continue
        C, K = int(RNG.integers(1, 3)), int(RNG.integers(1, 3))
        out = oracle.filter_apply(np.zeros((1, C, H, W), np.uint8), np.ones((K, 2 * r + 1, 2 * r + 1), np.float32), pad)
        assert out.shape == (1, C * K, H + 2 * pad - 2 * r, W + 2 * pad - 2 * r)


# -------------------------------------------------------------------- coding (O4, O5)
def test_threshold_examples():
    # [0.5, 0.005, 0.2] at 0.01 -> [0.5, 0, 0.2]; strict: 0.01 itself is zeroed.
    np.testing.assert_array_equal(oracle.threshold(np.array([0.5, 0.005, 0.2, 0.01], np.float32), 0.01),
                                  np.array([0.5, 0, 0.2, 0], np.float32))


def test_rank_code_hand_examples():
    # values [4,3,2,1], T=4 -> first spikes [0,1,2,3]; dense step 2 = [1,1,1,0].
    lat = oracle.rank_code(np.array([[4, 3, 2, 1]], np.float32), 4, 0.0)
    np.testing.assert_array_equal(lat, [[0, 1, 2, 3]])
    np.testing.assert_array_equal(oracle.lat_to_dense(lat, 4)[0, 2], [1, 1, 1, 0])
    # sort disabled: linear binning of the same values gives the same bins here.
    np.testing.assert_array_equal(oracle.rank_code(np.array([[4, 3, 2, 1]], np.float32), 4, 0.0, sort=False),
                                  [[0, 1, 2, 3]])
    # all zero (or below threshold) -> never fires
    np.testing.assert_array_equal(oracle.rank_code(np.zeros((1, 5), np.float32), 7, 0.01), [[7] * 5])
    np.testing.assert_array_equal(oracle.rank_code(np.full((1, 3), 0.01, np.float32), 7, 0.01), [[7] * 3])
    # ties broken by flat index: equal values spread over bins in index order
    np.testing.assert_array_equal(oracle.rank_code(np.ones((1, 4), np.float32), 4, 0.0), [[0, 1, 2, 3]])


def _brute_rank(v):
    n = len(v)
    pos = [i for i in range(n) if v[i] > 0]
    r = {}
    for i in pos:
        r[i] = sum(1 for j in pos if v[j] > v[i] or (v[j] == v[i] and j < i))
    return r, len(pos)


@pytest.mark.parametrize("T", [1, 4, 15, 30])
def test_rank_code_brute_force_and_invariants(T):
    for trial in range(20):
        n = int(RNG.integers(1, 60))
        v = RNG.normal(0, 1, n).astype(np.float32)
        v[RNG.random(n) < 0.2] = 0.0
        if trial % 3 == 0:  # force ties
            v = np.round(v * 2) / 2
        lat = oracle.rank_code(v[None], T, 0.0)[0]
        r, npos = _brute_rank(v)
        for i in range(n):
            if i in r:
                # bins of equal size up to one, earlier bins = higher intensity
                assert lat[i] == (r[i] * T) // npos
            else:
                assert lat[i] == T
        # each input spikes at most once and stays on: the dense train is cumulative
        S = oracle.lat_to_dense(lat[None], T)[0]
        assert np.all(np.diff(S.astype(int), axis=0) >= 0)
        np.testing.assert_array_equal(oracle.dense_to_lat(S[None])[0], lat)
        # monotone: v_i > v_j > 0 => lat_i <= lat_j
        for i in range(n):
            for j in range(n):
                if v[i] > v[j] > 0:
                    assert lat[i] <= lat[j]
        # bin sizes differ by at most one
        if npos:
            sizes = np.bincount(lat[lat < T], minlength=T)
            assert sizes.max() - sizes.min() <= 1 or npos < T
        # positive-scale invariance: multiplying by a power of two is exact
        np.testing.assert_array_equal(oracle.rank_code((v * 4)[None], T, 0.0)[0], lat)


def test_rank_code_sort_off_properties():
    # Sort disabled: latency is monotone non-increasing in intensity, max -> 0, min -> T-1 region.
    for _ in range(20):
        v = RNG.uniform(0.02, 1.0, 50).astype(np.float32)
        lat = oracle.rank_code(v[None], 15, 0.01, sort=False)[0]
        order = np.argsort(-v, kind="stable")
        assert np.all(np.diff(lat[order].astype(int)) >= 0)
        assert lat[np.argmax(v)] == 0
        assert lat[np.argmin(v)] == 14


# ----------------------------------------------------------------------- conv (O6)
def _brute_conv(S, W, s, p):
    B, T, Ci, Hi, Wi = S.shape
    Co, _, Kh, Kw = W.shape
    Ho, Wo = (Hi + 2 * p - Kh) // s + 1, (Wi + 2 * p - Kw) // s + 1
    out = np.zeros((B, T, Co, Ho, Wo))
    Sp = np.zeros((B, T, Ci, Hi + 2 * p, Wi + 2 * p))
    Sp[:, :, :, p:p + Hi, p:p + Wi] = S
    for y in range(Ho):
        for x in range(Wo):
            patch = Sp[:, :, :, y * s:y * s + Kh, x * s:x * s + Kw]  # B T Ci Kh Kw
            out[:, :, :, y, x] = np.tensordot(patch, W.astype(np.float64), axes=([2, 3, 4], [1, 2, 3]))
    return out


@pytest.mark.parametrize("s,p,K", [(1, 2, 5), (1, 1, 3), (2, 0, 3), (3, 0, 4), (2, 1, 2)])
def test_conv_brute_force_and_event_form(s, p, K):
    T = 5
    lat = RNG.integers(0, T + 1, (2, 3, 8, 7)).astype(np.uint8)
    S = oracle.lat_to_dense(lat, T)
    W = RNG.uniform(0, 1, (4, 3, K, K)).astype(np.float32)
    P = oracle.conv(S, W, (s, s), (p, p))
    np.testing.assert_allclose(P, _brute_conv(S, W, s, p), rtol=1e-12, atol=1e-12)
    # event form (independent derivation, P:L64 + P:L117) agrees
    np.testing.assert_allclose(oracle.conv_event(lat, T, W, (s, s), (p, p)), P, rtol=1e-12, atol=1e-12)
    # non-negative weights + cumulative input => potentials nondecreasing in t
    assert np.all(np.diff(P, axis=1) >= 0)


def test_conv_eq2_shapes_and_delta():
    # Eq. 2: 28, K5, P2 -> 28 (Listing 2 conv1); 28, K4, P0, S3 -> 9
    assert oracle.conv_out_hw(28, 28, 5, 5, 1, 1, 2, 2) == (28, 28)
    assert oracle.conv_out_hw(28, 28, 4, 4, 3, 3, 0, 0) == (9, 9)
    S = np.zeros((1, 1, 1, 7, 7), np.uint8)
    S[0, 0, 0, 3, 3] = 1
    W = np.arange(9, dtype=np.float32).reshape(1, 1, 3, 3)
    P = oracle.conv(S, W, (1, 1), (1, 1))[0, 0, 0]
    # cross-correlation of a delta gives the flipped kernel footprint around (3,3)
    np.testing.assert_array_equal(P[2:5, 2:5], W[0, 0, ::-1, ::-1])
    assert P.sum() == W.sum()


def test_conv_integer_weights_exact_and_time_permutation():
    lat = RNG.integers(0, 7, (1, 2, 6, 6)).astype(np.uint8)
    S = oracle.lat_to_dense(lat, 6)
    W = RNG.integers(0, 2, (3, 2, 3, 3)).astype(np.float32)  # quantised (Listing 4) weights
    P = oracle.conv(S, W, (1, 1), (1, 1))
    np.testing.assert_array_equal(P, np.round(P))
    perm = RNG.permutation(6)
    np.testing.assert_array_equal(oracle.conv(S[:, perm], W, (1, 1), (1, 1)), P[:, perm])


# ------------------------------------------------------------------ fire / pool (O7, O8)
def test_fire_examples():
    P = np.array([16.0, 15.9, 16.0000001, 0.0])
    np.testing.assert_array_equal(oracle.fire(P, 16.0), [0, 0, 1, 0])  # strict "higher than"
    Pt = np.cumsum(RNG.uniform(0, 3, (10, 50)), axis=0)  # nondecreasing over t
    S = oracle.fire(Pt, 7.0)
    assert np.all(np.diff(S.astype(int), axis=0) >= 0)
    lat = oracle.dense_to_lat(S.T[:, :, None])  # [50][T] -> first spike
    np.testing.assert_array_equal(lat[:, 0] == 10, Pt[-1] <= 7.0)


def test_pool_examples_and_min_latency_form():
    assert oracle.pool(np.zeros((1, 1, 1, 28, 28), np.uint8), (2, 2)).shape == (1, 1, 1, 14, 14)
    # window with first spikes {2, 5} -> 2
    lat = np.array([[[[2, 5]]]], np.uint8)
    out = oracle.dense_to_lat(oracle.pool(oracle.lat_to_dense(lat, 8), (1, 2)))
    assert out.ravel().tolist() == [2]
    # max over each t of cumulative trains == min latency over the window (zero pad = never)
    for (L, s, p) in [(2, 2, 0), (3, 3, 0), (3, 2, 1), (2, 1, 1)]:
        lat = RNG.integers(0, 9, (2, 3, 7, 8)).astype(np.uint8)
        got = oracle.dense_to_lat(oracle.pool(oracle.lat_to_dense(lat, 8), (L, L), (s, s), (p, p)))
        padl = np.pad(lat, ((0, 0), (0, 0), (p, p), (p, p)), constant_values=8)
        Ho, Wo = (7 + 2 * p - L) // s + 1, (8 + 2 * p - L) // s + 1
        ref = np.empty((2, 3, Ho, Wo), np.uint8)
        for y in range(Ho):
            for x in range(Wo):
                ref[:, :, y, x] = padl[:, :, y * s:y * s + L, x * s:x * s + L].min(axis=(2, 3))
        np.testing.assert_array_equal(got, ref)


# ----------------------------------------------------------------- inhibit / WTA (O9, O10)
def _rand_Q(B, T, C, H, W, dens=0.3):
    P = np.cumsum(RNG.uniform(0, 1, (B, T, C, H, W)) * (RNG.random((B, 1, C, H, W)) < dens), axis=1)
    return oracle.threshold(P, 1.5)


def test_inhibit_properties():
    Q = _rand_Q(2, 6, 1, 5, 5)
    np.testing.assert_array_equal(oracle.inhibit(Q), Q)  # single channel unchanged
    Q = _rand_Q(2, 6, 5, 5, 5, 0.6)
    Qi = oracle.inhibit(Q)
    np.testing.assert_array_equal(oracle.inhibit(Qi), Qi)  # idempotent
    fired = (Qi > 0).any(axis=1)  # B C H W
    assert fired.sum(axis=1).max() <= 1
    # hand case: channel 0 crosses at t=2, channel 1 at t=1 -> channel 0 zeroed
    Q = np.zeros((1, 4, 2, 1, 1))
    Q[0, 2:, 0] = 9.0
    Q[0, 1:, 1] = 3.0
    Qi = oracle.inhibit(Q)
    assert (Qi[0, :, 0] == 0).all() and (Qi[0, :, 1] == Q[0, :, 1]).all()
    # same crossing step: the higher potential at that step survives
    Q = np.zeros((1, 4, 2, 1, 1))
    Q[0, 1:, 0] = 3.0
    Q[0, 1:, 1] = 5.0
    Qi = oracle.inhibit(Q)
    assert (Qi[0, :, 0] == 0).all()


@pytest.mark.parametrize("C,survivor", [(2, 0), (3, 1), (5, 2)])
def test_inhibit_channel_index_tie(C, survivor):
    # R-INHIBIT-TIE: channels with the same (first-crossing step, potential at it) tie;
    # the LOWER channel index survives, every other channel is zeroed at all steps.  Channels
    # below `survivor` cross later (or never), channels above it tie with it exactly.
    T = 6
    Q = np.zeros((1, T, C, 1, 2))
    for c in range(survivor, C):
        Q[0, 2:, c, 0, 0] = 4.0          # cross at t=2 with P* = 4 ...
        Q[0, 4:, c, 0, 0] = 4.0 + c       # ... and differ only after the crossing
    for c in range(survivor):
        Q[0, 3:, c, 0, 0] = 9.0          # later crossing, higher potential: loses on time
    Q[0, 1:, C - 1, 0, 1] = 1.0           # the other location is untouched by location (0, 0)
    Qi = oracle.inhibit(Q)
    for c in range(C):
        if c == survivor:
            np.testing.assert_array_equal(Qi[0, :, c, 0, 0], Q[0, :, c, 0, 0])
        else:
            assert (Qi[0, :, c, 0, 0] == 0).all(), c
    np.testing.assert_array_equal(Qi[0, :, :, 0, 1], Q[0, :, :, 0, 1])


def _indep_wta(Q, count, radius):
    """Independent version: sort all firing neurons by key once, scan with a suppression mask."""
    B, T, C, H, W = Q.shape
    out = []
    for b in range(B):
        fired = Q[b] > 0
        lat = np.where(fired.any(0), fired.argmax(0), T)
        ps = np.take_along_axis(Q[b], np.minimum(lat, T - 1)[None], 0)[0]
        cand = [(int(lat[c, y, x]), -float(ps[c, y, x]), c * H * W + y * W + x)
                for c in range(C) for y in range(H) for x in range(W) if lat[c, y, x] < T]
        cand.sort()
        mask = np.zeros((C, H, W), bool)
        res = []
        for l, nps, idx in cand:
            c, y, x = idx // (H * W), (idx // W) % H, idx % W
            if mask[c, y, x]:
                continue
            res.append((b, l, c, y, x))
            mask[c] = True
            mask[:, max(0, y - radius):y + radius + 1, max(0, x - radius):x + radius + 1] = True
            if len(res) == count:
                break
        out.append(res)
    return out


def test_wta_exhaustive_cross_check():
    for _ in range(30):
        B, T, C, H, W = 2, int(RNG.integers(1, 5)), int(RNG.integers(1, 5)), int(RNG.integers(1, 7)), int(RNG.integers(1, 7))
        Q = _rand_Q(B, T, C, H, W, 0.5)
        if _ % 4 == 0:
            Q = np.round(Q)  # ties in potential
        count, radius = int(RNG.integers(1, 6)), int(RNG.integers(0, 4))
        win, nwin = oracle.wta(Q, count, radius)
        ref = _indep_wta(Q, count, radius)
        for b in range(B):
            assert nwin[b] == len(ref[b])
            got = [tuple(win[b, q, :5]) for q in range(nwin[b])]
            assert got == ref[b]
            assert (win[b, :nwin[b], 5] == 0).all()
            chans = win[b, :nwin[b], 2]
            assert len(set(chans.tolist())) == len(chans)  # distinct channels
            for i in range(nwin[b]):
                for j in range(i):
                    assert abs(win[b, i, 3] - win[b, j, 3]) > radius or abs(win[b, i, 4] - win[b, j, 4]) > radius
            assert nwin[b] <= min(count, C)


def test_wta_edge_cases():
    Q = np.zeros((1, 4, 3, 5, 5))
    win, nwin = oracle.wta(Q, 5, 1)
    assert nwin[0] == 0  # nothing above threshold
    Q[0, 2:, 1, 3, 4] = 7.0
    win, nwin = oracle.wta(Q, 5, 1)
    assert nwin[0] == 1 and win[0, 0, :5].tolist() == [0, 2, 1, 3, 4]  # single candidate
    Q = _rand_Q(1, 4, 3, 4, 4, 1.0)
    win, nwin = oracle.wta(Q, 2, 10)
    assert nwin[0] == 1  # radius covering the map suppresses every channel at every place


# ---------------------------------------------------------------------- STDP (O11, O12)
def _one_synapse(w, tj, ti, cfg):
    """Weight of a 1x1x1x1 layer after one winner: input fires at tj (None = never)."""
    T = 10
    lat = np.array([[[[T if tj is None else tj]]]], np.uint8)
    S = oracle.lat_to_dense(lat, T)
    W = np.array([[[[w]]]], np.float32)
    win = np.array([[[0, ti, 0, 0, 0, 0]]], np.int32)
    return float(oracle.stdp(W, S, win, np.array([1], np.int32), [cfg])[0, 0, 0, 0])


def test_stdp_hand_worked():
    # W=.5, L=0, U=1, A=.1, t_j <= t_i -> .5 + .1*.5*.5 = .525
    assert _one_synapse(0.5, 2, 3, (0.1, -0.1, 0.0, 1.0, 1)) == np.float32(0.525)
    # BASELINE.json dw = a+ w(1-w): .0004 -> .5001 ; a- = -.0003 -> .499925
    assert _one_synapse(0.5, 1, 1, (0.0004, -0.0003, 0.0, 1.0, 1)) == np.float32(0.5001)
    assert _one_synapse(0.5, 4, 1, (0.0004, -0.0003, 0.0, 1.0, 1)) == np.float32(0.499925)
    # never-firing input depresses (t_j = inf)
    assert _one_synapse(0.5, None, 9, (0.0004, -0.0003, 0.0, 1.0, 1)) == np.float32(0.499925)
    # W = U and W = L are fixed points of the stabilised rule
    assert _one_synapse(1.0, 0, 3, (0.1, -0.1, 0.0, 1.0, 1)) == 1.0
    assert _one_synapse(0.0, 0, 3, (0.1, -0.1, 0.0, 1.0, 1)) == 0.0
    # unstabilised (Eq. 5) + clamp (Eq. 6): A- = -.0003 at W = .0001 -> 0
    assert _one_synapse(0.0001, 5, 1, (0.0004, -0.0003, 0.0, 1.0, 0)) == 0.0
    assert _one_synapse(0.9999, 0, 1, (0.0004, -0.0003, 0.0, 1.0, 0)) == 1.0
    assert _one_synapse(0.5, 0, 1, (0.0004, -0.0003, 0.0, 1.0, 0)) == np.float32(np.float32(0.5) + np.float32(0.0004))


def test_stdp_bounds_sign_and_batch_split():
    T = 6
    lat = RNG.integers(0, T + 1, (3, 2, 6, 6)).astype(np.uint8)
    S = oracle.lat_to_dense(lat, T)
    W0 = RNG.uniform(0.05, 0.95, (4, 2, 3, 3)).astype(np.float32)
    win = np.zeros((3, 2, 6), np.int32)
    for b in range(3):
        for q in range(2):
            win[b, q] = [b, RNG.integers(0, T), RNG.integers(0, 4), RNG.integers(0, 6), RNG.integers(0, 6), 0]
    nwin = np.array([2, 1, 2], np.int32)
    cfg = [(0.05, -0.04, 0.0, 1.0, 1)]
    W = oracle.stdp(W0, S, win, nwin, cfg, (1, 1), (1, 1))
    assert W.min() >= 0 and W.max() <= 1
    # batch == sequential single-sample processing
    Ws = W0.copy()
    for b in range(3):
        wb = win[b:b + 1].copy()
        wb[..., 0] = 0
        Ws = oracle.stdp(Ws, S[b:b + 1], wb, nwin[b:b + 1], cfg, (1, 1), (1, 1))
    np.testing.assert_array_equal(W, Ws)
    # 1000 random single updates stay in [L, U] and move in the sign of A inside (L, U)
    for _ in range(200):
        w = float(RNG.uniform(0, 1))
        tj, ti = int(RNG.integers(0, 5)), int(RNG.integers(0, 5))
        w2 = _one_synapse(w, tj, ti, (0.3, -0.2, 0.0, 1.0, 1))
        assert 0.0 <= w2 <= 1.0
        if 0 < w < 1:
            assert (w2 >= w) if tj <= ti else (w2 <= w)


def test_rstdp_routing_and_eq7():
    win = np.array([[[0, 1, 45, 0, 0, 0]], [[1, 1, 45, 0, 0, 0]]], np.int32)
    routed = oracle.rstdp_route(win, np.array([1, 1], np.int32), np.array([2, 3], np.int32), 20)
    assert routed[:, 0, 5].tolist() == [0, 1]  # map 45 -> class 2: reward for label 2, punish for 3
    reward = (0.0004, -0.0003, 0.0, 1.0, 1)
    punish = (-0.0004, 0.0003, 0.0, 1.0, 1)
    w = 0.3
    s = np.float32(np.float32(w - 0) * np.float32(1 - w))
    # Eq. 7 reward: pre before post -> A+_r (W-L)(U-W); pre after post -> A-_r (W-L)(U-W)
    assert _one_synapse(w, 1, 3, reward) == np.float32(np.float32(w) + np.float32(0.0004) * s)
    assert _one_synapse(w, 5, 3, reward) == np.float32(np.float32(w) + np.float32(-0.0003) * s)
    # Eq. 7 punish: pre before post -> A-_p (depress); pre after post -> A+_p (potentiate)
    assert _one_synapse(w, 1, 3, punish) == np.float32(np.float32(w) + np.float32(-0.0004) * s)
    assert _one_synapse(w, 5, 3, punish) == np.float32(np.float32(w) + np.float32(0.0003) * s)


# --------------------------------------------------------------------------- gather (O13)
def test_gather_examples():
    T = 15
    lat = np.array([[4, 15, 0]], np.uint8)
    f = oracle.gather(oracle.lat_to_dense(lat, T))
    np.testing.assert_array_equal(f, np.array([[11 / 15, 0, 1]], np.float32))


# ------------------------------------------------------------------------ listing geometry
def test_listing_geometry_c2():
    # Listing 1-3 shapes: 28x28 -> LoG(3,.,pad=3) 6x28x28 -> conv 5 p2 28x28 -> pool 2 -> 14x14
    cfg = synth.load_config("c2")
    imgs = synth.images(cfg, 0, 1)
    Ws = synth.layer_weights(cfg)
    y, lat0, inputs = pipeline.forward(cfg, imgs, Ws, upto=2, event=True)
    assert y.shape == (1, 6, 28, 28)
    assert inputs[1].shape == (1, 15, 30, 14, 14)
    assert inputs[2].shape == (1, 15, 250, 4, 4)


# ------------------------------------------------------------------------ golden fixtures
def test_golden_hand_worked():
    import json
    from conftest import GOLDEN

    g = json.loads((GOLDEN / "hand_worked.json").read_text())
    for c in g["stdp"]:
        assert _one_synapse(c["w"], c["tj"], c["ti"], tuple(c["cfg"])) == np.float32(c["expect"]), c["cite"]
    for c in g["rank_code"]:
        got = oracle.rank_code(np.array([c["values"]], np.float32), c["T"], 0.0)[0].tolist()
        assert got == c["expect"], c["cite"]
    s0, s1, s2 = g["shapes"]
    img = np.zeros((1, 1, s0["H"], s0["H"]), np.uint8)
    k = oracle.log_kernels([1.0] * s0["n_std"], s0["radius"])
    assert list(oracle.filter_apply(img, k, s0["pad"]).shape[1:]) == s0["expect"]
    assert oracle.conv_out_hw(s1["Hi"], s1["Hi"], s1["K"], s1["K"], s1["S"], s1["S"], s1["P"], s1["P"])[0] == s1["expect"]
    S = np.zeros((1, 1, 1, s2["Hi"], s2["Hi"]), np.uint8)
    assert oracle.pool(S, (s2["L"],) * 2, (s2["S"],) * 2, (s2["P"],) * 2).shape[-1] == s2["expect"]
