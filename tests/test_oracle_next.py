"""Pins for the oracle's NEXT-3 / NEXT-4 functions (no GPU): rate coding and its generator,
rate-based pooling, quantize, the fully connected layer, fcwta, FC STDP and ZCA whitening.

Each test names the passage or closed form it checks; none re-types the oracle's formula
(library special cases, published constants, hand-worked values, independently written
brute force on tiny inputs, invariants)."""
import numpy as np
import pytest

import oracle
from oracle import zca

RNG = np.random.default_rng(77)


# ------------------------------------------------------------------ O14 generator
def test_splitmix64_published_values():
    # splitmix64 from state 0 (Steele, Lea, Flood 2014; the reference C of xoshiro's seeding):
    # 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F — our stream 0 is that sequence.
    assert oracle.splitmix64(0, 0) == 0xE220A8397B1DCDAF
    assert oracle.splitmix64(0, 1) == 0x6E789E6AA1B965F4
    assert oracle.splitmix64(0, 2) == 0x06C45D188009454F
    # seed s shifts the state: stream s, counter c == stream 0 at state s + (c+1)*golden
    g = 0x9E3779B97F4A7C15
    assert oracle.splitmix64(g, 0) == oracle.splitmix64(0, 1)


# ---------------------------------------------------------------- O15 rate coding
def test_rate_code_spec_examples():
    T = 300
    v = np.zeros((1, 200), np.float32)
    v[0, 0] = 2.0                   # the sample max: p = 1 -> fires at every step
    v[0, 1] = -1.0                  # non-positive: p = 0 -> never
    v[0, 2:102] = 1.0               # p = 0.5 exactly
    S = oracle.rate_code(v, T, seed=12345)
    assert S.shape == (1, T, 200) and set(np.unique(S)) <= {0, 1}
    assert S[0, :, 0].all() and not S[0, :, 1].any() and not S[0, :, 102:].any()
    counts = S[0, :, 2:102].sum(axis=0).astype(np.int64)
    # binomial(300, 1/2): mean count over 100 neurons within [135, 165]; each neuron
    # within 6 sigma (sigma = sqrt(75) = 8.7) of 150
    assert 135 <= counts.mean() <= 165
    assert np.abs(counts - 150).max() < 6 * np.sqrt(75)
    # bit-reproducible for the same seed, different for another seed
    np.testing.assert_array_equal(oracle.rate_code(v, T, seed=12345), S)
    assert (oracle.rate_code(v, T, seed=999) != S).any()


def test_rate_code_bernoulli_frequencies_and_independence():
    # P:L109 "stochastic ... modeled with a Poisson distribution", per-step form: the spike
    # frequency of each neuron is its intensity over the sample max (binomial bounds), and the
    # steps are independent (lag-1 autocorrelation near 0, no cumulative structure).
    T = 400
    p = np.array([0.05, 0.1, 0.25, 0.5, 0.75, 0.9], np.float32)
    v = np.repeat(p, 50)[None].astype(np.float32)
    v[0, 0] = 1.0
    S = oracle.rate_code(v, T, seed=7)[0].astype(np.float64)  # [T][N]
    freq = S.mean(axis=0)
    for q, pq in enumerate(p):
        f = freq[q * 50 + 1:(q + 1) * 50].mean()
        sd = np.sqrt(pq * (1 - pq) / (T * 49))
        assert abs(f - pq) < 5 * sd, (pq, f)
    x = S[:, 50:] - S[:, 50:].mean(0)
    ac = (x[1:] * x[:-1]).sum() / (x * x).sum()
    assert abs(ac) < 0.02
    assert (np.diff(S[:, 151:200], axis=0) < 0).any()  # spikes are not cumulative


def test_rate_code_per_sample_and_scale_invariant():
    # per-sample normalisation: a sample's train does not depend on other samples, and
    # scaling a sample by a power of two (exact in fp32) leaves p and the train unchanged
    y = RNG.uniform(0, 1, (3, 40)).astype(np.float32)
    S = oracle.rate_code(y, 50, seed=3)
    y2 = y.copy()
    y2[1] *= 8
    S2 = oracle.rate_code(y2, 50, seed=3)
    np.testing.assert_array_equal(S2, S)
    assert oracle.rate_code(np.zeros((1, 9), np.float32), 20, 1).sum() == 0
    # a shard coded with its global base row draws exactly the whole batch's numbers
    np.testing.assert_array_equal(oracle.rate_code(y[1:], 50, seed=3, b0=1), S[1:])


# --------------------------------------------------------------- O16 rate pooling
def _brute_pool_rates(S, r, L, s, p):
    B, T, C, H, W = S.shape
    Ho, Wo = (H + 2 * p - L) // s + 1, (W + 2 * p - L) // s + 1
    out = np.zeros((B, T, C, Ho, Wo), np.uint8)
    for b in range(B):
        for c in range(C):
            for y in range(Ho):
                for x in range(Wo):
                    cells = [(iy, ix) for iy in range(y * s - p, y * s - p + L) for ix in range(x * s - p, x * s - p + L)
                             if 0 <= iy < H and 0 <= ix < W]
                    if not cells:
                        continue
                    # highest rate, then lowest flat index
                    iy, ix = min(cells, key=lambda q: (-r[b, c, q[0], q[1]], q[0] * W + q[1]))
                    out[b, :, c, y, x] = S[b, :, c, iy, ix]
    return out


def test_pool_rates_hand_and_brute_force():
    # the window's higher-rate neuron is selected (its whole train is kept)
    S = np.zeros((1, 4, 1, 1, 2), np.uint8)
    S[0, :, 0, 0, 0] = [1, 0, 0, 0]
    S[0, :, 0, 0, 1] = [0, 1, 1, 0]
    r = oracle.gather(S)
    out = oracle.pool_rates(S, r, (1, 2))
    np.testing.assert_array_equal(out[0, :, 0, 0, 0], [0, 1, 1, 0])
    # equal rates -> lowest flat index (reading R-RATE-POOL-TIE)
    S[0, :, 0, 0, 1] = [0, 0, 1, 0]
    np.testing.assert_array_equal(oracle.pool_rates(S, oracle.gather(S), (1, 2))[0, :, 0, 0, 0], [1, 0, 0, 0])
    for (L, s, p) in [(2, 2, 0), (3, 3, 0), (3, 2, 1), (2, 1, 1)]:
        S = (RNG.random((2, 9, 3, 7, 8)) < 0.3).astype(np.uint8)
        r = oracle.gather(S)
        np.testing.assert_array_equal(oracle.pool_rates(S, r, (L, L), (s, s), (p, p)), _brute_pool_rates(S, r, L, s, p))


# ------------------------------------------------------------------- O17 quantize
def test_quantize_spec_examples():
    # Listing 4 quantize(kernel, 0, 0.5, 1); [0.1, 0.5, 0.9] -> [0, 1, 1] (mid -> upper)
    np.testing.assert_array_equal(oracle.quantize(np.array([0.1, 0.5, 0.9], np.float32), 0, 0.5, 1), [0, 1, 1])
    w = RNG.uniform(0, 1, 1000).astype(np.float32)
    q = oracle.quantize(w, 0, 0.5, 1)
    np.testing.assert_array_equal(q, (w >= 0.5).astype(np.float32))
    np.testing.assert_array_equal(oracle.quantize(q, 0, 0.5, 1), q)             # idempotent
    np.testing.assert_array_equal(oracle.quantize(w, 0.3, 0.5, 0.3), np.full(1000, 0.3, np.float32))  # lower = upper


# ------------------------------------------------------------------------- O18 FC
def test_fc_matches_matmul_and_identity():
    # out[b,t,o] = sum_i S[b,t,i] W[i,o]  (numpy matmul as the library check)
    S = (RNG.random((3, 5, 17)) < 0.4).astype(np.uint8)
    W = RNG.uniform(0, 1, (17, 6)).astype(np.float32)
    np.testing.assert_allclose(oracle.fc(S, W), S.astype(np.float64) @ W.astype(np.float64), rtol=1e-12)
    # identity weights -> output = input cast; zero spikes -> zero potentials
    np.testing.assert_array_equal(oracle.fc(S, np.eye(17, dtype=np.float32)), S.astype(np.float64))
    assert not oracle.fc(np.zeros_like(S), W).any()
    # an FC layer is the 1x1 convolution of a 1x1 map: the independent conv definition agrees
    P = oracle.conv(S[:, :, :, None, None], np.ascontiguousarray(W.T)[:, :, None, None])
    np.testing.assert_allclose(P[..., 0, 0], oracle.fc(S, W), rtol=1e-12)


def _indep_fcwta(Q, count, radius):
    B, T, O = Q.shape
    res = []
    for b in range(B):
        fired = Q[b] > 0
        lat = np.where(fired.any(0), fired.argmax(0), T)
        ps = np.take_along_axis(Q[b], np.minimum(lat, T - 1)[None], 0)[0]
        order = sorted((int(lat[o]), -float(ps[o]), o) for o in range(O) if lat[o] < T)
        dead = np.zeros(O, bool)
        got = []
        for l, _, o in order:
            if dead[o]:
                continue
            got.append((b, l, o))
            dead[max(0, o - radius):o + radius + 1] = True
            if len(got) == count:
                break
        res.append(got)
    return res


def test_fcwta_spec_examples_and_exhaustive():
    Q = np.zeros((1, 4, 1))
    Q[0, 2:, 0] = 3.0
    win, nwin = oracle.fcwta(Q, 3, 0)
    assert nwin[0] == 1 and win[0, 0].tolist() == [0, 2, 0, 0, 0, 0]  # O = 1 above threshold
    for _ in range(40):
        B, T, O = 2, int(RNG.integers(1, 6)), int(RNG.integers(1, 30))
        P = np.cumsum(RNG.uniform(0, 1, (B, T, O)) * (RNG.random((B, 1, O)) < 0.6), axis=1)
        if _ % 3 == 0:
            P = np.round(P)
        Q = oracle.threshold(P, 1.0)
        count, radius = int(RNG.integers(1, 6)), int(RNG.integers(0, 4))
        win, nwin = oracle.fcwta(Q, count, radius)
        ref = _indep_fcwta(Q, count, radius)
        for b in range(B):
            assert [tuple(win[b, q, :3]) for q in range(nwin[b])] == ref[b]
        if radius >= O:
            assert (nwin <= 1).all()  # radius covering every index: one winner


def test_fc_stdp_equals_conv_stdp_of_1x1_map():
    # FC STDP ("fully connected or convolution layers") == conv STDP of the 1x1 geometry
    # with the kernel transposed to [O][I][1][1] (independent O11 implementation)
    T, B, I_, O = 8, 3, 11, 5
    lat = RNG.integers(0, T + 1, (B, I_)).astype(np.uint8)
    S = oracle.lat_to_dense(lat, T)
    W = RNG.uniform(0.05, 0.95, (I_, O)).astype(np.float32)
    win = np.full((B, 2, 6), -1, np.int32)
    nwin = np.array([2, 1, 0], np.int32)
    for b in range(B):
        for q in range(nwin[b]):
            win[b, q] = [b, RNG.integers(0, T), RNG.integers(0, O), 0, 0, q % 2]
    cfgs = [(0.01, -0.008, 0.0, 1.0, 1), (-0.01, 0.008, 0.0, 1.0, 0)]
    got = oracle.fc_stdp(W, S, win, nwin, cfgs)
    ref = oracle.stdp(np.ascontiguousarray(W.T)[:, :, None, None], S[:, :, :, None, None], win, nwin, cfgs)
    np.testing.assert_array_equal(got, ref[:, :, 0, 0].T)


# ------------------------------------------------------------------------ ZCA (R-ZCA)
def test_zca_spec_examples():
    # the 2-feature toy set {(1,1),(-1,-1),(1,-1),(-1,1)} scaled -> output covariance = I
    X = np.array([[1, 1], [-1, -1], [1, -1], [-1, 1]], np.float64) * np.array([3.0, 0.5])
    mu, Wz = zca.fit(X, 0.0)
    Y = zca.apply(X, mu, Wz)
    np.testing.assert_allclose(np.cov(Y, rowvar=False), np.eye(2), atol=1e-12)
    np.testing.assert_allclose(Wz, Wz.T, atol=1e-14)  # symmetric
    # white data, eps = 0 -> apply is (almost) centering only
    Z = RNG.normal(0, 1, (20000, 3))
    Z = (Z - Z.mean(0)) @ np.linalg.inv(np.linalg.cholesky(np.cov(Z, rowvar=False))).T + 5.0
    mu, Wz = zca.fit(Z, 0.0)
    np.testing.assert_allclose(Wz, np.eye(3), atol=1e-9)
    np.testing.assert_allclose(zca.apply(Z, mu, Wz), Z - 5.0, atol=1e-8)


def test_zca_shrinkage_and_zero_phase():
    # with eps > 0 the output covariance is diag(lam/(lam+eps)) in the eigenbasis
    # (checked as E^T cov(Y) E); ZCA is the zero-phase whitening: of all whitening matrices it is
    # the symmetric one closest to identity — W^2 = C^-1 for eps = 0 (Bell & Sejnowski 1997)
    A = RNG.normal(0, 1, (6, 6))
    X = RNG.normal(0, 1, (5000, 6)) @ A
    eps = 0.3
    mu, Wz = zca.fit(X, eps)
    C = np.cov(X, rowvar=False)
    lam, E = np.linalg.eigh(C)
    D = E.T @ np.cov(zca.apply(X, mu, Wz), rowvar=False) @ E
    np.testing.assert_allclose(D, np.diag(lam / (lam + eps)), atol=1e-9)
    mu0, W0 = zca.fit(X, 0.0)
    np.testing.assert_allclose(W0 @ W0, np.linalg.inv(C), rtol=1e-8, atol=1e-10)
