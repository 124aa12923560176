"""GPU parity of the NEXT-3 / NEXT-4 steps against the CPU oracle:
rate coding (bit-exact, same counter-based stream), rate gather and rate pooling, the per-step
conv + fire on rate-coded step maps, the rate-coded C6 pipeline, quantize, the FC layer + fcwta +
FC STDP, and ZCA fit / apply.  Comparison rules: tests/parity.py."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import pipeline as opipe
from oracle import zca as ozca
from parity import ParityReport, assert_potentials, lat_and_pstar, near_threshold

pytestmark = pytest.mark.gpu
RNG = np.random.default_rng(4242)


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


# ------------------------------------------------------------------ NEXT-3 rate coding
@pytest.mark.parametrize("B,N,T", [(3, 4704, 300), (2, 1, 15), (4, 37, 1), (2, 5003, 30), (1, 301056, 4)])
def test_rate_code_bit_exact(spk, B, N, T):
    y = RNG.normal(0, 1, (B, N)).astype(np.float32)
    y[0, : N // 3] = np.abs(y[0, : N // 3])
    if B > 1:
        y[1] = -1.0  # nothing above threshold: never spikes
    seed, b0 = 0x1234_5678_9ABC, 7
    S = oracle.rate_code(oracle.threshold(y, 0.01), T, seed, b0)
    step = host(spk.rate_code(cu(y), T, 0.01, seed, b0=b0))
    np.testing.assert_array_equal(step, 1 - S)


def test_rate_gather_and_pool_rates_exact(spk):
    T = 40
    S = (RNG.random((3, T, 4, 9, 11)) < 0.3).astype(np.uint8)
    S[0, :, 0, :3, :3] = 1  # equal rates in a window: lowest flat index wins
    step = cu(1 - S)
    r = oracle.gather(S)
    gr = host(spk.rate_gather(step))
    np.testing.assert_array_equal(gr, r)
    for (L, s, p) in [(2, 2, 0), (3, 3, 0), (3, 2, 1), (2, 1, 1)]:
        ref = oracle.pool_rates(S, r, (L, L), (s, s), (p, p))
        got = host(spk.pool_rates(step, cu(gr), L, s, p))
        np.testing.assert_array_equal(got, 1 - ref)


@pytest.mark.parametrize("prec", ["event", "exact"])
@pytest.mark.parametrize("shape", [(2, 20, 6, 12, 13, 25, 5), (3, 9, 25, 14, 14, 50, 3), (1, 40, 6, 28, 28, 25, 5),
                                   (2, 5, 30, 9, 11, 70, 3)])
def test_rate_coded_conv_fire_per_step(spk, prec, shape):
    """Eq. 2 per step on non-cumulative trains: spk_conv on the step map with B' = B*T, T' = 1
    (tensor path: one time step per row, 128 pixels per M tile) equals the oracle's direct BTCHW
    conv (potentials) and its per-step fire (spikes), P* included."""
    B, T, Ci, H, W, Co, K = shape
    S = (RNG.random((B, T, Ci, H, W)) < 0.25).astype(np.uint8)
    w = oracle.quantize(RNG.uniform(0, 1, (Co, Ci, K, K)).astype(np.float32), 0, 0.5, 1)
    P = oracle.conv(S, w, (1, 1), ((K - 1) // 2,) * 2)
    x = cu((1 - S).reshape(B * T, Ci, H, W))
    got = host(spk.conv(x, cu(w), 1, 1, (K - 1) // 2, prec=prec, epi="potential")).reshape(P.shape)
    np.testing.assert_array_equal(got, P)  # binary weights: exact integers on every engine
    theta = float(np.percentile(P, 80)) + 0.5
    lat, ps = spk.conv(x, cu(w), 1, 1, (K - 1) // 2, prec=prec, epi="fire", theta=theta)
    S = oracle.fire(P, theta)
    np.testing.assert_array_equal(host(lat).reshape(B, T, Co, H, W), 1 - S)
    np.testing.assert_array_equal(host(ps).reshape(B, T, Co, H, W), np.where(S == 1, P, 0).astype(np.float32))


def test_rate_pipeline_c6(spk):
    """C6: rate-coded inference with quantized weights, 300 steps, rate pooling;
    every layer's step map, rates and the features equal the oracle's bit for bit (binary
    weights: integer potentials, no near-threshold ambiguity)."""
    from paper_2301_13659_b200.network import RateNetwork
    cfg = synth.load_config("c6")
    n, start = 3, 5
    imgs = synth.images(cfg, start, n)
    Ws = synth.layer_weights(cfg)
    ref = opipe.rate_infer(cfg, imgs, Ws, start)
    net = RateNetwork(cfg, n, prec="auto", start=start)
    net.img.copy_(cu(imgs))
    net.set_weights([cu(w) for w in Ws])
    net.infer()
    np.testing.assert_array_equal(host(net.step0), 1 - ref["S0"])
    for li in range(len(cfg["layers"])):
        np.testing.assert_array_equal(host(net.layers[li]["step"]), 1 - ref["steps"][li])
        np.testing.assert_array_equal(host(net.layers[li]["rates"]), ref["rates"][li])
        np.testing.assert_array_equal(host(net.layers[li]["pooled"]), 1 - ref["pooled"][li])
        ParityReport.latency(("C6 rate-coded inference, batch 3", f"conv{li} per-step fire"),
                             host(net.layers[li]["step"]), 1 - ref["steps"][li], None)
    np.testing.assert_array_equal(host(net.features), ref["features"])
    assert ref["features"].max() > 0  # something fires


def test_rate_pipeline_c6_graph_and_shards(spk):
    """C6 as bench.py runs it (CUDA graph replay), and two shards (global sample bases) whose
    concatenation equals the whole batch bit for bit (the stream runs over global indices)."""
    from paper_2301_13659_b200.network import RateNetwork
    cfg = synth.load_config("c6")
    n = 6
    imgs = synth.images(cfg, 0, n)
    Ws = [cu(w) for w in synth.layer_weights(cfg)]

    def run(start, m, graph):
        net = RateNetwork(cfg, m, prec="auto", start=start)
        net.img.copy_(cu(imgs[start:start + m]))
        net.set_weights(Ws)
        if graph:
            net.capture(warmup=1)
            net.replay()
        else:
            net.infer()
        return host(net.features)

    whole = run(0, n, True)
    np.testing.assert_array_equal(np.concatenate([run(0, 3, False), run(3, 3, False)]), whole)


# ------------------------------------------------------------------ NEXT-4 quantize, FC, fcwta
def test_quantize_exact(spk):
    w = RNG.uniform(-0.5, 1.5, (1000, 7)).astype(np.float32)
    w[0, :3] = [0.5, 0.4999999, 0.5000001]
    g = cu(w)
    spk.quantize(g, 0.0, 0.5, 1.0)
    np.testing.assert_array_equal(host(g), oracle.quantize(w, 0.0, 0.5, 1.0))
    with pytest.raises(spk.SpkError):
        spk.quantize(g, 1.0, 0.5, 0.0)


@pytest.mark.parametrize("prec", ["exact", "event", "fp32"])
@pytest.mark.parametrize("B,T,I,O", [(5, 15, 300, 40), (3, 30, 1000, 10), (2, 1, 17, 3), (37, 15, 3200, 200),
                                     (64, 30, 1000, 10), (8, 2, 17, 3)])
def test_fc_potentials_and_fire(spk, prec, B, T, I, O):
    lat = RNG.integers(0, T + 1, (B, I)).astype(np.uint8)
    W = RNG.uniform(0, 1, (I, O)).astype(np.float32)  # the paper's I x O kernel
    w_dev = cu(np.ascontiguousarray(W.T))              # stored output-major [O][I]
    if prec == "event" and spk.fc_workspace(B, T, I, O, "event") == 0:
        pytest.skip("event weight block does not fit")
    S = oracle.lat_to_dense(lat, T)
    P = oracle.fc(S, W)
    got = host(spk.fc(cu(lat), w_dev, T, prec=prec, epi="potential"))
    assert_potentials(got, P)
    theta = float(np.percentile(P[:, -1], 50)) + 0.0123
    glat, gps = spk.fc(cu(lat), w_dev, T, prec=prec, epi="fire", theta=theta)
    rlat, rps = lat_and_pstar(P[:, :, :, None, None], theta)
    excl = near_threshold(P[:, :, :, None, None], theta)[..., 0, 0]
    glat, gps = host(glat), host(gps)
    ParityReport.latency(("FC fire", prec), glat, rlat[..., 0, 0], excl)
    assert not ((glat != rlat[..., 0, 0]) & ~excl).any()
    ok = (glat == rlat[..., 0, 0]) & (glat < T)
    assert_potentials(gps[ok], rps[..., 0, 0][ok])


@pytest.mark.parametrize("O,k,r", [(10, 3, 0), (200, 5, 2), (1, 2, 1), (3000, 8, 10), (30000, 4, 3)])
def test_fcwta_exact(spk, O, k, r):
    B, T = 4, 12
    P = np.cumsum(RNG.uniform(0, 1, (B, T, O)) * (RNG.random((B, 1, O)) < 0.5), axis=1)
    P[1] = np.round(P[1] * 2) / 2  # ties
    P = P.astype(np.float32).astype(np.float64)
    Q = oracle.threshold(P, 1.1)
    win, nwin = oracle.fcwta(Q, k, r)
    lat, ps = lat_and_pstar(Q[:, :, :, None, None], 0.0)
    gw, gn = spk.fcwta(cu(lat[..., 0, 0]), cu(ps[..., 0, 0].astype(np.float32)), T, k, r)
    gw, gn = host(gw), host(gn)
    np.testing.assert_array_equal(gn, nwin)
    for b in range(B):
        np.testing.assert_array_equal(gw[b, :nwin[b]], win[b, :nwin[b]])
        assert (gw[b, nwin[b]:] == -1).all()


def test_fc_train_step_fire_fcwta_stdp(spk):
    """An FC layer's training step (Listing 3 with fc + fcwta): fire -> fcwta -> STDP on the
    1x1 geometry == oracle fc -> threshold -> fcwta -> fc_stdp (I x O weights), bit for bit
    (B = 21: the batched tensor path, samples as the pixels of one image)."""
    B, T, I, O = 21, 15, 800, 50
    lat = RNG.integers(0, T + 1, (B, I)).astype(np.uint8)
    W = np.clip(RNG.normal(0.5, 0.05, (I, O)), 0, 1).astype(np.float32)
    S = oracle.lat_to_dense(lat, T)
    P = oracle.fc(S, W)
    # a threshold in the middle of a gap of the potentials around their 70th percentile, so no
    # potential lies within the near-threshold band (the comparison below is then all exact)
    v = np.unique(P.ravel())
    target = np.percentile(P[:, -1], 70)
    ok = [i for i in range(len(v) - 1) if v[i + 1] - v[i] > 3e-4 * (v[i] + v[i + 1]) / 2 and v[i] > 0]
    i = min(ok, key=lambda q: abs(v[q] - target))  # the clear gap nearest the 70th percentile
    theta = float((v[i] + v[i + 1]) / 2)
    Q = oracle.threshold(P, theta)
    win, nwin = oracle.fcwta(Q, 3, 2)
    cfgs = [(0.004, -0.003, 0.0, 1.0, 1)]
    Wn = oracle.fc_stdp(W, S, win, nwin, cfgs)
    w_dev = cu(np.ascontiguousarray(W.T))
    glat, gps = spk.fc(cu(lat), w_dev, T, prec="exact", epi="fire", theta=theta)
    excl = near_threshold(P[:, :, :, None, None], theta)[..., 0, 0]
    assert not excl.any(), "re-seed: a potential near the threshold"
    gw, gn = spk.fcwta(glat, gps, T, 3, 2)
    np.testing.assert_array_equal(host(gn), nwin)
    spk.fc_stdp(w_dev, cu(lat), gw, gn, cfgs, T)
    np.testing.assert_array_equal(host(w_dev).T, Wn)


# ------------------------------------------------------------------------------- ZCA
@pytest.mark.parametrize("B,F,eps", [(1024, 784, 0.1), (500, 36, 0.0), (64, 200, 1e-2)])
def test_zca_fit_apply(spk, B, F, eps):
    A = RNG.normal(0, 1, (F, F)) / np.sqrt(F)
    X = (RNG.normal(0, 1, (B, F)) @ A + RNG.uniform(-1, 1, F)).astype(np.float32)
    if B <= F and eps == 0:
        pytest.skip("singular")
    mu, Wz = ozca.fit(X.astype(np.float64), eps)
    gm, gw = spk.zca_fit(cu(X), eps)
    np.testing.assert_allclose(host(gm), mu, rtol=1e-6, atol=1e-6)
    scale = np.abs(Wz).max()
    np.testing.assert_allclose(host(gw), Wz, rtol=0, atol=2e-5 * scale)
    Y = ozca.apply(X.astype(np.float64), mu, Wz)
    gy = host(spk.zca_apply(cu(X), gm, gw))
    err = np.abs(gy - Y).max() / np.abs(Y).max()
    ParityReport.potentials(("ZCA apply", f"B={B} F={F}"), gy, Y)
    assert err < 1e-4, err
    # whitened output covariance (eps = 0): identity
    if eps == 0:
        np.testing.assert_allclose(np.cov(gy.astype(np.float64), rowvar=False), np.eye(F), atol=2e-3)
