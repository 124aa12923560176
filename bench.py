"""Benchmark of the SDNN hot path (BASELINE.json metric) on 1..N B200s.

    python bench.py [--gpus N --steps K --warmup W --config c2 --impl ours|reference]

One step = one pass of the whole hot path over one batch: for configs[1] (C2,
the default) the layer-3 training step of the 3-layer STDP SDNN at batch 1024,
T = 15: DoG/LoG filter -> rank-order code -> conv1+fire -> pool -> conv2+fire ->
pool -> conv3+fire record -> lateral inhibition -> k-WTA -> STDP (in place).
With --gpus N > 1 (and no torchrun around it) the script relaunches itself under
torch.distributed.run with N ranks on 127.0.0.1.  Training configs at N > 1 run
the data-parallel mini-batch STDP of SURVEY NEXT-2 by default (one model, global
batch N x B, winners + trained-layer inputs all-gathered over NCCL, identical
update on every rank; --replicas trains N independent replicas instead);
forward configs (C5, C6) shard the global batch.  Timing: CUDA events on the
launching stream around each replayed CUDA graph, L2 flushed (256 MiB write)
between timed steps, max over ranks.  Prints one JSON line on rank 0.

Workloads: --config c2 (default, BASELINE configs[1]), c1, c3, c4, c5 (the other
BASELINE configs), c2q (Listing 4: layers 1-2 quantized to {0,1}, NEXT-4), c6
(rate-coded T=300 inference, NEXT-3).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SDNN images/s (T=15, forward+STDP) at 1/2/4/8 B200; % HBM / tensor roofline"
INT8_OVER_BF16 = 2.0  # guide's nominal dense ratio: 4.5 POPS int8 / 2.25 PFLOPS bf16


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--prec", default="auto", choices=["auto", "exact", "event", "fp32"],
                    help="conv engine: auto = event form for small-N layers, tcgen05 otherwise (bit-identical)")
    ap.add_argument("--dp", action="store_true",
                    help="data-parallel mini-batch STDP (SURVEY NEXT-2) also at N = 1 (the default at N > 1): "
                         "per-GPU batch fixed, winners + input maps all-gathered, same update on every rank")
    ap.add_argument("--replicas", action="store_true",
                    help="training configs at N > 1: N independent replicas instead of one data-parallel model")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=8, help="images in the oracle cpu_baseline sample")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained"), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class Clocks:
    """nvidia-smi clocks/throttle sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.index = index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait(timeout=10)
        self.f.flush()
        rows = [r.split(", ") for r in Path(self.f.name).read_text().strip().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def conv_flops(rec, B, T):
    g = rec["geom"]
    return 2.0 * B * T * rec["Ho"] * rec["Wo"] * g.Co * (g.Ci * g.Kh * g.Kw)


def event_adds(net, li):
    """Active-synapse adds of one event-form conv launch: every output map o and output pixel
    (y, x) adds the weight of each in-bounds input tap that fires (lat < T) once."""
    import torch

    g = net.layers[li]["geom"]
    act = (net.input_of(li) < net.T).float().sum(dim=1, keepdim=True)  # [B][1][Hi][Wi]
    ones = torch.ones((1, 1, g.Kh, g.Kw), device=act.device)
    per_px = torch.nn.functional.conv2d(act, ones, stride=(g.Sh, g.Sw), padding=(g.Ph, g.Pw))
    return float(per_px.sum().item()) * g.Co


SMEM_WORDS_PER_CLK_SM = 32  # 128 B/clk/SM shared-memory bandwidth / 4-byte weight per add


def _oracle_step(cfg, imgs, Ws, lab, start):
    """One step of the plain oracle on `imgs` (global indices start..)."""
    from oracle import pipeline as opipe

    if cfg.get("kind") == "fc":
        import oracle
        import synth
        S = oracle.lat_to_dense(synth.latencies(cfg, start, len(imgs), cfg["I"], cfg["T"], cfg["p_fire"]), cfg["T"])
        W = synth.fc_weights(cfg)
        Q = oracle.threshold(oracle.fc(S, W), cfg["theta"])
        win, nwin = oracle.fcwta(Q, cfg["wta"]["count"], cfg["wta"]["radius"])
        return {"W_new": oracle.fc_stdp(W, S, win, nwin, [tuple(c) for c in cfg["stdp"]])}
    if cfg.get("kind") == "zca":
        from oracle import zca as ozca
        X = imgs.reshape(len(imgs), -1).astype(np.float64) / 255.0
        return ozca.apply(X, *ozca.fit(X, cfg["eps"])) if len(imgs) > 1 else None
    if cfg.get("coding") == "rate":
        return opipe.rate_infer(cfg, imgs, Ws, start)
    if cfg["timed"] == "train":
        return opipe.train_step(cfg, imgs, Ws, lab)
    return opipe.infer(cfg, imgs, Ws)


def cpu_baseline(cfg, n_images):
    """The oracle as it stands (oracle/, single thread) on a bounded sample of the same workload."""
    import oracle
    import synth

    imgs = synth.images(cfg, 0, n_images)
    lab = synth.labels(cfg, 0, n_images)
    Ws = synth.layer_weights(cfg)
    crop = cfg.get("cpu_crop")  # C5: one 224x224 image takes the oracle ~5 min; time a corner crop
    frac = 1.0
    if crop:
        H, W = imgs.shape[-2:]
        imgs = np.ascontiguousarray(imgs[..., :crop, :crop])
        frac = crop * crop / (H * W)  # every step of the path is per output pixel: work ~ area
    oracle.lib()
    t0 = time.perf_counter()
    _oracle_step(cfg, imgs, Ws, lab, 0)
    dt = time.perf_counter() - t0
    what = (f"the top-left {crop}x{crop} crop of image 0 ({frac:.4f} of its area; value = area fraction "
            f"/ time)" if crop else f"{n_images} images of {cfg['name']} (global indices 0..{n_images - 1})")
    return {"value": n_images * frac / dt, "unit": "images/s", "cores": 1, "kind": "oracle", **host_info(),
            "sample": f"{what}, one full {cfg['timed']} step of the plain oracle (direct Eq. 2), "
                      f"1 host thread, {dt:.1f} s"}


def host_info():
    model = "unknown"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    per_step = max(1, args.cpu_sample // (8 if cfg.get("coding") == "rate" else 4))
    import oracle
    import synth

    oracle.lib()
    Ws = synth.layer_weights(cfg) if "layers" in cfg else None
    if cfg.get("kind") in ("fc", "zca"):
        per_step = max(per_step, 64)
    times = []
    for s in range(args.warmup + args.steps):
        imgs = (synth.images(cfg, s * per_step, per_step) if "image" in cfg
                else np.zeros((per_step, 1), np.uint8))  # FC: the step draws its own input latencies
        lab = synth.labels(cfg, s * per_step, per_step)
        t0 = time.perf_counter()
        r = _oracle_step(cfg, imgs, Ws, lab, s * per_step)
        if cfg["timed"] == "train" and "train_layer" in cfg:
            Ws[cfg["train_layer"]] = r["W_new"]
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    t = float(np.mean(times))
    v = per_step / t
    sample = f"{per_step} images of {cfg['name']} per step (consecutive global indices), plain oracle, 1 host thread"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "images/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg['name']}: {cfg['about']}", "global_batch": per_step, "T": cfg["T"],
                   "parallelism": "cpu oracle, rank 0 only"},
        "cpu_baseline": {"value": v, "unit": "images/s", "cores": 1, "kind": "oracle", "sample": sample,
                         **host_info()},
        "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def relaunch(args):
    """--gpus N > 1 without a launcher: run this script under torch.distributed.run, N ranks."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def stage_bytes(net, cfg, B):
    """Algorithmic HBM bytes of each bandwidth stage of one step (natural compact
    I/O types, no re-reads): the numerators of the per-stage HBM fractions."""
    T = cfg["T"]
    out = {}
    fr = cfg["front"]
    img = B * cfg["image"]["C"] * cfg["image"]["H"] * cfg["image"]["W"]
    y = net.y.numel()
    out["filter"] = img + 4 * y
    if cfg.get("coding") == "rate":
        out["rate_code"] = 4 * y + T * y  # f32 response in, one step-map byte per (t, neuron) out
        for li, rec in enumerate(net.layers):
            if rec["rates"] is not None:
                out[f"rates{li}"] = rec["step"].numel() + 4 * rec["rates"].numel()
                out[f"pool{li}"] = 4 * rec["rates"].numel() + 2 * rec["pooled"].numel()
        last = net.layers[-1]
        src = last["pooled"] if last["pooled"] is not None else last["step"]
        out["gather"] = src.numel() + 4 * net.features.numel()
        return out
    out["rank_code"] = 5 * y
    for li, rec in enumerate(net.layers):
        if rec.get("pooled") is not None and not rec.get("fused_pool"):
            out[f"pool{li}"] = rec["lat"].numel() + rec["pooled"].numel()
    tl = cfg.get("train_layer")
    if tl is not None and cfg["timed"] == "train":
        n = net.layers[tl]["lat"].numel()
        out["inhibit"] = 10 * n
        out["wta"] = 5 * n + 24 * net.k * B
    else:
        out["gather"] = 5 * net.features.numel()
    return out


def _trace(msg):
    if os.environ.get("SPK_BENCH_TRACE"):
        print(f"[bench] {msg}", file=sys.stderr, flush=True)


def fc_zca_line(args, cfg, value, ms, e2e_ms, h2d, d2h, launches, roof, live_ms, clk, cpu, extra=None):
    line = {"metric": METRIC, "value": value, "unit": "images/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32/int64 exact (FC)" if cfg["kind"] == "fc" else "f32",
            "data": "synthetic", "config": {"workload": f"{cfg['name']}: {cfg['about']}", "global_batch": cfg["batch"],
                                            "T": cfg["T"], "l2": "flushed between timed steps (256 MiB write)",
                                            "cuda_graph": True, **(extra or {})},
            "e2e": {"value": cfg["batch"] / (e2e_ms * 1e-3), "unit": "images/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches * args.steps), "roofline": roof, "stage_ms": live_ms, "clocks": clk}
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def io_graph(body, ins, outs):
    """The host-to-host step as one CUDA graph (copies in, body, copies out) — the e2e analogue of
    Network.capture_io for the workloads that call the C ABI directly."""
    import torch

    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for dst, src in ins:
            dst.copy_(src, non_blocking=True)
        body(lambda n: None)
        for dst, src in outs:
            dst.copy_(src, non_blocking=True)
    return g


def timed_graph(args, body, dev, stages):
    """Capture body(mark) in a CUDA graph; time K replays (L2 flushed between) with per-stage events."""
    import torch

    marks = []

    def mark(name):
        e = torch.cuda.Event(enable_timing=True, external=True)
        e.record(torch.cuda.current_stream(dev))
        marks.append((name, e))

    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    _trace("warm-up body on a side stream")
    with torch.cuda.stream(s):
        body(lambda n: None)
    torch.cuda.current_stream(dev).wait_stream(s)
    torch.cuda.synchronize()
    _trace("capture")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        mark("start")
        body(mark)
    _trace("captured")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        g.replay()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    _trace("replays")
    clocks = Clocks(dev.index or 0)
    clocks.start()
    time.sleep(0.3)
    evs, live = [], {}
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
        evs.append((e0, e1))
        e1.synchronize()
        for (n1, m1), (n2, m2) in zip(marks[:-1], marks[1:]):
            live.setdefault(n2, []).append(m1.elapsed_time(m2))
    torch.cuda.synchronize()
    ms = float(sum(a.elapsed_time(b) for a, b in evs) / args.steps)
    g.spk_marks = marks  # the graph's event-record nodes point at these events: keep them alive
    return g, ms, {k: float(np.mean(v)) for k, v in live.items()}, clocks, flush


def run_fc(args, cfg):
    """NEXT-4 FC training step: spk_fc(FIRE) -> spk_fcwta -> FC STDP (spk_stdp, 1x1 geometry)."""
    import torch

    import synth
    from paper_2301_13659_b200 import spk

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    B, T, I_, O = cfg["batch"], cfg["T"], cfg["I"], cfg["O"]
    lat_h = torch.from_numpy(synth.latencies(cfg, 0, B, I_, T, cfg["p_fire"]))
    W = synth.fc_weights(cfg)
    w = torch.from_numpy(np.ascontiguousarray(W.T)).to(dev)  # output-major [O][I] (R-FC-LAYOUT)
    w0 = w.clone()
    lat = lat_h.to(dev)
    prec = "event" if spk.fc_workspace(B, T, I_, O, "event") > 0 else "exact"
    ws = torch.empty(max(1, spk.fc_workspace(B, T, I_, O, prec)), dtype=torch.uint8, device=dev)
    out_lat = torch.empty((B, O), dtype=torch.uint8, device=dev)
    out_ps = torch.empty((B, O), dtype=torch.float32, device=dev)
    k, r = cfg["wta"]["count"], cfg["wta"]["radius"]
    win = torch.empty((B, k, 6), dtype=torch.int32, device=dev)
    nwin = torch.empty((B,), dtype=torch.int32, device=dev)
    g = spk.ConvGeom(B, T, I_, 1, 1, O, 1, 1, 1, 1, 0, 0)
    sws = torch.empty(spk.stdp_workspace(g, k), dtype=torch.uint8, device=dev)
    carr = spk.stdp_configs(cfg["stdp"])

    def body(mark):
        spk.fc(lat, w, T, prec=prec, epi="fire", theta=cfg["theta"], out0=out_lat, out1=out_ps, ws=ws)
        mark("fc")
        spk.fcwta(out_lat, out_ps, T, k, r, win=win, nwin=nwin)
        mark("fcwta")
        spk.fc_stdp(w, lat, win, nwin, None, T, ws=sws, cfg_arr=carr)
        mark("stdp")

    _trace(f"fc eager step (engine {prec})")
    n0 = spk.launch_count()
    body(lambda n: None)
    torch.cuda.synchronize()
    launches = spk.launch_count() - n0
    _trace("fc eager step done")
    w.copy_(w0)
    graph, ms, live, clocks, flush = timed_graph(args, body, dev, 3)
    stream = torch.cuda.current_stream(dev)
    h_lat, h_win = lat_h.pin_memory(), torch.empty((B, k, 6), dtype=torch.int32).pin_memory()
    gio = io_graph(body, [(lat, h_lat)], [(h_win, win)])
    w.copy_(w0)
    gio.replay()  # warm-up
    evs = []
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        gio.replay()
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    clk = clocks.stop()
    e2e_ms = float(sum(a.elapsed_time(b) for a, b in evs) / args.steps)
    _, bf16, _, src = peaks()
    flops = 2.0 * B * T * O * I_
    if prec == "exact":
        ach = flops / (live["fc"] * 1e-3) / 1e12
        roof = {"bound": "tensor", "kernel": "conv_tc_kernel (FC as 1x1 conv)", "achieved": ach,
                "peak": bf16 * INT8_OVER_BF16, "unit": "TFLOP/s", "frac": ach / (bf16 * INT8_OVER_BF16),
                "traffic": None, "algorithmic_flops_per_launch": flops, "launch_ms": live["fc"],
                "peak_note": "int8 dense (measured bf16 x 2); an FC layer is one pixel per sample, so the "
                             "time-tiled M tile (8 pixels x 16 steps) holds one valid pixel: ceiling 1/8 of 1/3"}
    else:
        adds = float((lat < T).sum().item()) * O
        sm = clk.get("sm_mhz") or 1965.0
        peak_g = 148 * SMEM_WORDS_PER_CLK_SM * sm * 1e6 / 1e9
        ach = adds / (live["fc"] * 1e-3) / 1e9
        roof = {"bound": "alu", "kernel": "conv_event_kernel (FC as 1x1 conv)", "achieved": ach, "peak": peak_g,
                "unit": "Gadd/s", "frac": ach / peak_g, "traffic": None, "launch_ms": live["fc"]}
    cpu = None
    if not args.no_cpu_baseline:
        import oracle
        n = 64
        t0 = time.perf_counter()
        S = oracle.lat_to_dense(lat_h[:n].numpy(), T)
        P = oracle.fc(S, W)
        Q = oracle.threshold(P, cfg["theta"])
        wn, nw = oracle.fcwta(Q, k, r)
        oracle.fc_stdp(W, S, wn, nw, [tuple(c) for c in cfg["stdp"]])
        dt = time.perf_counter() - t0
        cpu = {"value": n / dt, "unit": "images/s", "cores": 1, "kind": "oracle", **host_info(),
               "sample": f"{n} rows, one FC train step of the plain oracle, 1 host thread, {dt:.2f} s"}
    fc_zca_line(args, cfg, B / (ms * 1e-3), ms, e2e_ms, h_lat.numel(), h_win.numel() * 4, launches, roof, live, clk,
                cpu, {"engine": prec, "I": I_, "O": O})


def run_zca(args, cfg):
    """NEXT-4 ZCA: fit once (reported), timed step = apply to the batch."""
    import torch

    import synth
    from paper_2301_13659_b200 import spk

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    B = cfg["batch"]
    x_h = torch.from_numpy((synth.images(cfg, 0, B).reshape(B, -1).astype(np.float32) / np.float32(255)))
    F = x_h.shape[1]
    x = x_h.to(dev)
    torch.cuda.synchronize()
    _trace("zca fit")
    t0 = time.perf_counter()
    mean, wz = spk.zca_fit(x, cfg["eps"])
    _trace("zca fit done")
    fit_s = time.perf_counter() - t0
    y = torch.empty_like(x)

    def body(mark):
        spk.zca_apply(x, mean, wz, out=y)
        mark("zca_apply")

    n0 = spk.launch_count()
    body(lambda n: None)
    torch.cuda.synchronize()
    launches = spk.launch_count() - n0
    graph, ms, live, clocks, flush = timed_graph(args, body, dev, 1)
    stream = torch.cuda.current_stream(dev)
    h_x, h_y = x_h.pin_memory(), torch.empty_like(x_h).pin_memory()
    evs = []
    for _ in range(args.steps):  # copies around the graph: measured no slower than one I/O graph here
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        x.copy_(h_x, non_blocking=True)
        graph.replay()
        h_y.copy_(y, non_blocking=True)
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    clk = clocks.stop()
    e2e_ms = float(sum(a.elapsed_time(b) for a, b in evs) / args.steps)
    sm = clk.get("sm_mhz") or 1965.0
    peak = 148 * 128 * 2 * sm * 1e6 / 1e12  # FP32 FMA lanes x 2 flop at the sampled clock
    flops = 2.0 * B * F * F
    ach = flops / (live["zca_apply"] * 1e-3) / 1e12
    roof = {"bound": "alu", "kernel": "zca_apply_kernel (fp32 CUDA-core GEMM)", "achieved": ach, "peak": peak,
            "unit": "TFLOP/s", "frac": ach / peak, "traffic": None, "algorithmic_flops_per_launch": flops,
            "launch_ms": live["zca_apply"],
            "peak_note": "148 SMs x 128 fp32 FMA lanes x 2 flop at the sampled SM clock (fp32 so the whitened "
                         "values keep the oracle's 1e-4 tolerance; tf32 tensor cores would not)"}
    cpu = None
    if not args.no_cpu_baseline:
        from threadpoolctl import threadpool_limits

        from oracle import zca as ozca
        with threadpool_limits(1):
            mu, Wz = ozca.fit(x_h.numpy().astype(np.float64), cfg["eps"])
            t0 = time.perf_counter()
            ozca.apply(x_h.numpy(), mu, Wz)
            dt = time.perf_counter() - t0
        cpu = {"value": B / dt, "unit": "images/s", "cores": 1, "kind": "oracle", **host_info(),
               "sample": f"apply to the {B}-image batch, numpy fp64 (1 BLAS thread), {dt:.3f} s"}
    fc_zca_line(args, cfg, B / (ms * 1e-3), ms, e2e_ms, h_x.numel() * 4, h_y.numel() * 4, launches, roof, live, clk,
                cpu, {"F": F, "eps": cfg["eps"], "fit_s": fit_s})


def main():
    args = parse()
    if os.environ.get("SPK_BENCH_WATCHDOG"):  # debugging aid: dump every thread's stack, then exit
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["SPK_BENCH_WATCHDOG"]), exit=True)
    import synth

    cfg = synth.load_config(args.config)
    if args.impl == "reference":
        return run_reference(args, cfg)
    if cfg.get("kind") == "fc":
        return run_fc(args, cfg)
    if cfg.get("kind") == "zca":
        return run_zca(args, cfg)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)

    import torch
    import torch.distributed as dist

    from paper_2301_13659_b200 import spk
    from paper_2301_13659_b200.network import Network, RateNetwork

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        t = torch.ones(1, device=dev)
        dist.all_reduce(t)  # communicator up before timing
        print(f"bench.py rank {rank}/{world}: NCCL communicator initialised on cuda:{local} "
              f"({torch.cuda.get_device_name(dev)}), all_reduce check {int(t.item())} == {world}",
              file=sys.stderr, flush=True)

    from paper_2301_13659_b200 import parallel

    T = cfg["T"]
    rate = cfg.get("coding") == "rate"
    forward = cfg["timed"] == "forward"
    if forward:
        # sharded batched forward: the global batch is split across ranks (strong scaling)
        start, B = parallel.shard_range(cfg["batch"], world, rank)
    else:
        # training: per-GPU batch fixed (weak scaling); data-parallel by default at N > 1
        B = cfg["batch"]
        start = rank * B
    imgs = synth.images_parallel(cfg, start, B)
    labels = synth.labels(cfg, start, B)
    Ws = synth.layer_weights(cfg)
    if rate:
        net = RateNetwork(cfg, B, device=dev, prec=args.prec, start=start)
    else:
        net = Network(cfg, B, device=dev, prec=args.prec)
    dp = (not forward) and (args.dp or (world > 1 and not args.replicas))
    if dp:
        net.enable_dp(start, B * world, parallel.allgather_equal)
    # NCCL collectives stay outside CUDA graphs: a data-parallel step at N > 1 runs eagerly
    use_graph = not (dp and world > 1)
    net.img.copy_(torch.from_numpy(imgs))
    if hasattr(net, "labels"):
        net.labels.copy_(torch.from_numpy(labels))
    net.set_weights([torch.from_numpy(w) for w in Ws])
    stream = torch.cuda.current_stream(dev)
    bcast_ms = 0.0
    if forward and world > 1:
        # rank 0's weights reach every rank over NCCL (timed apart from the step)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        parallel.broadcast_weights(net.weights)
        e1.record(stream)
        torch.cuda.synchronize()
        bcast_ms = e0.elapsed_time(e1)
        net.set_weights([w.clone() for w in net.weights])  # re-pack the broadcast weights

    # kernels per step (counted at the ABI)
    n0 = spk.launch_count()
    net.step()
    torch.cuda.synchronize()
    launches_per_step = spk.launch_count() - n0

    net.set_weights([torch.from_numpy(w) for w in Ws])
    # stage boundaries as external event nodes inside the graph: the dominant kernel's
    # duration is measured live in every timed step (on the launching stream)
    gmarks = []

    def gmark(name):
        e = torch.cuda.Event(enable_timing=True, external=True)
        e.record(torch.cuda.current_stream(dev))
        gmarks.append((name, e))

    if use_graph:
        net.capture(warmup=1, mark=gmark)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    for _ in range(args.warmup):
        if use_graph:
            net.replay()
        else:
            net.step()
    torch.cuda.synchronize()

    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = []
    live_ms = {}
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if use_graph:
            net.replay()
        else:
            gmarks.clear()
            net.step_marked(gmark)
        e1.record(stream)
        evs.append((e0, e1))
        e1.synchronize()  # the graph's stage events are reused by the next replay
        for (n1, m1), (n2, m2) in zip(gmarks[:-1], gmarks[1:]):
            live_ms.setdefault(n2, []).append(m1.elapsed_time(m2))
    torch.cuda.synchronize()
    live_ms = {k: float(np.mean(v)) for k, v in live_ms.items()}
    if world > 1:
        dist.barrier()
    ms = float(sum(a.elapsed_time(b) for a, b in evs) / args.steps)

    # end to end through the public API: pinned host images in, winners (or features) out, every step
    h_img = torch.from_numpy(imgs).pin_memory()
    h_lab = torch.from_numpy(labels).pin_memory()
    train = hasattr(net, "win") and not forward
    h_win = torch.empty(net.win.shape, dtype=torch.int32).pin_memory() if train else None
    h_nwin = torch.empty(net.nwin.shape, dtype=torch.int32).pin_memory() if train else None
    h_feat = None if train else torch.empty(net.features.shape, dtype=torch.float32).pin_memory()
    e2e_evs = []
    io_in = [(net.img, h_img)] + ([(net.labels, h_lab)] if cfg["learning"] == "rstdp" else [])
    io_out = [(h_win, net.win), (h_nwin, net.nwin)] if h_win is not None else [(h_feat, net.features)]
    if use_graph:  # the public API's host-to-host step: copies in, the step, copies out, one graph
        net.capture_io(io_in, io_out)
        net.replay_io()  # warm-up replay (one more STDP update; the timed steps below measure the same work)
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if use_graph:
            net.replay_io()
        else:
            for dst, src in io_in:
                dst.copy_(src, non_blocking=True)
            net.step()
            for dst, src in io_out:
                dst.copy_(src, non_blocking=True)
        e1.record(stream)
        e2e_evs.append((e0, e1))
    torch.cuda.synchronize()
    clk = clocks.stop()
    e2e_ms = float(sum(a.elapsed_time(b) for a, b in e2e_evs) / args.steps)
    h2d = h_img.numel() + (h_lab.numel() * 4 if cfg["learning"] == "rstdp" else 0)
    d2h = (h_win.numel() * 4 + h_nwin.numel() * 4) if h_win is not None else h_feat.numel() * 4

    if world > 1:
        t = torch.tensor([ms, e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_ms = float(t[0]), float(t[1])

    if rank == 0:
        hbm, bf16, bf16_sus, src = peaks()
        # dominant kernel: the conv stage with the largest share of the step
        convs = {k: v for k, v in live_ms.items() if k.startswith("conv")}
        dom = max(convs, key=convs.get)
        li = int(dom[4:])
        rec = net.layers[li]
        Bk = B * T if rate else B  # samples of that launch (rate coding: one image per step, T' = 1)
        Tk = 1 if rate else T
        flops = 2.0 * Bk * Tk * rec["Ho"] * rec["Wo"] * rec["geom"].Co * (rec["geom"].Ci * rec["geom"].Kh *
                                                                          rec["geom"].Kw)
        achieved = flops / (convs[dom] * 1e-3) / 1e12
        peak = bf16 * INT8_OVER_BF16
        traffic = None
        tf = ROOT / "profiles" / "ncu_traffic.json"
        if tf.exists():
            traffic = json.loads(tf.read_text()).get(f"{cfg['name']}:{dom}")
        total_imgs = cfg["batch"] if forward else world * B
        if rec["prec"] == "event":
            # event form on CUDA cores: one shared-memory weight read + integer add per active synapse
            g = rec["geom"]
            x = net.input_of(li)
            x = x.reshape((g.B, g.Ci, g.Hi, g.Wi))
            act = (x < g.T).float().sum(dim=1, keepdim=True)
            ones = torch.ones((1, 1, g.Kh, g.Kw), device=act.device)
            adds = float(torch.nn.functional.conv2d(act, ones, stride=(g.Sh, g.Sw), padding=(g.Ph, g.Pw))
                         .sum().item()) * g.Co
            sm_mhz = clk.get("sm_mhz") or 1965.0
            peak_g = 148 * SMEM_WORDS_PER_CLK_SM * sm_mhz * 1e6 / 1e9
            ach_g = adds / (convs[dom] * 1e-3) / 1e9
            roof = {"bound": "alu", "kernel": f"conv_event_kernel ({dom})", "achieved": ach_g, "peak": peak_g,
                    "unit": "Gadd/s", "frac": ach_g / peak_g, "traffic": traffic,
                    "peak_note": "148 SMs x 32 four-byte shared-memory weight reads/clk (128 B/clk/SM) at the "
                                 "sampled SM clock; one read + int add per active synapse (DESIGN §5.1b)",
                    "algorithmic_adds_per_launch": adds, "launch_ms": convs[dom]}
        else:
            roof = {"bound": "tensor", "kernel": f"conv_tc_kernel ({dom})",
                    "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                    "traffic": traffic,
                    "peak_note": f"int8 dense = {src} bf16 burst {bf16} x {INT8_OVER_BF16} (nominal 4.5/2.25); "
                                 "the exact path issues one int8 MMA per live digit plane per algorithmic MAC "
                                 "(3 for fp32 weights: ceiling 1/3; 1 for quantized binary weights)",
                    "algorithmic_flops_per_launch": flops, "launch_ms": convs[dom]}
        sb = stage_bytes(net, cfg, B)
        hbm_frac = {k: {"bytes": v, "ms": live_ms[k], "GBps": v / (live_ms[k] * 1e-3) / 1e9,
                        "frac": v / (live_ms[k] * 1e-3) / 1e9 / hbm}
                    for k, v in sb.items() if k in live_ms and live_ms[k] > 0}
        line = {
            "metric": METRIC,
            "value": total_imgs / (ms * 1e-3),
            "unit": "images/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong" if forward else "weak",
            "vs_baseline": None,
            "dtype": ("int32/int64 exact: u8 spikes x 23-bit fixed-point weights" if args.prec != "fp32" else "f32"),
            "data": "synthetic (seeded images, N(mean, std) initial weights" +
                    (", quantized to {0,1} (Listing 4)" if any(L.get("quantize") for L in cfg["layers"]) else "") + ")",
            "config": {"workload": f"{cfg['name']}: {cfg['about']}", "global_batch": total_imgs, "per_gpu_batch": B,
                       "T": T, "precision": args.prec,
                       "conv_engines": {f"conv{i}": r["prec"] for i, r in enumerate(net.layers)},
                       "parallelism": (f"dp{world}: image shards, NCCL weight broadcast ({bcast_ms:.3f} ms, untimed)"
                                       if forward else
                                       f"dp{world}: one model, mini-batch STDP over {world * B} images, all-gather of "
                                       "winners + trained-layer input maps (NCCL), identical update on every rank"
                                       if dp else f"replicas x{world} (no data-path collective)"),
                       "l2": "flushed between timed steps (256 MiB write)", "cuda_graph": use_graph},
            "e2e": {"value": total_imgs / (e2e_ms * 1e-3), "unit": "images/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches_per_step * args.steps),
            "roofline": roof,
            "hbm_frac": hbm_frac,
            "hbm_frac_note": f"algorithmic bytes per stage (SURVEY §8(d)-2) / live stage time, against {hbm} GB/s",
            "stage_ms": live_ms,
            "stage_ms_note": "per-stage device time inside the timed graph replays (external event nodes)",
            "clocks": clk,
        }
        if not args.no_cpu_baseline and world == 1:  # the oracle baseline is an N = 1 figure
            line["cpu_baseline"] = cpu_baseline(cfg, 1 if cfg.get("cpu_crop") else 2 if rate else args.cpu_sample)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
