"""The paper's network steps composed from libspk calls (configs/*.json).

* front end   Listing 1: DoG/LoG/Gabor filter -> threshold -> rank code
* inference   Listing 5: [conv -> fire -> pool] * L -> gather
* train layer Listing 3: forward to the layer's input, conv ->
              threshold/fire record (lat, P*) -> inhibit -> convwta -> stdp
* R-STDP      P:L180-194: winners routed to reward/punish configs by label

Buffers are allocated once per (config, batch) so a step can be captured in a
CUDA graph; every stage is a libspk kernel.
"""
from __future__ import annotations

import torch

from . import spk


def _nomark(name: str) -> None:
    pass


class Network:
    def __init__(self, cfg: dict, batch: int, device="cuda", prec: str = "exact", fuse_inhibit: bool = True):
        """prec: "exact" (tcgen05 EXACT_I8 for every conv), "event" (latency-sorted form
        on CUDA cores where its weight block fits), "auto" (event for the first layer and
        for narrow layers, Co <= 64; tensor cores otherwise) or "fp32".  exact/event/auto
        give bit-identical outputs."""
        self.cfg = cfg
        self.B = batch
        self.T = cfg["T"]
        self.dev = torch.device(device)
        self.prec = prec
        # trained layer: inhibition fused into the WTA (spk_inhibit_wta; the inhibited record is
        # then not materialised) when its maps are small enough, else spk_inhibit + spk_wta
        self.fuse_inhibit = fuse_inhibit
        im, fr = cfg["image"], cfg["front"]
        self.img = torch.zeros((batch, im["C"], im["H"], im["W"]), dtype=torch.uint8, device=self.dev)
        self.labels = torch.zeros((batch,), dtype=torch.int32, device=self.dev)
        if fr["kind"] == "dog":
            self.filters = ("dog", [tuple(p) for p in fr["pairs"]])
        elif fr["kind"] == "log":
            self.filters = ("log", [float(v) for v in fr["stds"]])
        else:
            self.filters = ("gabor", [tuple(p) for p in fr["params"]])
        K = len(self.filters[1]) * (2 if self.filters[0] == "log" else 1)
        e = 2 * fr["radius"] + 1
        H, W = im["H"] + 2 * fr["pad"] - e + 1, im["W"] + 2 * fr["pad"] - e + 1
        self.y = torch.empty((batch, im["C"] * K, H, W), dtype=torch.float32, device=self.dev)
        self.lat0 = torch.empty((batch, im["C"] * K, H, W), dtype=torch.uint8, device=self.dev)
        self.weights: list[torch.Tensor] = []
        self.layers = []
        ci, h, w = im["C"] * K, H, W
        tl = cfg.get("train_layer")
        for li, L in enumerate(cfg["layers"]):
            Ho = (h + 2 * L["pad"] - L["K"]) // L["stride"] + 1
            Wo = (w + 2 * L["pad"] - L["K"]) // L["stride"] + 1
            geom = spk.ConvGeom(batch, self.T, ci, h, w, L["Co"], L["K"], L["K"], L["stride"], L["stride"],
                                L["pad"], L["pad"])
            lp = prec
            if prec in ("auto", "event"):
                ok = spk.conv_workspace(geom, "event") > 0
                # event form where its per-active-synapse cost wins: narrow layers, and the first
                # layer, whose rank-coded input is sparse (C5 conv0: 11 % of inputs fire,
                # 304 vs 436 ms on tcgen05; C2 conv1, 46 % dense and 250 maps: 2.0 vs 1.04 ms)
                lp = "event" if ok and (prec == "event" or L["Co"] <= 64 or li == 0) else "exact"
            rec = dict(
                L=L, geom=geom, Ho=Ho, Wo=Wo, prec=lp,
                lat=torch.empty((batch, L["Co"], Ho, Wo), dtype=torch.uint8, device=self.dev),
                # P* (potential at the first crossing) is only needed by the trained layer
                pstar=(torch.empty((batch, L["Co"], Ho, Wo), dtype=torch.float32, device=self.dev)
                       if li == tl else None),
                ws=torch.empty(max(1, spk.conv_workspace(geom, lp)), dtype=torch.uint8, device=self.dev),
            )
            # weight scale: the layer's bound (STDP upper bounds of the trained layer, else the init
            # clip [0, 1]); set_weights rejects weights outside [0, w_max] (R-NONNEG)
            rec["w_max"] = max([1.0] + [float(c[3]) for c in cfg.get("stdp") or []]) if li == tl else 1.0
            # weights of every layer but the trained one are constant within a step: packed once
            rec["prepacked"] = li != tl and lp in ("exact", "event")
            rec["fused_pool"] = bool(L["pool"]) and li != tl and lp == "event" and spk.conv_fire_pool_supported(
                geom, lp, L["pool"]["kernel"], L["pool"]["stride"], L["pool"]["pad"])
            if L["pool"]:
                p = L["pool"]
                Hp = (Ho + 2 * p["pad"] - p["kernel"]) // p["stride"] + 1
                Wp = (Wo + 2 * p["pad"] - p["kernel"]) // p["stride"] + 1
                rec["pooled"] = torch.empty((batch, L["Co"], Hp, Wp), dtype=torch.uint8, device=self.dev)
                h, w = Hp, Wp
            else:
                rec["pooled"] = None
                h, w = Ho, Wo
            ci = L["Co"]
            self.layers.append(rec)
            self.weights.append(torch.zeros((L["Co"], geom.Ci, L["K"], L["K"]), dtype=torch.float32,
                                            device=self.dev))
        self.fused_inhibit = False
        if tl is not None:
            rec = self.layers[tl]
            wk = rec["L"]["wta"]
            self.fused_inhibit = fuse_inhibit and rec["Ho"] * rec["Wo"] <= 12288  # one cluster slice
            self.k = wk["count"]
            self.win = torch.empty((batch, self.k, 6), dtype=torch.int32, device=self.dev)
            self.nwin = torch.empty((batch,), dtype=torch.int32, device=self.dev)
            self.stdp_ws = torch.empty(spk.stdp_workspace(rec["geom"], self.k), dtype=torch.uint8, device=self.dev)
            self.stdp_cfg = spk.stdp_configs(cfg["stdp"])
        last = self.layers[-1]
        src = last["pooled"] if last["pooled"] is not None else last["lat"]
        self.features = torch.empty(src.shape, dtype=torch.float32, device=self.dev)
        self.graph = None
        self.dp = None

    def enable_dp(self, b0: int, batch_total: int, allgather):
        """Data-parallel mini-batch STDP (SURVEY §8(f) NEXT-2, P:L178 / R-BATCH): this replica
        forwards the samples [b0, b0 + B) of a global mini-batch of `batch_total` with the
        pre-batch weights; its winners are rebased to global sample indices and
        `allgather(dst, src)` collects every replica's winner records and trained-layer
        input latency maps in rank order, so every replica applies the same sequential
        update to the same weights — bit-identical to single-GPU training on the global
        batch, with no weight broadcast."""
        tl = self.cfg["train_layer"]
        rec = self.layers[tl]
        src = self.input_of(tl)
        self.dp = dict(
            b0=b0, Bt=batch_total, gather=allgather,
            lat=torch.empty((batch_total,) + tuple(src.shape[1:]), dtype=torch.uint8, device=self.dev),
            win=torch.empty((batch_total, self.k, 6), dtype=torch.int32, device=self.dev),
            nwin=torch.empty((batch_total,), dtype=torch.int32, device=self.dev))
        g = spk.ConvGeom(batch_total, self.T, rec["geom"].Ci, rec["geom"].Hi, rec["geom"].Wi, rec["L"]["Co"],
                         rec["L"]["K"], rec["L"]["K"], rec["L"]["stride"], rec["L"]["stride"], rec["L"]["pad"],
                         rec["L"]["pad"])
        self.stdp_ws = torch.empty(spk.stdp_workspace(g, self.k), dtype=torch.uint8, device=self.dev)

    # ------------------------------------------------------------ data in
    def set_weights(self, ws):
        for li, (rec, dst, src) in enumerate(zip(self.layers, self.weights, ws)):
            dst.copy_(torch.as_tensor(src))
            if rec["L"].get("quantize"):  # Listing 4: a layer quantized after its training
                spk.quantize(dst, *rec["L"]["quantize"])
            lo, hi = float(dst.min()), float(dst.max())
            if lo < 0.0 or hi > rec["w_max"]:
                raise ValueError(f"layer {li}: weights in [{lo}, {hi}] outside [0, w_max={rec['w_max']}] "
                                 "(the latency-map conv needs non-negative weights, R-NONNEG)")
            if rec["prepacked"]:
                spk.conv_prepack(dst, rec["geom"], rec["prec"], rec["w_max"], rec["ws"])

    def input_of(self, li: int) -> torch.Tensor:
        if li == 0:
            return self.lat0
        prev = self.layers[li - 1]
        return prev["pooled"] if prev["pooled"] is not None else prev["lat"]

    # ------------------------------------------------------------ stages
    def front(self, mark=_nomark):
        fr = self.cfg["front"]
        kind, filt = self.filters
        if kind == "dog":
            spk.dog(self.img, filt, fr["radius"], fr["pad"], out=self.y)
        elif kind == "log":
            spk.log(self.img, filt, fr["radius"], fr["pad"], out=self.y)
        else:
            spk.gabor(self.img, filt, fr["radius"], fr["pad"], out=self.y)
        mark("filter")
        spk.rank_code(self.y, self.T, fr["thresh"], fr["sort"], out=self.lat0)
        mark("rank_code")

    def layer(self, li: int, pstar: bool = False, mark=_nomark):
        rec = self.layers[li]
        L = rec["L"]
        if rec["fused_pool"] and not pstar:  # layer output only feeds the next layer: conv + pool fused
            p = L["pool"]
            spk.conv_fire_pool(self.input_of(li), self.weights[li], self.T, L["stride"], L["pad"], prec=rec["prec"],
                               theta=L["theta"], w_max=rec["w_max"], pool_kernel=p["kernel"], pool_stride=p["stride"],
                               pool_pad=p["pad"], out=rec["pooled"], ws=rec["ws"], prepacked=rec["prepacked"])
            mark(f"conv{li}")
            return
        spk.conv(self.input_of(li), self.weights[li], self.T, L["stride"], L["pad"], prec=rec["prec"], epi="fire",
                 theta=L["theta"], w_max=rec["w_max"], out0=rec["lat"], out1=rec["pstar"] if pstar else None,
                 ws=rec["ws"], want_pstar=pstar, prepacked=rec["prepacked"])
        mark(f"conv{li}")
        if rec["pooled"] is not None and not pstar:
            p = L["pool"]
            spk.pool(rec["lat"], self.T, p["kernel"], p["stride"], p["pad"], out=rec["pooled"])
            mark(f"pool{li}")

    def train_step(self, mark=_nomark):
        """Listing 3 train_layer{l} for l = cfg['train_layer'] (R-STDP if cfg['learning'] == 'rstdp')."""
        mark("start")
        self.train_forward(mark)
        self.train_update(mark)

    def train_forward(self, mark=_nomark):
        """Forward to the trained layer's (lat, P*) record -> inhibit -> convwta (-> R-STDP routing)."""
        tl = self.cfg["train_layer"]
        self.front(mark)
        for li in range(tl):
            self.layer(li, mark=mark)
        self.layer(tl, pstar=True, mark=mark)
        rec = self.layers[tl]
        L = rec["L"]
        if self.fused_inhibit:
            spk.inhibit_wta(rec["lat"], rec["pstar"], self.T, self.k, L["wta"]["radius"], win=self.win, nwin=self.nwin)
            mark("inhibit_wta")
        else:
            spk.inhibit(rec["lat"], rec["pstar"], self.T)
            mark("inhibit")
            spk.wta(rec["lat"], rec["pstar"], self.T, self.k, L["wta"]["radius"], win=self.win, nwin=self.nwin)
            mark("wta")
        if self.cfg["learning"] == "rstdp":
            spk.rstdp_route(self.win, self.nwin, self.labels, self.cfg["maps_per_class"])
            mark("rstdp_route")

    def train_update(self, mark=_nomark):
        """conv.stdp with this step's winners (after the data-parallel exchange, if enabled)."""
        tl = self.cfg["train_layer"]
        L = self.layers[tl]["L"]
        lat_in, win, nwin = self.input_of(tl), self.win, self.nwin
        if self.dp is not None:  # exchange winners + receptive-field inputs (NCCL all-gather on GPUs)
            d = self.dp
            spk.winners_rebase(self.win, self.nwin, d["b0"])
            d["gather"](d["win"], self.win)
            d["gather"](d["nwin"], self.nwin)
            d["gather"](d["lat"], lat_in)
            lat_in, win, nwin = d["lat"], d["win"], d["nwin"]
            mark("allgather")
        spk.stdp(self.weights[tl], lat_in, win, nwin, None, self.T, L["stride"], L["pad"],
                 ws=self.stdp_ws, cfg_arr=self.stdp_cfg)
        mark("stdp")

    def infer(self, mark=_nomark):
        """Listing 5: every layer conv -> fire -> pool, then gather."""
        mark("start")
        self.front(mark)
        for li in range(len(self.layers)):
            self.layer(li, mark=mark)
        last = self.layers[-1]
        src = last["pooled"] if last["pooled"] is not None else last["lat"]
        spk.gather(src, self.T, out=self.features)
        mark("gather")

    def step(self):
        self.step_marked(_nomark)

    def step_marked(self, mark):
        if self.cfg["timed"] == "train":
            self.train_step(mark)
        else:
            self.infer(mark)

    # ------------------------------------------------------------ CUDA graph
    def capture(self, warmup: int = 1, mark=None):
        """Capture one step in a CUDA graph; `mark(name)` hooks (e.g. external timing
        events) are captured with it as graph nodes."""
        s = torch.cuda.Stream(device=self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.step()
        torch.cuda.current_stream(self.dev).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step_marked(mark or _nomark)
        self.graph = g
        return g

    def replay(self):
        if self.graph is None:
            self.step()
        else:
            self.graph.replay()

    def capture_io(self, inputs, outputs):
        """Capture one step TOGETHER with its host I/O in one CUDA graph: `inputs` = [(device
        tensor, pinned host tensor)] copied in first, `outputs` = [(pinned host tensor, device
        tensor)] copied out last — a user's whole step from host buffers to host buffers is then
        one graph launch (`replay_io`) instead of separate copy calls around the step."""
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for dst, src in inputs:
                dst.copy_(src, non_blocking=True)
            self.step()
            for dst, src in outputs:
                dst.copy_(src, non_blocking=True)
        self.io_graph = g
        return g

    def replay_io(self):
        self.io_graph.replay()


class RateNetwork:
    """Rate-coded inference ("the inference is done with 300 time
    steps and rate coding"): Listing 1 front end with rate coding instead of rank order, then per
    layer conv -> fire on every step (Eq. 2 and P:L125 per step, spikes not cumulative) -> pool by
    firing rates, and the last layer's firing rates as features.

    Trains are step maps u8 [B][T][C][H][W] (0 = spike at that step), i.e. one-step latency maps:
    the conv runs on B' = B*T images with T' = 1 (include/spk.h NEXT-3).  Weights of layers with a
    "quantize" entry are quantized on the device at set_weights (Listing 4)."""

    def __init__(self, cfg: dict, batch: int, device="cuda", prec: str = "auto", start: int = 0):
        self.cfg = cfg
        self.B = batch
        self.T = T = cfg["T"]
        self.start = start  # global index of sample 0 (the rate-code stream runs over global indices)
        self.dev = torch.device(device)
        im, fr = cfg["image"], cfg["front"]
        self.img = torch.zeros((batch, im["C"], im["H"], im["W"]), dtype=torch.uint8, device=self.dev)
        K = {"log": 2 * len(fr.get("stds", [])), "dog": len(fr.get("pairs", [])),
             "gabor": len(fr.get("params", []))}[fr["kind"]]
        e = 2 * fr["radius"] + 1
        H, W = im["H"] + 2 * fr["pad"] - e + 1, im["W"] + 2 * fr["pad"] - e + 1
        self.y = torch.empty((batch, im["C"] * K, H, W), dtype=torch.float32, device=self.dev)
        self.step0 = torch.empty((batch, T, im["C"] * K, H, W), dtype=torch.uint8, device=self.dev)
        self.rc_ws = torch.empty(max(4, 4 * batch), dtype=torch.uint8, device=self.dev)
        self.layers, self.weights = [], []
        ci, h, w = im["C"] * K, H, W
        for li, L in enumerate(cfg["layers"]):
            Ho = (h + 2 * L["pad"] - L["K"]) // L["stride"] + 1
            Wo = (w + 2 * L["pad"] - L["K"]) // L["stride"] + 1
            g = spk.ConvGeom(batch * T, 1, ci, h, w, L["Co"], L["K"], L["K"], L["stride"], L["stride"], L["pad"], L["pad"])
            lp = prec
            if prec == "auto":  # one time step per row on the tensor cores (TP = 1), else the event form
                lp = "exact" if spk.conv_workspace(g, "exact") > 0 else "event"
            rec = dict(L=L, geom=g, prec=lp, Ho=Ho, Wo=Wo,
                       step=torch.empty((batch, T, L["Co"], Ho, Wo), dtype=torch.uint8, device=self.dev),
                       ws=torch.empty(max(1, spk.conv_workspace(g, lp)), dtype=torch.uint8, device=self.dev))
            p = L["pool"]
            if p:
                Hp = (Ho + 2 * p["pad"] - p["kernel"]) // p["stride"] + 1
                Wp = (Wo + 2 * p["pad"] - p["kernel"]) // p["stride"] + 1
                rec["rates"] = torch.empty((batch, L["Co"], Ho, Wo), dtype=torch.float32, device=self.dev)
                rec["pooled"] = torch.empty((batch, T, L["Co"], Hp, Wp), dtype=torch.uint8, device=self.dev)
                h, w = Hp, Wp
            else:
                rec["rates"] = rec["pooled"] = None
                h, w = Ho, Wo
            self.layers.append(rec)
            self.weights.append(torch.zeros((L["Co"], ci, L["K"], L["K"]), dtype=torch.float32, device=self.dev))
            ci = L["Co"]
        last = self.layers[-1]
        src = last["pooled"] if last["pooled"] is not None else last["step"]
        self.features = torch.empty((batch,) + tuple(src.shape[2:]), dtype=torch.float32, device=self.dev)
        self.graph = None

    def set_weights(self, ws):
        for rec, dst, src in zip(self.layers, self.weights, ws):
            L = rec["L"]
            dst.copy_(torch.as_tensor(src))
            if L.get("quantize"):
                spk.quantize(dst, *L["quantize"])
            if float(dst.min()) < 0.0 or float(dst.max()) > 1.0:
                raise ValueError("weights outside [0, 1] (R-NONNEG)")
            if rec["prec"] in ("exact", "event"):  # forward only: every layer packed once
                spk.conv_prepack(dst, rec["geom"], rec["prec"], 1.0, rec["ws"])

    def input_of(self, li: int) -> torch.Tensor:
        if li == 0:
            return self.step0
        prev = self.layers[li - 1]
        return prev["pooled"] if prev["pooled"] is not None else prev["step"]

    def front(self, mark=_nomark):
        fr = self.cfg["front"]
        if fr["kind"] == "gabor":
            spk.gabor(self.img, fr["params"], fr["radius"], fr["pad"], out=self.y)
        elif fr["kind"] == "log":
            spk.log(self.img, fr["stds"], fr["radius"], fr["pad"], out=self.y)
        else:
            spk.dog(self.img, [tuple(p) for p in fr["pairs"]], fr["radius"], fr["pad"], out=self.y)
        mark("filter")
        spk.rate_code(self.y, self.T, fr["thresh"], self.cfg["rate_seed"], b0=self.start, out=self.step0, ws=self.rc_ws)
        mark("rate_code")

    def layer(self, li: int, mark=_nomark):
        rec = self.layers[li]
        L, B, T = rec["L"], self.B, self.T
        src = self.input_of(li)
        x = src.view((B * T,) + tuple(src.shape[2:]))
        out = rec["step"].view((B * T,) + tuple(rec["step"].shape[2:]))
        spk.conv(x, self.weights[li], 1, L["stride"], L["pad"], prec=rec["prec"], epi="fire", theta=L["theta"],
                 w_max=1.0, out0=out, ws=rec["ws"], want_pstar=False, prepacked=rec["prec"] in ("exact", "event"))
        mark(f"conv{li}")
        p = L["pool"]
        if p:
            spk.rate_gather(rec["step"], out=rec["rates"])
            mark(f"rates{li}")
            if L.get("pool_rates"):
                spk.pool_rates(rec["step"], rec["rates"], p["kernel"], p["stride"], p["pad"], out=rec["pooled"])
            else:
                po = rec["pooled"].view((B * T,) + tuple(rec["pooled"].shape[2:]))
                spk.pool(out, 1, p["kernel"], p["stride"], p["pad"], out=po)
            mark(f"pool{li}")

    def infer(self, mark=_nomark):
        mark("start")
        self.front(mark)
        for li in range(len(self.layers)):
            self.layer(li, mark=mark)
        last = self.layers[-1]
        src = last["pooled"] if last["pooled"] is not None else last["step"]
        spk.rate_gather(src, out=self.features)
        mark("gather")

    def step(self):
        self.infer()

    def step_marked(self, mark):
        self.infer(mark)

    capture = Network.capture
    replay = Network.replay
    capture_io = Network.capture_io
    replay_io = Network.replay_io
