"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel host logic.

The sharded forward must be bitwise equal to the single-process forward
(SURVEY §8(e)): every rank generates its own image shard from (seed, global
index), receives rank 0's weights by broadcast, runs the per-sample path and the
gathered features equal the whole-batch result.  The per-sample compute here is
the CPU oracle (tests may use it); the GPU path is covered by -m gpu tests.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from oracle import pipeline as opipe
from paper_2301_13659_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partitions():
    for n in (1, 7, 1024, 4096, 1023):
        for world in (1, 2, 3, 4, 8):
            got = [parallel.shard_range(n, world, r) for r in range(world)]
            assert sum(c for _, c in got) == n
            assert got[0][0] == 0
            for (s0, c0), (s1, _) in zip(got, got[1:]):
                assert s1 == s0 + c0
            assert max(c for _, c in got) - min(c for _, c in got) <= 1


def test_synth_shards_are_bitwise_slices():
    cfg = synth.load_config("c2")
    full = synth.images(cfg, 0, 10)
    for world in (2, 3):
        parts = [synth.images(cfg, *parallel.shard_range(10, world, r)) for r in range(world)]
        np.testing.assert_array_equal(np.concatenate(parts), full)


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.load_config("c1")
    cfg["layers"][0]["pool"] = {"kernel": 2, "stride": 2, "pad": 0}
    n = 5
    start, count = parallel.shard_range(n, world, rank)
    imgs = synth.images(cfg, start, count)
    # rank 0 owns the weights; other ranks start from garbage and must receive them
    Ws = synth.layer_weights(cfg)
    w = torch.from_numpy(Ws[0].copy()) if rank == 0 else torch.full_like(torch.from_numpy(Ws[0]), -7.0)
    parallel.broadcast_weights([w])
    feat = opipe.infer(cfg, imgs, [w.numpy()], event=True)
    full = parallel.gather_rows(torch.from_numpy(feat), n)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_forward_equals_single_process(tmp_path, world):
    out = str(tmp_path / "feat.npy")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    cfg = synth.load_config("c1")
    cfg["layers"][0]["pool"] = {"kernel": 2, "stride": 2, "pad": 0}
    ref = opipe.infer(cfg, synth.images(cfg, 0, 5), synth.layer_weights(cfg), event=True)
    np.testing.assert_array_equal(np.load(out), ref)


def _dp_worker(rank, world, port, out_path, n):
    """Data-parallel mini-batch STDP: each rank forwards its shard with the
    pre-batch weights, rebases its winners to global sample indices, all-gathers winners and
    the trained layer's input trains, and applies the global sequential update."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.load_config("c1")
    start, count = parallel.shard_range(n, world, rank)
    Ws = synth.layer_weights(cfg)
    r = opipe.train_step(cfg, synth.images(cfg, start, count), Ws, event=True)
    win = r["win"].copy()
    for b in range(count):  # the product does this on the GPU (spk_winners_rebase)
        win[b, : r["nwin"][b], 0] += start
    g_win = torch.empty((n,) + win.shape[1:], dtype=torch.int32)
    g_nwin = torch.empty((n,), dtype=torch.int32)
    S_in = r["S_in"]
    g_S = torch.empty((n,) + S_in.shape[1:], dtype=torch.uint8)
    parallel.allgather_equal(g_win, torch.from_numpy(win))
    parallel.allgather_equal(g_nwin, torch.from_numpy(r["nwin"].astype(np.int32)))
    parallel.allgather_equal(g_S, torch.from_numpy(S_in.astype(np.uint8)))
    L = cfg["layers"][0]
    W = oracle.stdp(Ws[0], g_S.numpy(), g_win.numpy(), g_nwin.numpy(), [tuple(c) for c in cfg["stdp"]],
                    (L["stride"],) * 2, (L["pad"],) * 2)
    np.save(out_path.replace(".npy", f"_{rank}.npy"), W)
    dist.barrier()
    dist.destroy_process_group()


def test_data_parallel_stdp_equals_single_process(tmp_path):
    world, n = 2, 4
    out = str(tmp_path / "w.npy")
    mp.spawn(_dp_worker, args=(world, _free_port(), out, n), nprocs=world, join=True)
    cfg = synth.load_config("c1")
    ref = opipe.train_step(cfg, synth.images(cfg, 0, n), synth.layer_weights(cfg), event=True)
    assert ref["nwin"].sum() > 0
    for r in range(world):  # every replica holds the single-process batch-trained weights, bit for bit
        np.testing.assert_array_equal(np.load(out.replace(".npy", f"_{r}.npy")), ref["W_new"])
