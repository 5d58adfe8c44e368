"""Multi-rank host logic on CPU (gloo, world_size 2): pair sharding, packed all_gather of the
per-pair MV fields + statistics, reassembly.  The per-rank search is the oracle here (no GPU);
on B200 ranks run libme.so and gather with NCCL through the same code (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_0806_0689_b200 import dist as mdist
from paper_0806_0689_b200 import synth


def test_shard_ranges():
    for n, w in [(239, 8), (959, 8), (29, 2), (1, 4), (7, 2), (16, 4)]:
        ranges = [mdist.shard(n, w, r) for r in range(w)]
        assert ranges[0][0] == 0 and ranges[-1][1] == n
        for (a, b), (c, d) in zip(ranges, ranges[1:]):
            assert b == c and a <= b
        assert max(b - a for a, b in ranges) == mdist.shard_size(n, w)


def test_pack_roundtrip():
    g = torch.Generator().manual_seed(0)
    for nb in (99, 396, 7):
        n = 3
        mv = torch.randint(-32, 33, (n, nb, 2), generator=g, dtype=torch.int16)
        sad = torch.randint(0, 65281, (n, nb), generator=g, dtype=torch.int32)
        pts = torch.randint(1, 4226, (n, nb), generator=g, dtype=torch.int16)
        st = torch.randint(0, 2**40, (n, 3), generator=g, dtype=torch.int64)
        rec = mdist.pack_fields(mv, sad, pts, st, 5)
        assert rec.shape[0] == 5
        m2, s2, p2, t2 = mdist.unpack_fields(rec[:n], nb)
        assert torch.equal(m2, mv) and torch.equal(s2, sad) and torch.equal(p2, pts) and torch.equal(t2, st)


def _oracle_fields(frames, B, p):
    mvs, sads, ptss, sts = [], [], [], []
    for t in range(frames.shape[0]):
        mv, sad, pts = oracle.dcds(frames[t, 0], frames[t, 1], B, p)
        _, sse = oracle.mc_psnr(frames[t, 0], frames[t, 1], B, mv)
        mvs.append(mv)
        sads.append(sad.astype(np.int32))
        ptss.append(pts.astype(np.int16))
        sts.append([int(pts.astype(np.int64).sum()), int(sad.astype(np.int64).sum()), sse])
    return (torch.from_numpy(np.stack(mvs)), torch.from_numpy(np.stack(sads)),
            torch.from_numpy(np.stack(ptss)), torch.tensor(sts, dtype=torch.int64))


def _worker(rank, world, port, frames, B, p, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = frames.shape[0]
    lo, hi = mdist.shard(n, world, rank)
    mv, sad, pts, st = _oracle_fields(frames[lo:hi], B, p)
    if hi == lo:
        nb = (frames.shape[3] // B) * (frames.shape[2] // B)
        mv = torch.zeros(0, nb, 2, dtype=torch.int16)
        sad = torch.zeros(0, nb, dtype=torch.int32)
        pts = torch.zeros(0, nb, dtype=torch.int16)
        st = torch.zeros(0, 3, dtype=torch.int64)
    g = mdist.gather_fields(mv, sad, pts, st, n)
    if rank == 0:
        out_q.put([t.numpy() for t in g])
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world,npairs", [(2, 7), (2, 2)])
def test_gloo_gather_matches_single_rank(world, npairs):
    cfg = synth.CONFIGS["c1"]
    frames = synth.make_sequence(cfg, pairs=range(1, npairs + 1)).numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, frames, cfg.B, cfg.p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    ref = [t.numpy() for t in _oracle_fields(frames, cfg.B, cfg.p)]
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)


def _flat_worker(rank, world, port, frames, B, p, out_q, packed=False):
    """Weak-scaling layout of bench.py: every rank searches its own n pairs into one flat
    buffer (the 10-byte arrays, or with packed=True the 6-byte transport record) and the
    buffers are all_gathered as they are."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = frames.shape[0] // world
    nb = (frames.shape[3] // B) * (frames.shape[2] // B)
    buf = mdist.alloc_flat(n, nb, "cpu", packed=packed)
    mv, sad, pts, st = mdist.flat_views(buf, n, nb, packed)
    omv, osad, opts, ost = _oracle_fields(frames[rank * n:(rank + 1) * n], B, p)
    mv.copy_(omv.to(mv.dtype)); sad.copy_(osad.to(sad.dtype)); pts.copy_(opts); st.copy_(ost)
    out = mdist.alloc_flat(n, nb, "cpu", world, packed)
    mdist.gather_flat(buf, out)
    if rank == 0:
        parts = mdist.unpack_gathered(out, n, nb, packed)
        got = [torch.cat([pr[k] for pr in parts]) for k in range(4)]
        if packed:  # back to the arrays' types (int8 MV, uint16 SAD)
            got[0] = got[0].to(torch.int16)
            got[1] = got[1].to(torch.int32) & 0xFFFF
        out_q.put([t.numpy() for t in got])
    dist.barrier()
    dist.destroy_process_group()


def test_flat_layout_alignment():
    for n, nb in [(1, 99), (3, 7), (239, 32640)]:
        o_mv, o_sad, o_pts, o_st, total = mdist.flat_layout(n, nb)
        assert o_sad % 4 == 0 and o_pts % 2 == 0 and o_st % 8 == 0 and total >= o_st + 24 * n
        o_mv, o_sad, o_pts, o_st, ptotal = mdist.flat_layout(n, nb, packed=True)
        assert o_sad % 2 == 0 and o_pts % 2 == 0 and o_st % 8 == 0 and ptotal >= o_st + 24 * n
        assert ptotal < total and o_st - 6 * n * nb < 8   # 6 bytes per block


@pytest.mark.parametrize("packed", [False, True])
def test_gloo_flat_gather_matches_single_rank(packed):
    world, n = 2, 2
    cfg = synth.CONFIGS["c1"]
    frames = synth.make_sequence(cfg, pairs=range(1, world * n + 1)).numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_flat_worker, args=(r, world, port, frames, cfg.B, cfg.p, q, packed))
             for r in range(world)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    ref = [t.numpy() for t in _oracle_fields(frames, cfg.B, cfg.p)]
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)


def _step_worker(rank, world, port, frames_all, B, p, out_q, scaling, gather, packed, npairs):
    """bench.py's multi-GPU step (GatherStep) on gloo: this rank's pairs (weak or strong
    sharding, rank_pairs) searched into the padded flat buffer (the oracle stands in for the
    kernel), then all_gather / gather-to-root; rank 0 reassembles all pairs in order."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nb = (frames_all.shape[3] // B) * (frames_all.shape[2] // B)
    mine = mdist.rank_pairs(npairs, world, rank, scaling)
    per = npairs if scaling == "weak" else mdist.shard_size(npairs, world)
    step = mdist.GatherStep(len(mine), per, nb, "cpu", world, rank, packed, gather)

    def search(mv, sad, pts, st):
        omv, osad, opts, ost = _oracle_fields(frames_all[mine.start:mine.stop], B, p)
        mv.copy_(omv.to(mv.dtype)); sad.copy_(osad.to(sad.dtype)); pts.copy_(opts); st.copy_(ost)

    for k in range(3):  # several steps: the buffers alternate
        step.step(k, search)
    step.drain()
    g = step.gathered(npairs, scaling)
    if rank == 0 or gather == "all":
        got = list(g)
        if packed:
            got[0] = got[0].to(torch.int16)
            got[1] = got[1].to(torch.int32) & 0xFFFF
        if rank == 0:
            out_q.put([t.numpy() for t in got])
    else:
        assert g is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("scaling,gather,packed,npairs", [
    ("strong", "root", True, 3),    # uneven shards: 2 + 1
    ("strong", "all", False, 3),
    ("strong", "root", False, 1),   # rank 1 has no pairs (empty shard)
    ("weak", "root", True, 2),
    ("weak", "all", True, 1),
])
def test_gloo_gather_step(scaling, gather, packed, npairs):
    world = 2
    cfg = synth.CONFIGS["c1"]
    total = npairs * world if scaling == "weak" else npairs
    frames = synth.make_sequence(cfg, pairs=range(1, total + 1)).numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, world, port, frames, cfg.B, cfg.p, q, scaling, gather,
                                                    packed, npairs)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    ref = [t.numpy() for t in _oracle_fields(frames, cfg.B, cfg.p)]
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)


def test_rank_pairs():
    assert [list(mdist.rank_pairs(5, 2, r, "strong")) for r in range(2)] == [[0, 1, 2], [3, 4]]
    assert [list(mdist.rank_pairs(3, 2, r, "weak")) for r in range(2)] == [[0, 1, 2], [3, 4, 5]]
    assert list(mdist.rank_pairs(1, 4, 3, "strong")) == []
