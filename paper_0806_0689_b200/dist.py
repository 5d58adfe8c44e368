"""Multi-GPU plumbing for the DCDS batch path (BASELINE.json north_star).

Frame pairs are independent units (every block's search depends only on its own pair),
so ranks shard pairs with no data-path exchange.  The only collective gathers the per-pair
outputs -- the MV field (mv, SAD, points per block) and the per-pair statistics
(sum points, sum SAD, SSE) -- with NCCL (torch.distributed) over NVLink, to rank 0 or to every
rank.  This module holds the host logic (sharding, padded gathers, reassembly, the
double-buffered step of bench.py) so it can be tested with the gloo backend on CPU; it contains
none of the method's arithmetic.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(npairs: int, world: int, rank: int):
    """Contiguous pair range [lo, hi) of `rank` (ceil split; trailing ranks may be short or
    empty, e.g. 239 pairs over 8 ranks = 7 x 30 + 29)."""
    per = -(-npairs // world)
    lo = min(npairs, rank * per)
    return lo, min(npairs, lo + per)


def shard_size(npairs: int, world: int) -> int:
    return -(-npairs // world)


def pack_fields(mv: torch.Tensor, sad: torch.Tensor, pts: torch.Tensor, stats: torch.Tensor,
                pad_to: int) -> torch.Tensor:
    """One contiguous int32 record per pair: [nb*2 mv (int16 pairs as int32 words) | nb sad |
    nb/2 points (int16 pairs) | 6 stats words], padded with zero pairs to `pad_to` pairs."""
    n = mv.shape[0]
    nb = mv.shape[1]
    mvw = mv.contiguous().view(n, nb * 2).view(torch.int32) if n else mv.new_zeros((0, nb), dtype=torch.int32)
    sadw = sad.contiguous().view(n, nb)
    pt = pts.contiguous().view(n, nb)
    if nb % 2:
        pt = torch.cat([pt, pt.new_zeros((n, 1))], 1)
    ptw = pt.view(torch.int32) if n else pt.new_zeros((0, (nb + 1) // 2), dtype=torch.int32)
    stw = stats.contiguous().view(n, 3).view(torch.int32) if n else stats.new_zeros((0, 6), dtype=torch.int32)
    rec = torch.cat([mvw, sadw, ptw, stw], 1)
    if n < pad_to:
        rec = torch.cat([rec, rec.new_zeros((pad_to - n, rec.shape[1]))], 0)
    return rec


def unpack_fields(rec: torch.Tensor, nb: int):
    """Inverse of pack_fields for [n, words] int32 records."""
    n = rec.shape[0]
    o = 0
    mv = rec[:, o:o + nb].contiguous().view(torch.int16).view(n, nb, 2)
    o += nb
    sad = rec[:, o:o + nb].contiguous()
    o += nb
    npw = (nb + 1) // 2
    pts = rec[:, o:o + npw].contiguous().view(torch.int16)[:, :nb]
    o += npw
    st = rec[:, o:o + 6].contiguous().view(torch.int64)
    return mv, sad, pts, st


def gather_fields(mv, sad, pts, stats, npairs_total: int, group=None):
    """all_gather the per-pair records of every rank (equal padded sizes) and return the
    concatenated (mv, sad, points, stats) of all npairs_total pairs in pair order.  Works with
    NCCL (CUDA tensors) and gloo (CPU tensors)."""
    world = dist.get_world_size(group)
    per = shard_size(npairs_total, world)
    nb = mv.shape[1]
    rec = pack_fields(mv, sad, pts, stats, per)
    out = rec.new_empty((world * per, rec.shape[1]))
    if hasattr(dist, "all_gather_into_tensor") and rec.is_cuda:
        dist.all_gather_into_tensor(out, rec, group=group)
    else:
        dist.all_gather(list(out.chunk(world, 0)), rec, group=group)
    keep = torch.cat([torch.arange(r * per, r * per + (shard(npairs_total, world, r)[1] - shard(npairs_total, world, r)[0]))
                      for r in range(world)])
    return unpack_fields(out[keep.to(out.device)], nb)


# ---------------------------------------------------------------------------------------
# Flat output buffers: the batched search writes its four outputs into ONE device buffer
# [mv | sad | points | stats], so the gather sends it as-is and the gathered result is unpacked
# by views -- no packing copies on the step's critical path (bench.py, N > 1).
# ---------------------------------------------------------------------------------------
def flat_layout(n: int, nb: int, packed: bool = False):
    """Byte offsets and total size of the flat output buffer of n pairs x nb blocks:
    mv [n, nb, 2] int16 | sad [n, nb] int32 | points [n, nb] int16 | stats [n, 3] int64, or with
    packed=True the 6-byte transport record of me_dcds_batch_packed: mv [n, nb, 2] int8 | sad
    [n, nb] uint16 | points [n, nb] uint16 | stats (stats 8-byte aligned; every part meets the C
    ABI's alignment)."""
    w_mv, w_sad = (2, 2) if packed else (4, 4)
    o_mv = 0
    o_sad = o_mv + w_mv * n * nb
    o_pts = o_sad + w_sad * n * nb
    o_st = (o_pts + 2 * n * nb + 7) & ~7
    total = o_st + 24 * n
    return o_mv, o_sad, o_pts, o_st, total


def flat_views(buf: torch.Tensor, n: int, nb: int, packed: bool = False):
    """(mv, sad, points, stats) views of a flat uint8 buffer laid out by flat_layout."""
    o_mv, o_sad, o_pts, o_st, total = flat_layout(n, nb, packed)
    assert buf.dtype == torch.uint8 and buf.numel() >= total
    if packed:
        mv = buf[o_mv:o_sad].view(torch.int8).view(n, nb, 2)
        sad = buf[o_sad:o_pts].view(torch.int16).view(n, nb)
    else:
        mv = buf[o_mv:o_sad].view(torch.int16).view(n, nb, 2)
        sad = buf[o_sad:o_pts].view(torch.int32).view(n, nb)
    pts = buf[o_pts:o_pts + 2 * n * nb].view(torch.int16).view(n, nb)
    st = buf[o_st:o_st + 24 * n].view(torch.int64).view(n, 3)
    return mv, sad, pts, st


def alloc_flat(n: int, nb: int, device, world: int = 1, packed: bool = False):
    """A flat output buffer, or the [world, size] receive buffer of its gather."""
    total = flat_layout(n, nb, packed)[4]
    return torch.empty((world, total) if world > 1 else total, dtype=torch.uint8, device=device)


def gather_flat(buf: torch.Tensor, out: torch.Tensor, group=None):
    """all_gather of every rank's flat buffer into out [world, size] (NCCL: one collective)."""
    if hasattr(dist, "all_gather_into_tensor") and buf.is_cuda:
        dist.all_gather_into_tensor(out.view(-1), buf, group=group)
    else:
        dist.all_gather(list(out.unbind(0)), buf, group=group)
    return out


def unpack_gathered(out: torch.Tensor, n: int, nb: int, packed: bool = False):
    """Per-rank (mv, sad, points, stats) views of a gathered [world, size] buffer; rank r's
    pairs are the global pairs r*n .. r*n+n-1 (weak scaling: every rank searches n pairs)."""
    return [flat_views(out[r], n, nb, packed) for r in range(out.shape[0])]


# ---------------------------------------------------------------------------------------
# The multi-GPU step of bench.py: search this rank's pairs into a flat buffer,
# then gather the buffers of all ranks -- double-buffered, the gather of step k on a comm
# stream overlapping the search of step k+1.
# ---------------------------------------------------------------------------------------
def rank_pairs(npairs: int, world: int, rank: int, scaling: str):
    """Global pair indices (0-based) this rank searches.  weak: every rank its own npairs
    pairs (rank r: r*npairs ..); strong: the configured npairs split in contiguous ceil
    shards (shard), the last ones possibly short or empty."""
    if scaling == "weak":
        return range(rank * npairs, (rank + 1) * npairs)
    lo, hi = shard(npairs, world, rank)
    return range(lo, hi)


class GatherStep:
    """One step = search of this rank's pairs (search_fn(views) writes mv / sad / points /
    stats into the views of a flat buffer of `per` pairs -- the padded shard size, so every
    rank's buffer has the same size) + the collective over that buffer:
      gather="all":  all_gather_into_tensor into [world, size] on every rank;
      gather="root": gather to rank 0 (NCCL send/recv under torch.distributed.gather), the
                     other ranks only send -- the north star's "gathered".
    With world == 1 there is no collective.  Two flat buffers alternate: the search that
    next writes a buffer waits on the event recorded after that buffer's last gather."""

    def __init__(self, n_local: int, per: int, nb: int, device, world: int, rank: int,
                 packed: bool, gather: str = "root", comm_stream=None, stream=None, nbuf=None,
                 collective: bool | None = None):
        assert gather in ("all", "root")
        self.n, self.per, self.nb, self.world, self.rank = n_local, per, nb, world, rank
        self.packed, self.gather = packed, gather
        # world == 1 has nothing to gather; collective=True runs the NCCL call anyway (tests)
        self.coll = world > 1 if collective is None else collective
        self.nbuf = nbuf or (2 if self.coll else 1)
        self.flats = [alloc_flat(per, nb, device, packed=packed) for _ in range(self.nbuf)]
        for f in self.flats:
            f.zero_()  # padding pairs of a short shard gather as zeros
        self.views = [flat_views(f, per, nb, packed) for f in self.flats]
        recv = self.coll and (gather == "all" or rank == 0)
        self.outs = ([alloc_flat(per, nb, device, world, packed).view(world, -1) for _ in range(self.nbuf)]
                     if recv else None)
        # CPU (gloo tests): synchronous, no streams or events
        self.cuda = torch.device(device).type == "cuda"
        self.stream = self.comm = None
        if self.cuda:
            self.stream = stream if stream is not None else torch.cuda.current_stream(device)
            self.comm = comm_stream
            if self.coll and self.comm is None:
                # high priority: NCCL's blocks get SM slots as soon as search CTAs retire
                self.comm = torch.cuda.Stream(device, priority=-1)
        self.ready = [torch.cuda.Event() for _ in range(self.nbuf)] if self.cuda else None
        self.freed = [torch.cuda.Event() for _ in range(self.nbuf)] if self.cuda else None
        self.used = [False] * self.nbuf
        self.last = 0

    def local_views(self, b):
        """this rank's n pairs of buffer b (the leading part of the padded buffer)"""
        mv, sad, pts, st = self.views[b]
        return mv[: self.n], sad[: self.n], pts[: self.n], st[: self.n]

    def claim(self, k: int) -> int:
        b = k % self.nbuf
        if self.used[b] and self.cuda:
            self.stream.wait_event(self.freed[b])
        return b

    def _collective(self, b: int):
        if self.gather == "all":
            gather_flat(self.flats[b], self.outs[b])
        else:
            gl = list(self.outs[b].unbind(0)) if self.rank == 0 else None
            dist.gather(self.flats[b], gl, dst=0)

    def collect(self, b: int):
        if not self.coll:
            return
        if not self.cuda:
            self._collective(b)
            return
        self.ready[b].record(self.stream)
        self.comm.wait_event(self.ready[b])
        with torch.cuda.stream(self.comm):
            self._collective(b)
        self.freed[b].record(self.comm)
        self.used[b] = True

    def step(self, k: int, search_fn):
        b = self.claim(k)
        if self.n:
            search_fn(*self.local_views(b))
        self.collect(b)
        self.last = b
        return b

    def drain(self):
        if self.cuda and self.comm is not None:
            self.stream.wait_stream(self.comm)

    def gathered(self, npairs_total: int, scaling: str):
        """(mv, sad, points, stats) of all ranks' pairs in global pair order from the last
        step's receive buffer (rank 0, or every rank with gather="all"); None elsewhere."""
        if not self.coll:
            return tuple(t.clone() for t in self.local_views(self.last))
        if self.outs is None:
            return None
        parts = [flat_views(self.outs[self.last][r], self.per, self.nb, self.packed) for r in range(self.world)]
        sizes = [len(rank_pairs(npairs_total, self.world, r, scaling)) for r in range(self.world)]
        return tuple(torch.cat([pr[k][:s] for pr, s in zip(parts, sizes)]) for k in range(4))
