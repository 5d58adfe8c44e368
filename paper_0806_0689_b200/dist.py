"""Multi-GPU plumbing for the DCDS batch path (BASELINE.json north_star).

Frame pairs are independent units (every block's search depends only on its own pair),
so ranks shard pairs with no data-path exchange.  The only collective gathers the per-pair
outputs -- the MV field (mv, SAD, points per block) and the per-pair statistics
(sum points, sum SAD, SSE) -- with NCCL (torch.distributed) over NVLink.  This module holds
the host logic (sharding, padded all_gather, reassembly) so it can be tested with the gloo
backend on CPU; it contains none of the method's arithmetic.
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
