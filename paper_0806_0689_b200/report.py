"""Table-IX-style per-pair quality report (MAD, MSE, NSP, PSNR, distance to the FS MVs,
probability of finding them) from the device outputs of the searches.

Host-side formatting of the per-pair sums the kernels produce (stats_out of me_dcds_batch /
me_fullsearch_batch and me_quality_batch); the sequence value of each column is the mean of
the per-pair values (reading C18, consistent with Table IX).
"""
from __future__ import annotations

import math

import torch

from . import me


def pair_rows(stats, quality, W: int, H: int, B: int):
    """stats: [n, 3] (sum points, sum SAD, SSE); quality: [n, 2] (hits, sum distance) or None."""
    nb = (W // B) * (H // B)
    st = stats.detach().cpu().tolist()
    q = quality.detach().cpu().tolist() if quality is not None else [[float(nb), 0.0]] * len(st)
    rows = []
    for (pts, sad, sse), (hits, dsum) in zip(st, q):
        rows.append({
            "mad": sad / (nb * B * B),
            "mse": sse / (W * H),
            "nsp": pts / nb,
            "psnr_db": math.inf if sse == 0 else 10.0 * math.log10(255.0 * 255.0 * W * H / sse),
            "dist": dsum / nb,
            "prob": hits / nb,
        })
    return rows


def sequence_means(rows):
    keys = ("mad", "mse", "nsp", "psnr_db", "dist", "prob")
    out = {k: sum(r[k] for r in rows) / len(rows) for k in keys if k != "psnr_db"}
    finite = [r["psnr_db"] for r in rows if math.isfinite(r["psnr_db"])]
    out["psnr_db"] = sum(finite) / len(finite) if finite else math.inf
    out["psnr_inf_pairs"] = len(rows) - len(finite)
    return out


def compare_dcds_fs(frames: torch.Tensor, B: int, p: int):
    """Run DCDS and FS on device frames [n, 2, H, W]; return the Table-IX rows of both."""
    n, _, H, W = frames.shape
    nb = (W // B) * (H // B)
    d = me.alloc_outputs(n, nb, frames.device)
    f = me.alloc_outputs(n, nb, frames.device)
    me.me_dcds_batch(frames, B, p, *d)
    me.me_fullsearch_batch(frames, B, p, *f)
    q = me.me_quality_batch(d[0], f[0])
    qfs = me.me_quality_batch(f[0], f[0])
    torch.cuda.synchronize()
    return {"DCDS": sequence_means(pair_rows(d[3], q, W, H, B)),
            "FS": sequence_means(pair_rows(f[3], qfs, W, H, B))}
