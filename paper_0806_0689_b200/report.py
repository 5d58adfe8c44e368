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


# The paper's Table IX compares DCDS with the other BMAs on the same sequences;
# ALGS of the comparison (me.ALGS names) in the order the report prints them.
TABLE9_ALGS = ("dcds", "dcds_s", "cds", "ds", "hexbs_h", "hexbs_v")


def compare_bmas(frames: torch.Tensor, B: int, p: int, algs=TABLE9_ALGS, fs: bool = True, reps: int = 0):
    """Table-IX-style rows (MAD, MSE, NSP, PSNR, distance and hit probability against FS) of
    every algorithm on device frames [n, 2, H, W], plus the NSP speed-up of DCDS over each
    (NSP_alg / NSP_DCDS - 1, the paper's "up to 54.9%" measure, P:9).  With reps > 0
    each search is also timed (CUDA events, mean of reps launches) -> "blocks_per_s"."""
    n, _, H, W = frames.shape
    nb = (W // B) * (H // B)
    f = me.alloc_outputs(n, nb, frames.device)
    me.me_fullsearch_batch(frames, B, p, *f)
    out = {}
    for alg in algs:
        d = me.alloc_outputs(n, nb, frames.device)
        me.me_bma_batch(alg, frames, B, p, *d)
        q = me.me_quality_batch(d[0], f[0])
        torch.cuda.synchronize()
        row = sequence_means(pair_rows(d[3], q, W, H, B))
        if reps:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                me.me_bma_batch(alg, frames, B, p, *d)
            b.record()
            torch.cuda.synchronize()
            row["blocks_per_s"] = n * nb * reps / (a.elapsed_time(b) * 1e-3)
        out[alg] = row
    if fs:
        torch.cuda.synchronize()
        out["fs"] = sequence_means(pair_rows(f[3], me.me_quality_batch(f[0], f[0]), W, H, B))
    if "dcds" in out:
        base = out["dcds"]["nsp"]
        for alg, row in out.items():
            row["nsp_speedup_of_dcds"] = row["nsp"] / base - 1.0
    return out


def pair_series(frames: torch.Tensor, B: int, p: int, algs=("dcds", "dcds_s", "fs"), first_frame: int = 1):
    """Per-pair (per-frame) series of the paper's frame-wise comparison (Figs. 8-9:
    PSNR and NSP frame by frame; plus MAD, MSE, distance and probability against FS): a list of
    {"frame", "algorithm", "mad", "mse", "nsp", "psnr_db", "dist", "prob"} in frame order, the
    frame number of pair t being first_frame + t (the current frame of the pair)."""
    n, _, H, W = frames.shape
    nb = (W // B) * (H // B)
    f = me.alloc_outputs(n, nb, frames.device)
    me.me_fullsearch_batch(frames, B, p, *f)
    per = {}
    for alg in algs:
        if alg == "fs":
            d = f
        else:
            d = me.alloc_outputs(n, nb, frames.device)
            me.me_bma_batch(alg, frames, B, p, *d)
        q = me.me_quality_batch(d[0], f[0])
        torch.cuda.synchronize()
        per[alg] = pair_rows(d[3], q, W, H, B)
    out = []
    for t in range(n):
        for alg in algs:
            out.append({"frame": first_frame + t, "algorithm": alg, **per[alg][t]})
    return out


def series_csv(rows) -> str:
    """SPEC's per-frame CSV layout: frame, algorithm, mad, mse, nsp, psnr_db, dist,
    prob with 6 decimals and an `inf` sentinel for an exact match."""
    lines = ["frame,algorithm,mad,mse,nsp,psnr_db,dist,prob"]
    for r in rows:
        ps = "inf" if math.isinf(r["psnr_db"]) else f"{r['psnr_db']:.6f}"
        lines.append(f"{r['frame']},{r['algorithm']},{r['mad']:.6f},{r['mse']:.6f},{r['nsp']:.6f},{ps},"
                     f"{r['dist']:.6f},{r['prob']:.6f}")
    return "\n".join(lines) + "\n"
