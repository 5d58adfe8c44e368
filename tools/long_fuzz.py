"""Long seeded fuzz of the GPU searches against the oracle (the test suite runs 96 cases of the
same generator, tests/test_fuzz_gpu.py): random frame sizes (ragged tiles, frames smaller
than a tile), windows 1..32, both block sizes, mixed content (noise, flat, binary ties,
translated and shifted textures), 1-3 pairs per launch; every algorithm (DCDS, DCDS^S, CDS,
DS, h-/v-HEXBS, and FS where the oracle is cheap) bit for bit on mv / SAD / points and the
per-pair statistics.  The oracle side runs in one process per host core.

  python tools/long_fuzz.py [--cases 3000] [--seed0 10000] [--out f.json]

Test infrastructure (it imports oracle/).
"""
import argparse
import json
import os
import sys
import time
from multiprocessing import get_context

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

ALGS = ["dcds", "dcds_s", "cds", "ds", "hexbs_h", "hexbs_v"]


def make_case(case):
    from paper_0806_0689_b200 import synth
    rng = np.random.default_rng(806689 + case)
    B = int(rng.choice([8, 16]))
    W = 16 * int(rng.integers(1, 21))
    H = B * int(rng.integers(1, 22 if B == 8 else 12))
    p = int(rng.choice([1, 2, 3, 4, 5, 6, 7, 8, 9, 12, 15, 16, 17, 20, 24, 31, 32]))
    npairs = int(rng.integers(1, 4))
    kinds = rng.choice(["noise", "flat", "binary", "translated", "texture"], npairs)
    pairs = []
    for i, k in enumerate(kinds):
        seed = 1000 * case + i
        if k == "noise":
            pr = synth.random_pair(W, H, seed)
        elif k == "flat":
            pr = synth.flat_pair(W, H, int(rng.integers(0, 256)))
        elif k == "binary":
            pr = synth.binary_pair(W, H, seed)
        else:
            tex = synth.texture(W, H, (1.5, 4.0), seed).numpy()
            if k == "translated":
                pr = synth.translated_pair(tex, int(rng.integers(-6, 7)), int(rng.integers(-6, 7)))
            else:
                cur = np.clip(tex.astype(np.int16) + rng.integers(-6, 7, tex.shape), 0, 255).astype(np.uint8)
                pr = (cur, np.ascontiguousarray(np.roll(tex, (int(rng.integers(-3, 4)), int(rng.integers(-9, 10))), (0, 1))))
        pairs.append(np.stack(pr))
    return B, p, np.stack(pairs), [str(k) for k in kinds]


def oracle_case(arg):
    """the oracle's outputs of one case: {alg: [(mv, sad, pts, stats) per pair]}"""
    case, host, B, p = arg
    import oracle
    out = {}
    algs = ALGS + (["fs"] if p <= 16 and host.shape[2] * host.shape[3] <= 160 * 160 else [])
    for alg in algs:
        res = []
        for t in range(host.shape[0]):
            if alg == "fs":
                mv, sad, pts = oracle.fullsearch(host[t, 0], host[t, 1], B, p)
            else:
                mv, sad, pts = oracle.bma(host[t, 0], host[t, 1], B, p, alg)
            sse = oracle.mc_psnr(host[t, 0], host[t, 1], B, mv)[1]
            res.append((mv, sad, pts, (int(pts.astype(np.int64).sum()), int(sad.astype(np.int64).sum()), int(sse))))
        out[alg] = res
    return case, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=3000)
    ap.add_argument("--seed0", type=int, default=10000, help="first case index (the tests use 0..95)")
    ap.add_argument("--out", default="")
    ap.add_argument("--procs", type=int, default=len(os.sched_getaffinity(0)))
    args = ap.parse_args()
    import torch
    import oracle
    import paper_0806_0689_b200 as me
    oracle.build()
    me.me_init(0)
    me.me_set_stream(torch.cuda.current_stream())
    t0 = time.time()
    cases = {}
    for c in range(args.seed0, args.seed0 + args.cases):
        cases[c] = make_case(c)
    gpu = {}
    for c, (B, p, host, kinds) in cases.items():
        fr = torch.from_numpy(host.copy()).cuda()
        n, _, H, W = host.shape
        nb = (W // B) * (H // B)
        r = {}
        for alg in ALGS + ["fs"]:
            mv, sad, pts, st = me.alloc_outputs(n, nb, "cuda")
            if alg == "fs":
                me.me_fullsearch_batch(fr, B, p, mv, sad, pts, st)
            else:
                me.me_bma_batch(alg, fr, B, p, mv, sad, pts, st)
            r[alg] = (mv, sad, pts, st)
        torch.cuda.synchronize()
        gpu[c] = {k: tuple(x.cpu().numpy() for x in v) for k, v in r.items()}
    bad = []
    checked = 0
    blocks = 0
    with get_context("spawn").Pool(args.procs) as pool:
        work = [(c, cases[c][2], cases[c][0], cases[c][1]) for c in cases]
        for c, out in pool.imap_unordered(oracle_case, work, chunksize=4):
            B, p, host, kinds = cases[c]
            for alg, res in out.items():
                gmv, gsad, gpts, gst = gpu[c][alg]
                for t, (mv, sad, pts, st) in enumerate(res):
                    checked += 1
                    blocks += len(sad)
                    ok = ((gmv[t] == mv).all() and (gsad[t].astype(np.uint32) == sad).all()
                          and (gpts[t].astype(np.uint16) == pts).all()
                          and tuple(int(x) for x in gst[t].astype(np.uint64)) == st)
                    if not ok:
                        bad.append({"case": c, "alg": alg, "pair": t, "W": host.shape[3], "H": host.shape[2],
                                    "B": B, "p": p, "kind": kinds[t]})
    res = {"cases": args.cases, "first_case": args.seed0, "pair_checks": checked, "blocks_checked": blocks,
           "mismatches": bad, "seconds": round(time.time() - t0, 1), "procs": args.procs}
    print(json.dumps({k: v for k, v in res.items() if k != "mismatches"}), "mismatches:", len(bad))
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)
    sys.exit(0 if not bad else 1)


if __name__ == "__main__":
    main()
