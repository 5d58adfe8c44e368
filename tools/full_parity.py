"""Full-size parity sweep: every pair of every config, GPU (libme.so) against the oracle,
bit-exact on mv, SAD and points of every block and on the per-pair statistics (sum points, sum
SAD, SSE).  The oracle runs in one process per host core over disjoint pairs (frames shared
through shared memory), so c4's 959 2160p pairs take seconds, not minutes.

  python tools/full_parity.py [--configs c0,c1,c2,c3,c4] [--algs dcds,dcds_s,cds,ds,hexbs_h,hexbs_v,fs]
                              [--out f.json]          (fs is skipped at c4)

Test infrastructure (it imports oracle/); the pytest suites sample the large configs, this
tool covers them whole.
"""
import argparse
import json
import os
import sys
import time
from multiprocessing import get_context, shared_memory

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

_W = None


def _init(name, shape, B, p, alg):
    global _W
    import oracle
    shm = shared_memory.SharedMemory(name=name)
    _W = (shm, np.ndarray(shape, np.uint8, buffer=shm.buf), B, p, alg, oracle)


def _pair(t):
    _, fr, B, p, alg, oracle = _W
    if alg == "fs":
        mv, sad, pts = oracle.fullsearch(fr[t, 0], fr[t, 1], B, p)
    else:
        mv, sad, pts = oracle.bma(fr[t, 0], fr[t, 1], B, p, alg)
    _, sse = oracle.mc_psnr(fr[t, 0], fr[t, 1], B, mv)
    return t, mv, sad, pts, (int(pts.astype(np.int64).sum()), int(sad.astype(np.int64).sum()), int(sse))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c0,c1,c2,c3,c4")
    ap.add_argument("--algs", default="dcds,dcds_s,cds,ds,hexbs_h,hexbs_v,fs")
    ap.add_argument("--out", default="")
    ap.add_argument("--procs", type=int, default=len(os.sched_getaffinity(0)))
    args = ap.parse_args()
    import torch
    import oracle
    import paper_0806_0689_b200 as me
    from paper_0806_0689_b200 import synth
    oracle.build()
    me.me_init(0)
    me.me_set_stream(torch.cuda.current_stream())
    res = {"procs": args.procs, "configs": {}}
    for name in args.configs.split(","):
        cfg = synth.CONFIGS[name]
        fr = synth.make_sequence(cfg, device="cuda:0")
        host = fr.cpu().numpy()
        shm = shared_memory.SharedMemory(create=True, size=host.nbytes)
        np.ndarray(host.shape, np.uint8, buffer=shm.buf)[:] = host
        try:
            for alg in args.algs.split(","):
                if alg == "fs" and name == "c4":
                    continue  # 4225 candidates x 256 px x 31 M blocks: hours of oracle (tests sample it)
                mv, sad, pts, st = me.alloc_outputs(cfg.npairs, cfg.nb, "cuda:0")
                if alg == "fs":
                    me.me_fullsearch_batch(fr, cfg.B, cfg.p, mv, sad, pts, st)
                elif alg == "dcds":
                    me.me_dcds_batch(fr, cfg.B, cfg.p, mv, sad, pts, st)
                else:
                    me.me_bma_batch(alg, fr, cfg.B, cfg.p, mv, sad, pts, st)
                torch.cuda.synchronize()
                g = [mv.cpu().numpy(), sad.cpu().numpy().astype(np.uint32), pts.cpu().numpy().astype(np.uint16),
                     st.cpu().numpy().astype(np.uint64)]
                t0 = time.time()
                bad_pairs, bad_blocks = [], 0
                with get_context("spawn").Pool(args.procs, initializer=_init,
                                               initargs=(shm.name, host.shape, cfg.B, cfg.p, alg)) as pool:
                    for t, omv, osad, opts, ost in pool.imap_unordered(_pair, range(cfg.npairs), chunksize=1):
                        bb = int(((g[0][t] != omv).any(1) | (g[1][t] != osad) | (g[2][t] != opts)).sum())
                        if bb or tuple(int(x) for x in g[3][t]) != ost:
                            bad_pairs.append(t)
                            bad_blocks += bb
                r = {"pairs": cfg.npairs, "blocks": cfg.npairs * cfg.nb, "mismatched_pairs": len(bad_pairs),
                     "mismatched_blocks": bad_blocks, "oracle_seconds": round(time.time() - t0, 1),
                     "mean_nsp": float(g[2].astype(np.float64).mean())}
                res["configs"].setdefault(name, {})[alg] = r
                print(name, alg, r, flush=True)
        finally:
            shm.close()
            shm.unlink()
    ok = all(r["mismatched_blocks"] == 0 and r["mismatched_pairs"] == 0
             for c in res["configs"].values() for r in c.values())
    res["all_bit_exact"] = ok
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)
    print("ALL BIT-EXACT" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
