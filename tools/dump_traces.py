"""Dump DCDS pass traces (me_dcds_trace_batch) of a few pairs of a config, for offline
simulation of the kernel's shared-memory access pattern (tools/sim_banks.py)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_0806_0689_b200 as me
from paper_0806_0689_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--pairs", default="0,1")
ap.add_argument("--cap", type=int, default=40)
ap.add_argument("--out", default="gpurun_out/traces_c3.npz")
args = ap.parse_args()
cfg = synth.CONFIGS[args.config]
pairs = [int(x) for x in args.pairs.split(",")]
me.me_init(0)
me.me_set_stream(torch.cuda.current_stream())
fr = synth.make_sequence(cfg, device="cuda", pairs=pairs)
n = len(pairs)
mv, sad, pts, _ = me.alloc_outputs(n, cfg.nb, "cuda", stats=False)
tr = torch.zeros(n, cfg.nb, args.cap, dtype=torch.int64, device="cuda")
tl = torch.zeros(n, cfg.nb, dtype=torch.int16, device="cuda")
me.me_dcds_trace_batch(0, fr, cfg.B, cfg.p, mv, sad, pts, tr, tl)
torch.cuda.synchronize()
np.savez_compressed(args.out, trace=tr.cpu().numpy(), tlen=tl.cpu().numpy(), pts=pts.cpu().numpy(),
                    W=cfg.W, H=cfg.H, B=cfg.B, p=cfg.p)
print("saved", args.out, "max passes", int(tl.max()))
