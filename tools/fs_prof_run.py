import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_0806_0689_b200 as me
from paper_0806_0689_b200 import synth
me.me_init(0); me.me_set_stream(torch.cuda.current_stream())
cfg = synth.CONFIGS[sys.argv[1]]
fr = synth.make_sequence(cfg, device="cuda:0", pairs=range(1, 5))
o = me.alloc_outputs(4, cfg.nb, "cuda:0")
for _ in range(3): me.me_fullsearch_batch(fr, cfg.B, cfg.p, *o)
torch.cuda.synchronize()
