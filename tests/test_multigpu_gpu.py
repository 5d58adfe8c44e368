"""The multi-GPU step of bench.py on the GPU under NCCL.

Only one GPU is available, so the NCCL process group has world size 1, but the step runs its
collective anyway (GatherStep(collective=True)): me_dcds_batch_packed writes the 6-byte
transport records into the flat buffer, NCCL gathers it (gather-to-root and all_gather), and
the gathered records, unpacked, must equal the oracle on sampled c3 blocks and the 10-byte
arrays of me_dcds_batch on every block.  Host logic at world size 2 is covered with gloo in
tests/test_dist_cpu.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import oracle
import paper_0806_0689_b200 as me
from paper_0806_0689_b200 import dist as mdist
from paper_0806_0689_b200 import synth

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    me.me_init(0)
    me.me_set_stream(torch.cuda.current_stream())
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("gather", ["root", "all"])
@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_gather_step_c3_under_nccl(nccl, gather, scaling):
    cfg = synth.CONFIGS["c3"]
    npairs = 3
    dev = torch.device("cuda", 0)
    mine = mdist.rank_pairs(npairs, 1, 0, scaling)
    frames = synth.make_sequence(cfg, device=dev, pairs=range(1 + mine.start, 1 + mine.stop))
    stream = torch.cuda.current_stream()
    step = mdist.GatherStep(len(mine), npairs, cfg.nb, dev, 1, 0, True, gather, stream=stream,
                            collective=True)
    for k in range(4):  # the two buffers alternate; every step searches and gathers
        step.step(k, lambda *v: me.me_dcds_batch_packed(frames, cfg.B, cfg.p, *v))
    step.drain()
    torch.cuda.synchronize()
    mv8, sad16, pts, st = step.gathered(npairs, scaling)
    mv = mv8.to(torch.int16).cpu().numpy()
    sad = (sad16.to(torch.int32) & 0xFFFF).cpu().numpy().astype(np.uint32)
    pts = pts.cpu().numpy().astype(np.uint16)
    st = st.cpu().numpy().astype(np.uint64)
    # every block against the parity-tested 10-byte arrays of me_dcds_batch
    rmv, rsad, rpts, rst = me.alloc_outputs(npairs, cfg.nb, dev)
    me.me_dcds_batch(frames, cfg.B, cfg.p, rmv, rsad, rpts, rst)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(mv, rmv.cpu().numpy())
    np.testing.assert_array_equal(sad, rsad.cpu().numpy().astype(np.uint32))
    np.testing.assert_array_equal(pts, rpts.cpu().numpy().astype(np.uint16))
    np.testing.assert_array_equal(st, rst.cpu().numpy().astype(np.uint64))
    # sampled blocks of every pair against the oracle (full-size c3 frames)
    host = frames.cpu().numpy()
    rng = np.random.default_rng(7 + len(gather) + len(scaling))
    nbx = cfg.W // cfg.B
    for t in range(npairs):
        for i in rng.choice(cfg.nb, 150, replace=False):
            bx, by = (i % nbx) * cfg.B, (i // nbx) * cfg.B
            omv, osad, opts = oracle.dcds_block(host[t, 0], host[t, 1], cfg.B, cfg.p, bx, by)
            assert tuple(mv[t, i]) == tuple(omv) and sad[t, i] == osad and pts[t, i] == opts, (t, i)
