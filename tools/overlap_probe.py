"""One-GPU probe of the multi-GPU step's overlap (bench.py --gpus N): the DCDS search on the
main stream while a communication-like kernel (a fixed number of CTAs streaming the bytes a
rank receives in an 8-GPU all_gather of the c3 outputs: 7 x 47 MB as the 6-byte record,
PROBE_RECORD=10 for the 10-byte arrays) runs on a high-priority stream, as NCCL's kernels do.
Prints ms per step alone and with the concurrent copy."""
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0806_0689_b200 as me  # noqa: E402
from paper_0806_0689_b200 import synth  # noqa: E402

here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "probe", "copy_probe.so")
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                       "-shared", "-Xcompiler", "-fPIC", "-o", so, os.path.join(here, "probe", "copy_probe.cu")])
lib = ctypes.CDLL(so)
lib.probe_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]

me.me_init(0)
main = torch.cuda.current_stream()
me.me_set_stream(main)
cfg = synth.CONFIGS["c3"]
fr = synth.make_sequence(cfg, device="cuda")
outs = me.alloc_outputs(cfg.npairs, cfg.nb, "cuda")
rec = int(os.environ.get("PROBE_RECORD", "6"))  # bytes per block: 6 (packed) or 10 (arrays)
nbytes = 7 * cfg.npairs * (cfg.nb * rec + 24)
src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
comm = torch.cuda.Stream(priority=-1)


def run(steps, nctas):
    for _ in range(3):
        me.me_dcds_batch(fr, cfg.B, cfg.p, *outs)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for _ in range(steps):
        me.me_dcds_batch(fr, cfg.B, cfg.p, *outs)
        if nctas:
            ev = torch.cuda.Event()
            ev.record(main)
            comm.wait_event(ev)  # as bench.py: the gather of step k follows its search
            lib.probe_copy(src.data_ptr(), dst.data_ptr(), nbytes, nctas, comm.cuda_stream)
    main.wait_stream(comm)
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def copy_alone(nctas):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(comm)
    for _ in range(10):
        lib.probe_copy(src.data_ptr(), dst.data_ptr(), nbytes, nctas, comm.cuda_stream)
    b.record(comm)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 10


print(f"search alone: {run(20, 0):.3f} ms/step; copy bytes {nbytes / 1e6:.0f} MB")
for n in (16, 32, 64):
    print(f"copy {n} CTAs alone {copy_alone(n):.3f} ms; search + concurrent copy: {run(20, n):.3f} ms/step")
