"""bench.py -- DCDS throughput on B200 (BASELINE.json metric: DCDS macroblocks/s and 1080p
frames/s per GPU and across GPUs, with the fraction of roofline).

Workload (N=1 default): config c3 -- 1920x1088 8-bit luma, 8x8 blocks, +-16 window, 239
independent frame pairs per GPU (the metric names 1080p frames/s).  A step is one pass of the
hot path over the batch: DCDS search of every block of every pair (Steps 1-4) with the fused
motion-compensated SSE and per-pair statistics (sum NSP, sum SAD, SSE), one launch through
the C ABI (me_dcds_batch); with N > 1 the per-pair MV fields and statistics are then gathered
with NCCL (the only collective; BASELINE.json north_star).  Full search (the quality
reference) is timed separately in the same run and reported under "fullsearch".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU)

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_0806_0689_b200 import synth  # noqa: E402

METRIC = "DCDS macroblocks/sec"
UNIT = "blocks/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget")
    ap.add_argument("--no-fs", action="store_true")
    ap.add_argument("--fs-pairs", type=int, default=32,
                    help="pairs of the full-search side measurement (rank 0)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cmp", action="store_true", help="skip the comparison-BMA section")
    ap.add_argument("--no-mcsse", action="store_true", help="skip the standalone MC-SSE timing")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every GPU searches the config's whole sequence (per-GPU work fixed); "
                         "strong: the sequence's pairs are sharded over the GPUs (ceil shards)")
    ap.add_argument("--gather", default="root", choices=["root", "all"],
                    help="N > 1: NCCL gather of the MV records to rank 0, or all_gather to every rank")
    ap.add_argument("--no-other-scaling", action="store_true",
                    help="N > 1: skip the second (other --scaling) measurement")
    ap.add_argument("--graph", action="store_true",
                    help="N=1: capture the K timed steps in one CUDA graph and replay it (small "
                         "configs c0-c2, whose launches are a few microseconds)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------------------------------
# clocks during the timed region (nvidia-smi sampler)
# ------------------------------------------------------------------------------------------
REASON_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    """nvidia-smi sampler started before the timed region; only samples taken between
    mark_start() and mark_end() are summarised (nvidia-smi needs ~0.5 s to start)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def __enter__(self):
        if self.index < 0:  # not sampled
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            deadline = time.time() + 5.0
            while not self.lines and time.time() < deadline:
                time.sleep(0.02)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        lines = self.lines
        if self.t0 is not None and self.t1 is not None:
            inside = [x for x in lines if self.t0 <= x[0] <= self.t1]
            if not inside and lines:  # region shorter than the sampling period: nearest sample
                inside = [min(lines, key=lambda x: abs(x[0] - (self.t0 + self.t1) / 2))]
            lines = inside
        for _, ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 4:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                bits = int(parts[3], 16)
            except ValueError:
                continue
            for b, n in REASON_BITS.items():
                if bits & b and n != "gpu_idle":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_int_peak():
    """Measured VABSDIFF4 lane-op rate (profiles/int_peaks.json, tools/int_peaks.cu)."""
    p = os.path.join(ROOT, "profiles", "int_peaks.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["vabsdiff4_add"]["lane_ops_per_sm_per_clk"], d.get("sms", 148)
    return None, 148


# ------------------------------------------------------------------------------------------
# the oracle, timed on host cores (cpu_baseline leg and --impl reference)
# ------------------------------------------------------------------------------------------
def _oracle_worker_init(shm_name, shape, B, p):
    global _W
    from multiprocessing import shared_memory
    import oracle  # test infrastructure; only the CPU legs of bench.py use it
    shm = shared_memory.SharedMemory(name=shm_name)
    _W = (shm, np.ndarray(shape, dtype=np.uint8, buffer=shm.buf), B, p, oracle)


def _oracle_worker_pair(t):
    _, fr, B, p, oracle = _W
    oracle.dcds(fr[t, 0], fr[t, 1], B, p)
    return t


def oracle_procs():
    """host cores the oracle legs use: one single-threaded oracle process per core"""
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    cap = int(os.environ.get("ME_ORACLE_PROCS", "64"))
    return max(1, min(n, cap))


class OraclePool:
    """The oracle as it stands (single-threaded C), one process per host core over disjoint
    pairs, frames shared through one shared-memory block (no per-task copies)."""

    def __init__(self, frames_host: np.ndarray, cfg, nprocs: int):
        import multiprocessing as mp
        from multiprocessing import shared_memory
        import oracle
        oracle.build()  # compile once, before the workers load it
        self.shm = shared_memory.SharedMemory(create=True, size=frames_host.nbytes)
        np.ndarray(frames_host.shape, np.uint8, buffer=self.shm.buf)[:] = frames_host
        self.n = frames_host.shape[0]
        self.nprocs = nprocs
        self.pool = mp.get_context("spawn").Pool(
            nprocs, initializer=_oracle_worker_init,
            initargs=(self.shm.name, frames_host.shape, cfg.B, cfg.p))
        self.pool.map(_oracle_worker_pair, [0] * nprocs)  # warm: every worker loaded the oracle

    def run(self, pairs):
        t0 = time.perf_counter()
        for _ in self.pool.imap_unordered(_oracle_worker_pair, pairs, chunksize=1):
            pass
        return time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()
        self.shm.close()
        self.shm.unlink()


def oracle_rate(frames_host: np.ndarray, cfg, budget_s: float):
    """blocks/s of the oracle on the host cores over a bounded sample of the pairs: rounds of
    one pair per process until the budget is spent; returns (rate, pairs, seconds, procs)."""
    nprocs = min(oracle_procs(), frames_host.shape[0])
    pool = OraclePool(frames_host, cfg, nprocs)
    try:
        done, dt, t = 0, 0.0, 0
        while done < frames_host.shape[0] and dt < budget_s:
            batch = list(range(t, min(t + nprocs, frames_host.shape[0])))
            dt += pool.run(batch)
            done += len(batch)
            t += len(batch)
    finally:
        pool.close()
    return done * cfg.nb / dt, done, dt, nprocs


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    """--impl reference: the oracle as it stands (single-threaded C), one process per host
    core over disjoint pairs; each step is one bounded sample (one pair per process) of the
    same config, metric and unit as the b200 arm."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.config]
    dev = "cuda:0" if torch.cuda.is_available() else "cpu"
    nprocs = oracle_procs()
    npairs = min(cfg.npairs, nprocs)
    fr = synth.make_sequence(cfg, device=dev, pairs=range(1, npairs + 1)).cpu().numpy()
    pool = OraclePool(fr, cfg, npairs)
    times = []
    try:
        for s in range(args.steps + args.warmup):
            dt = pool.run(list(range(npairs)))
            if s >= args.warmup:
                times.append(dt)
    finally:
        pool.close()
    tot = sum(times)
    value = cfg.nb * npairs * len(times) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded; SURVEY 8(d) generator)",
        "config": {"workload": f"{cfg.name}: {cfg.W}x{cfg.H}, {cfg.B}x{cfg.B} blocks, +-{cfg.p}",
                   "sample_per_step": f"{npairs} frame pairs, one per oracle process"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": npairs, "kind": "oracle",
                         "sample": f"{npairs} pairs per step ({npairs} single-threaded oracle "
                                   f"processes), {len(times)} steps; {cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# the B200 arm
# ------------------------------------------------------------------------------------------
def timed_run(args, cfg, me, mdist, dist, ws, rank, dev, stream, scaling, sample_clocks=True):
    """W warm-up + K timed steps of the hot path on this rank.

    scaling "weak": every rank searches its own cfg.npairs pairs; "strong": the configured
    cfg.npairs pairs are split into contiguous shards (dist.rank_pairs), the last one short.
    A step = me_dcds_batch (N = 1) or me_dcds_batch_packed into a flat buffer followed by the
    NCCL gather of the MV fields + statistics (N > 1: gather-to-rank-0 or all_gather,
    --gather), the gather of step k overlapping the search of step k+1 (dist.GatherStep).
    Time: CUDA events on the launch stream between a barrier + synchronize on both sides,
    max over ranks."""
    mine = mdist.rank_pairs(cfg.npairs, ws, rank, scaling)
    n = len(mine)
    per = cfg.npairs if scaling == "weak" else mdist.shard_size(cfg.npairs, ws)
    frames = (synth.make_sequence(cfg, device=dev, pairs=range(1 + mine.start, 1 + mine.stop)) if n else
              torch.empty(0, 2, cfg.H, cfg.W, dtype=torch.uint8, device=dev))
    packed = ws > 1  # the 6-byte transport record (me_dcds_batch_packed): 40% fewer bytes to gather
    step = mdist.GatherStep(n, per, cfg.nb, dev, ws, rank, packed, args.gather, stream=stream)
    search_fn = me.me_dcds_batch_packed if packed else me.me_dcds_batch

    def search(mv, sad, pts, st):
        search_fn(frames, cfg.B, cfg.p, mv, sad, pts, st)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    torch.cuda.synchronize()
    with ClockSampler(dev.index if sample_clocks else -1) as clk:  # warm-up also brings clocks up
        for k in range(max(args.warmup, 0)):
            step.step(k, search)
        step.drain()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        launches0 = me.me_launch_count()
        torch.cuda.synchronize()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        if args.graph and ws == 1:
            # the K steps as one CUDA graph (captured on torch's capture stream, which the
            # library launches on while capturing); one replay is the timed region
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                me.me_set_stream(torch.cuda.current_stream())
                for k in range(args.steps):
                    search(*step.local_views(0))
            me.me_set_stream(stream)
            # (launches0 was read before the capture: the delta is the captured launches, which
            # the timed replay runs once)
            graph.replay()  # warm the graph
            torch.cuda.synchronize()
            clk.mark_start()
            t_start.record(stream)
            graph.replay()
            t_end.record(stream)
            torch.cuda.synchronize()
            clk.mark_end()
            ev = None
        else:
            clk.mark_start()
            t_start.record(stream)
            for k in range(args.steps):
                b = step.claim(k)  # (a wait on the previous gather is not kernel time)
                ev[k][0].record(stream)
                if n:
                    search(*step.local_views(b))
                ev[k][1].record(stream)
                step.collect(b)
                step.last = b
            step.drain()  # the last gathers are inside the timed region
            t_end.record(stream)
            torch.cuda.synchronize()
            clk.mark_end()
    launches = me.me_launch_count() - launches0
    total_ms = t_start.elapsed_time(t_end)
    kern_ms = [a.elapsed_time(b) for a, b in ev] if ev else [total_ms / args.steps] * args.steps
    if ws > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    local = step.local_views(step.last)
    pairs_all = ws * cfg.npairs if scaling == "weak" else cfg.npairs
    out = {"n": n, "frames": frames, "total_ms": total_ms, "kern_ms": kern_ms, "launches": launches,
           "clocks": clk.summary(), "local": local, "step": step, "pairs_all": pairs_all,
           "value": pairs_all * cfg.nb / (total_ms / args.steps * 1e-3), "scaling": scaling}
    if ws > 1:  # the gathered copy of this rank's pairs equals its own output
        g = step.gathered(cfg.npairs, scaling)
        if g is not None and n:
            off = mine.start
            assert torch.equal(g[0][off:off + n], local[0]) and torch.equal(g[3][off:off + n], local[3])
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    ws, rank, local = dist_env()
    if ws > 1:
        import datetime

        import torch.distributed as dist
        # a hung or failed peer aborts the run instead of stalling it (pairs are stateless:
        # a failed run is simply re-run)
        os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                timeout=datetime.timedelta(minutes=5))
    else:
        dist = None
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_0806_0689_b200 as me
    me.me_init(local)
    stream = torch.cuda.current_stream()
    me.me_set_stream(stream)

    cfg = synth.CONFIGS[args.config]
    from paper_0806_0689_b200 import dist as mdist
    run = timed_run(args, cfg, me, mdist, dist, ws, rank, dev, stream, args.scaling)
    mv, sad, pts, st = run["local"]
    n, frames, total_ms, kern_ms, launches, clocks = (run["n"], run["frames"], run["total_ms"], run["kern_ms"],
                                                     run["launches"], run["clocks"])
    in_bytes = frames.numel()
    ms_per_step = total_ms / args.steps
    stats = st.cpu().numpy().astype(np.float64)
    sum_pts = float(stats[:, 0].sum())
    value = run["value"]

    # roofline of the dominant kernel (dcds_kernel), algorithmic bytes / ops per launch
    hbm_peak, hbm_src = load_peaks()
    kern_avg_s = statistics.mean(kern_ms) * 1e-3
    bytes_per_pair = 2 * cfg.W * cfg.H + 10 * cfg.nb + 24
    alg_bytes = n * bytes_per_pair
    achieved_gbs = alg_bytes / kern_avg_s / 1e9
    lane_ops = sum_pts * cfg.B * cfg.B / 4.0            # VABSDIFF4 lane-ops the method needs
    r_clk, sms = load_int_peak()
    roofline = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved_gbs / hbm_peak, "traffic": None, "peak_source": hbm_src,
                "alg_bytes_per_launch": alg_bytes}
    if r_clk is not None:
        clk_mhz = clocks["sm_mhz"] or 1965.0
        int_peak = r_clk * sms * clk_mhz * 1e6          # lane-ops/s at the clock seen
        t_hbm = alg_bytes / (hbm_peak * 1e9)
        t_int = lane_ops / int_peak
        roofline["int_peak_lane_ops_per_s"] = int_peak
        roofline["int_achieved_lane_ops_per_s"] = lane_ops / kern_avg_s
        roofline["t_roof_ms"] = {"hbm": t_hbm * 1e3, "alu": t_int * 1e3}
        if t_int > t_hbm:
            roofline.update({"bound": "alu", "achieved": lane_ops / kern_avg_s / 1e12,
                             "peak": int_peak / 1e12, "unit": "Tlane-op/s",
                             "frac": (lane_ops / kern_avg_s) / int_peak,
                             "peak_source": "measured VABSDIFF4 rate (profiles/int_peaks.json) x SMs x median SM clock"})
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        d = json.load(open(tp)).get(cfg.name)
        if d:
            roofline["traffic"] = d.get("dram_bytes_per_launch")
            # what actually limits the kernel (same ncu capture): % of peak per resource
            if d.get("limiters_pct"):
                roofline["ncu_limiters_pct"] = d["limiters_pct"]
            # SURVEY 8(d) evidence of the same capture (tools/ncu_evidence.py): halo
            # over-fetch L2 -> SM, executed / algorithmic VABSDIFF4 lane-ops, per-block budget
            for k in ("l2_to_sm_over_alg", "vabsdiff4_exec_over_alg", "vabsdiff4_exec_over_alg_plus_fused_sse",
                      "warp_inst_per_block", "smem_wavefronts_per_block", "source"):
                if k in d:
                    roofline["ncu_" + k] = d[k]

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded; SURVEY 8(d) generator; paper's sequences unavailable)",
        "config": {
            "workload": f"{cfg.name}: {cfg.W}x{cfg.H} luma, {cfg.B}x{cfg.B} blocks, +-{cfg.p} window, "
                        + (f"{cfg.npairs} frame pairs per GPU" if args.scaling == "weak" else
                           f"{cfg.npairs} frame pairs sharded over {ws} GPU(s)"),
            "pairs_per_gpu": n, "pairs_all_gpus": run["pairs_all"], "blocks_per_pair": cfg.nb,
            "W": cfg.W, "H": cfg.H, "block": cfg.B, "p": cfg.p,
            "frames_per_sec": run["pairs_all"] / (ms_per_step * 1e-3),
            "mean_nsp": sum_pts / (n * cfg.nb),
            "l2": (f"inputs {in_bytes / 2**20:.0f} MiB per GPU > 126 MB L2 (no flush needed)"
                   if in_bytes > 126e6 else
                   f"inputs {in_bytes / 2**20:.1f} MiB per GPU fit the 126 MB L2: L2-resident, not flushed "
                   "(a small parity config, not the bench line)"),
            "cuda_graph": bool(args.graph and ws == 1),
            "parallelism": (f"dp{ws} (frame pairs sharded; NCCL "
                            + ("gather to rank 0" if args.gather == "root" else "all_gather")
                            + " of the 6-byte MV records + stats, overlapped with the next search)")
                           if ws > 1 else "single GPU",
        },
        "gpu_launches": int(launches),
        "kernel_ms_mean": statistics.mean(kern_ms),
        "roofline": roofline,
        "clocks": clocks,
    }

    if ws > 1 and not args.no_other_scaling:
        # the other sharding of the same sequence, measured in the same run (the driver's
        # scaling run compares per-N values of the main line)
        other = "strong" if args.scaling == "weak" else "weak"
        r2 = timed_run(args, cfg, me, mdist, dist, ws, rank, dev, stream, other, sample_clocks=False)
        line["other_scaling"] = {"scaling": other, "value": r2["value"], "unit": UNIT,
                                 "ms_per_step": r2["total_ms"] / args.steps,
                                 "pairs_all_gpus": r2["pairs_all"], "pairs_per_gpu_rank0": r2["n"],
                                 "kernel_ms_mean_rank0": statistics.mean(r2["kern_ms"])}

    if rank == 0 and not args.no_fs:
        # FS (quality reference), same pairs, small sample: timed beside the path
        nfs = min(n, max(1, args.fs_pairs))
        fsub = frames[:nfs]
        fo = me.alloc_outputs(nfs, cfg.nb, dev)
        me.me_fullsearch_batch(fsub, cfg.B, cfg.p, *fo)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        a.record(stream)
        for _ in range(reps):
            me.me_fullsearch_batch(fsub, cfg.B, cfg.p, *fo)
        b.record(stream)
        torch.cuda.synchronize()
        fs_s = a.elapsed_time(b) * 1e-3 / reps
        fs_ops = nfs * cfg.nb * (2 * cfg.p + 1) ** 2 * cfg.B * cfg.B / 4.0
        fsline = {"value": nfs * cfg.nb / fs_s, "unit": UNIT, "pairs": nfs, "ms": fs_s * 1e3,
                  "lane_ops_per_s": fs_ops / fs_s}
        if r_clk is not None:
            fsline["alu_frac"] = (fs_ops / fs_s) / roofline["int_peak_lane_ops_per_s"]
        line["fullsearch"] = fsline

    if rank == 0 and not args.no_mcsse:
        # the motion-compensated SSE (P:342 aspect 4) standalone over every pair at the DCDS MV
        # field ("MC-PSNR fused and standalone"; fused it is part of the step)
        mvf = mv if mv.dtype == torch.int16 else None
        if mvf is None:
            mvf = me.alloc_outputs(n, cfg.nb, dev)[0]
            me.me_dcds_batch(frames, cfg.B, cfg.p, mvf, *me.alloc_outputs(n, cfg.nb, dev)[1:3])
        sse = torch.empty(n, dtype=torch.int64, device=dev)
        me.me_mc_sse_batch(frames, cfg.B, mvf, sse)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        a.record(stream)
        for _ in range(reps):
            me.me_mc_sse_batch(frames, cfg.B, mvf, sse)
        b.record(stream)
        torch.cuda.synchronize()
        mc_s = a.elapsed_time(b) * 1e-3 / reps
        if mv.dtype == torch.int16:  # equals the SSE the fused search reported
            assert torch.equal(sse, st[:, 2]), "standalone MC-SSE != fused"
        mc_bytes = n * (2 * cfg.W * cfg.H + 4 * cfg.nb + 8)
        line["mc_sse_standalone"] = {"value": n * cfg.nb / mc_s, "unit": UNIT, "ms": mc_s * 1e3, "pairs": n,
                                     "alg_bytes": mc_bytes, "achieved_gbs": mc_bytes / mc_s / 1e9,
                                     "frac_hbm": mc_bytes / mc_s / 1e9 / hbm_peak}

    if rank == 0 and not args.no_cmp:
        # the paper's comparison (Table IX): every BMA on a
        # sample of the same pairs -- NSP, PSNR, distance / probability vs FS, NSP speed-up of
        # DCDS over each (the "up to 54.9%" measure, P:9), and its own kernel throughput
        from paper_0806_0689_b200 import report
        ncmp = min(n, 16)
        rows = report.compare_bmas(frames[:ncmp], cfg.B, cfg.p, reps=3)
        line["comparison"] = {"pairs": ncmp, "algs": {
            a: {k: (round(v, 6) if isinstance(v, float) else v) for k, v in r.items()} for a, r in rows.items()}}

    if not args.no_e2e:
        # end to end through the C ABI on HOST buffers, on every rank: H2D of the frames
        # (pinned), search, D2H of the MV field + stats, every step; max over ranks
        e2e_s = 0.0
        if n:
            hfr = frames.cpu().pin_memory()
            hout = [t.pin_memory() for t in me.alloc_outputs(n, cfg.nb, "cpu")]
            me.me_dcds_batch_host(hfr, cfg.B, cfg.p, *hout)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        if n:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(args.e2e_steps):
                me.me_dcds_batch_host(hfr, cfg.B, cfg.p, *hout)
            b.record(stream)
            torch.cuda.synchronize()
            e2e_s = a.elapsed_time(b) * 1e-3 / args.e2e_steps
            assert np.array_equal(hout[0].numpy(), mv.cpu().numpy().astype(np.int16))
        if ws > 1:
            t = torch.tensor([e2e_s], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        pa = run["pairs_all"]
        line["e2e"] = {"value": pa * cfg.nb / e2e_s, "unit": UNIT,
                       "h2d_bytes_per_step": int(pa * 2 * cfg.W * cfg.H),
                       "d2h_bytes_per_step": int(pa * (cfg.nb * 10 + 24)),
                       "ms_per_step": e2e_s * 1e3, "steps": args.e2e_steps,
                       "note": "all ranks, each on its own pairs and PCIe link; max time over ranks"}

    if rank == 0 and not args.no_cpu and ws == 1:
        host = frames.cpu().numpy()  # the budget (--cpu-seconds) bounds the sample
        rate, npairs_done, dt, procs = oracle_rate(host, cfg, args.cpu_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": procs, "kind": "oracle",
                                "sample": f"{npairs_done} pairs of {cfg.name} ({npairs_done * cfg.nb} blocks) "
                                          f"in {dt:.1f} s, {procs} single-threaded oracle processes "
                                          f"(gcc -O2) over disjoint pairs; {cpu_model()}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
