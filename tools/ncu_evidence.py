"""SURVEY 8(d) evidence from one `ncu --set full` capture of a search kernel, written into
profiles/ncu_traffic.json (bench.py copies it into its roofline object):

  * DRAM bytes per launch against the algorithmic bytes (2 W H + 10 nb + 24 per pair);
  * L2 -> SM bytes (l1tex__m_xbar2l1tex_read_bytes: the TMA staging incl. the search-window
    halo re-reads) and all L2 traffic (lts__t_sectors x 32) against the algorithmic bytes;
  * executed VABSDIFF4 lane-ops (thread-level instruction count of the VABSDIFF4 opcodes from
    the per-SASS source page) against the algorithmic ones, sum NSP x B^2 / 4 (+ the fused
    MC-SSE, 2 x B^2 / 4 per block on the IDP.4A / VABSDIFF4 side, reported apart) -- ~1.0 means
    no speculative SAD work;
  * warp-instructions and shared-memory wavefronts per macroblock, pipe utilisations.

usage: python tools/ncu_evidence.py <report.ncu-rep> <config> <bench.json of the same command>
       [--kernel REGEX] [--key NAME]
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def raw(rep, kernel=None):
    cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"] + (["-k", "regex:" + kernel] if kernel else [])
    rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def opcode_threads(rep, kernel=None):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if kernel:
        cmd += ["-k", "regex:" + kernel]
    rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    ct = h.index("Thread Instructions Executed")
    out = {}
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        src = r[1].strip()
        if src.startswith("@"):
            src = src.split(None, 1)[1]
        op = src.split()[0] if src else "?"
        out[op] = out.get(op, 0.0) + float(r[ct] or 0)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("config")
    ap.add_argument("bench")
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--key", default=None, help="entry name in ncu_traffic.json (default: config)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_traffic.json"))
    a = ap.parse_args()
    from paper_0806_0689_b200 import synth
    cfg = synth.CONFIGS[a.config]
    b = json.load(open(a.bench))
    npairs = b["config"]["pairs_per_gpu"]
    mean_nsp = b["config"]["mean_nsp"]
    nblk = npairs * cfg.nb
    v, u = raw(a.rep, a.kernel)
    dram = to_bytes(v["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) + \
        to_bytes(v["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
    l2sm = to_bytes(v["l1tex__m_xbar2l1tex_read_bytes.sum"], u["l1tex__m_xbar2l1tex_read_bytes.sum"])
    lts = float(v["lts__t_sectors.sum"]) * 32
    alg = npairs * (2 * cfg.W * cfg.H + 10 * cfg.nb + 24)
    ops = opcode_threads(a.rep, a.kernel)
    vabs = sum(x for k, x in ops.items() if k.startswith("VABSDIFF4"))
    idp = sum(x for k, x in ops.items() if k.startswith("IDP"))
    alg_vabs = nblk * mean_nsp * cfg.B * cfg.B / 4.0
    sse_lane_ops = nblk * cfg.B * cfg.B / 4.0  # one VABSDIFF4 per 4 pixels of the fused MC-SSE
    pct = lambda k: round(float(v[k]), 1) if k in v and v[k] not in ("", "no data") else None
    d = {
        "kernel": next((k for k in [v.get("Kernel Name"), v.get("Function Name")] if k), None),
        "duration_ms_ncu": float(v["gpu__time_duration.sum"]) / (1e6 if u["gpu__time_duration.sum"] == "ns" else
                                                                 (1e3 if u["gpu__time_duration.sum"] == "us" else 1)),
        "dram_bytes_per_launch": int(dram),
        "alg_bytes_per_launch": int(alg),
        "dram_over_alg": dram / alg,
        "l2_to_sm_bytes_per_launch": int(l2sm),
        "l2_to_sm_over_alg": l2sm / alg,
        "lts_bytes_per_launch": int(lts),
        "vabsdiff4_lane_ops_executed": int(vabs),
        "vabsdiff4_lane_ops_algorithmic": int(alg_vabs),
        "vabsdiff4_exec_over_alg": vabs / alg_vabs,
        "vabsdiff4_exec_over_alg_plus_fused_sse": vabs / (alg_vabs + sse_lane_ops),
        "idp4a_lane_ops_executed": int(idp),
        "warp_inst_per_block": float(v["smsp__inst_executed.sum"]) / nblk,
        "smem_wavefronts_per_block": float(v["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]) / nblk,
        "active_lanes_per_warp_inst": pct("smsp__thread_inst_executed_per_inst_executed.ratio"),
        "registers_per_thread": pct("launch__registers_per_thread"),
        "limiters_pct": {
            "shared_pipe_wavefronts": pct("l1tex__throughput.avg.pct_of_peak_sustained_active"),
            "issue_active": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "alu_pipe": pct("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "fma_pipe": pct("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "dram_throughput": pct("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "warps_active": pct("sm__warps_active.avg.pct_of_peak_sustained_active"),
        },
        "source": f"ncu --set full --clock-control none ({os.path.relpath(a.rep, ROOT)}); "
                  f"bench config {a.config}, {npairs} pairs, mean NSP {mean_nsp:.4f}",
    }
    allj = json.load(open(a.out)) if os.path.exists(a.out) else {}
    allj[a.key or a.config] = d
    json.dump(allj, open(a.out, "w"), indent=1)
    print(json.dumps(d, indent=1))
