"""Summarise an ncu report: key metrics + stall mix + instruction distribution (run here, not on the GPU)."""
import csv, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "launch__registers_per_thread", "sm__maximum_warps_per_active_cycle_pct",
        "launch__shared_mem_per_block_dynamic", "smsp__thread_inst_executed_per_inst_executed.ratio"]

if __name__ == "__main__":
    v, u = raw(sys.argv[1])
    nblk = float(sys.argv[2]) if len(sys.argv) > 2 else 0
    for k in KEYS:
        if k in v:
            print(f"{k:60s} {v[k]} {u[k]}")
    if nblk:
        print("warp-inst per block %.1f" % (float(v["smsp__inst_executed.sum"]) / nblk))
        print("smem wavefronts per block %.1f" % (float(v["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]) / nblk))
    st = [(k, float(v[k] or 0)) for k in v if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    for k, x in sorted(st, key=lambda t: -t[1])[:10]:
        print("  stall %-28s %.3f" % (k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], x))
