"""Summarise an ncu report (development aid): key throughput metrics, stall
breakdown, and the hottest source lines by warp stall samples."""
import csv, io, subprocess, sys

def run(args):
    return subprocess.run(["ncu", "-i", sys.argv[1]] + args, capture_output=True, text=True).stdout

raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
h, units, v = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed_op_shared_atom.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
for i, n in enumerate(h):
    if n in want:
        print(f"{n:70s} {v[i]} {units[i]}")
stalls = []
for i, n in enumerate(h):
    if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
        try:
            stalls.append((float(v[i]), n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
print("stalls per issue:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(stalls, reverse=True)[:8]))
if len(sys.argv) > 2:
    src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "cuda"]))))
    hdr = src[0]
    try:
        ci = hdr.index("Warp Stall Sampling (All Samples)")
    except ValueError:
        ci = None
    if ci is not None:
        rows = [r for r in src[1:] if len(r) > ci and r[ci].replace('.', '', 1).isdigit()]
        rows.sort(key=lambda r: -float(r[ci]))
        tot = sum(float(r[ci]) for r in rows) or 1
        for r in rows[:int(sys.argv[2])]:
            print(f"{100*float(r[ci])/tot:5.1f}%  L{r[0]}: {r[1].strip()[:110]}")
