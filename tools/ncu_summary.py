"""Per-kernel summary of an ncu report (`--set full`) as JSON for bench.py.

    python tools/ncu_summary.py report.ncu-rep profiles/ncu_<name>.json [note]

For every profiled launch: device time, DRAM bytes (read + write), and the
speed-of-light throughputs of the memory/compute units as a fraction of peak.
`binding` is the unit with the highest fraction -- the roof the kernel sits
under (HBM for a streaming kernel, L1/shared for the tile sweep's scatter,
issue for the probe loops).  step_* sums the launches of the batch.
"""
import csv
import io
import json
import subprocess
import sys

UNITS = {
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "HBM (dram__throughput)",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "L2 (lts__throughput)",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "L1 / shared memory (l1tex__throughput)",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "LSU pipe (sm__inst_executed_pipe_lsu)",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "SM issue / pipes (sm__throughput)",
}
EXTRA = ["sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
         "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
         "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
         "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
         "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
         "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
         "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
         "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main():
    rep, out = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    kernels, launches = {}, []
    for r in data:
        name = r[col["Kernel Name"]].split("(")[0].split("<")[0].split("::")[-1]
        ns = num(r[col["gpu__time_duration.sum"]])
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "us": 1e-3, "ns": 1e-6}.get(units[col["gpu__time_duration.sum"]], 1e-6)
        rd = num(r[col["dram__bytes_read.sum"]]) or 0.0
        wr = num(r[col["dram__bytes_write.sum"]]) or 0.0
        bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[col["dram__bytes_read.sum"]], 1)
        wscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[col["dram__bytes_write.sum"]], 1)
        fr = {UNITS[m]: num(r[col[m]]) / 100.0 for m in UNITS if m in col and num(r[col[m]]) is not None}
        bind = max(fr, key=fr.get) if fr else None
        k = dict(ms=ns * scale, dram_bytes=rd * bscale + wr * wscale, dram_read=rd * bscale,
                 dram_write=wr * wscale, unit_fracs=fr, binding=bind, binding_frac=fr.get(bind),
                 extra={m: num(r[col[m]]) for m in EXTRA if m in col})
        launches.append(dict(kernel=name, **k))
        if name not in kernels or kernels[name]["ms"] < k["ms"]:
            kernels[name] = k
    res = dict(report=rep, note=note, kernels=kernels, launches=launches,
               step_ms=sum(x["ms"] for x in launches), step_dram_bytes=sum(x["dram_bytes"] for x in launches if x["dram_bytes"] == x["dram_bytes"]))
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    for n, k in kernels.items():
        print(f"{n:28s} {k['ms']:9.3f} ms  dram {k['dram_bytes'] / 1e9:8.2f} GB  bind {k['binding']} "
              f"{(k['binding_frac'] or 0):.2f}")


if __name__ == "__main__":
    main()
