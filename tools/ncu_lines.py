"""Per-source-line hot spots of an ncu report (development aid).

    python tools/ncu_lines.py report.ncu-rep [N]

Walks every file section of `ncu --page source --print-source cuda` and prints
the N lines with the most warp-stall samples, with instructions executed and
shared-memory wavefronts (ideal vs actual: the excess is bank conflicts)."""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, fname, hdr = [], "?", None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname, hdr = r[1].rsplit("/", 1)[-1], None
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("Function Name", "File Name"):
            continue
        if len(r) > 2 and r[2] != "-":  # a SASS row; keep the per-line aggregates
            continue
        d = dict(zip(hdr[4:], r[4:]))
        d["Line No"], d["Source"] = r[0], r[1]
        try:
            st = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
        except ValueError:
            continue
        def f(k):
            try:
                return float(d.get(k, 0) or 0)
            except ValueError:
                return 0.0
        rows.append((st, fname, d["Line No"], d["Source"].strip(), f("Instructions Executed"),
                     f("L1 Wavefronts Shared"), f("L1 Wavefronts Shared Ideal")))
    tot = sum(x[0] for x in rows) or 1.0
    toti = sum(x[4] for x in rows) or 1.0
    print(f"{'stall%':>6} {'instr%':>6} {'smem wf':>10} {'ideal':>10}  file:line  source")
    for st, fn, ln, src, ins, wf, wfi in sorted(rows, key=lambda x: -x[0])[:n]:
        print(f"{100 * st / tot:6.1f} {100 * ins / toti:6.1f} {wf:10.3g} {wfi:10.3g}  {fn}:{ln}  {src[:90]}")


if __name__ == "__main__":
    main()
