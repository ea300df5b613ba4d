"""Top SASS instructions of an ncu report by warp-stall samples / executed count."""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
S = hdr.index("Warp Stall Sampling (All Samples)"); E = hdr.index("Instructions Executed")
body = [r for r in rows[2:] if len(r) > E]
tot_s = sum(float(r[S] or 0) for r in body); tot_e = sum(float(r[E] or 0) for r in body)
print(f"total samples {tot_s:.0f}  total warp-instr {tot_e:.3g}")
key = S if len(sys.argv) < 4 else E
idx = sorted(range(len(body)), key=lambda i: -float(body[i][key] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]
stall_cols = [i for i, n in enumerate(hdr) if n.startswith("stall_")]
for i in sorted(idx):
    r = body[i]
    st = sorted(((float(r[c] or 0), hdr[c][6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{i:5d} {100*float(r[S] or 0)/tot_s:5.1f}% ex={float(r[E] or 0)/tot_e*100:5.2f}%  {r[1].strip()[:60]:60s} {st[0][1]}:{st[0][0]:.0f} {st[1][1]}:{st[1][0]:.0f}")
