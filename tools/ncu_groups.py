"""Group SASS instructions of an ncu report by execution count (loop bodies)."""
import csv, io, subprocess, sys
from collections import defaultdict
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; E = hdr.index("Instructions Executed"); S = hdr.index("Warp Stall Sampling (All Samples)")
body = rows[2:]
ex = [float(r[E] or 0) for r in body]; st = [float(r[S] or 0) for r in body]
tot = sum(ex); tots = sum(st)
c = defaultdict(lambda: [0, 0, []])
for i, e in enumerate(ex):
    c[e][0] += e; c[e][1] += st[i]; c[e][2].append(i)
print("total instr", tot)
for val, (s, ss, idx) in sorted(c.items(), key=lambda x: -x[1][1])[:10]:
    print(f"count {val:.3g} x{len(idx)} = {100*s/tot:.1f}% instr, {100*ss/tots:.1f}% stalls  idx {idx[0]}..{idx[-1]}")
stall_cols = [i for i, n in enumerate(hdr) if n.startswith("stall_") and "Not Issued" not in n]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 14
for i in sorted(sorted(range(len(body)), key=lambda i: -st[i])[:n]):
    r = body[i]
    s2 = sorted(((float(r[c] or 0), hdr[c][6:]) for c in stall_cols), reverse=True)[:2]
    print(i, f"{100*st[i]/tots:.1f}%", r[E], r[1].strip()[:60], s2)
