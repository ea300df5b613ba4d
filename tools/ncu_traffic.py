"""Convert an ncu --csv metrics log of the fused kernel into profiles/ncu_traffic.json
(dram bytes per launch, used by bench.py's roofline.traffic)."""
import csv, json, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "second": 1}
vals = {}
for r in rows[1:]:
    if sys.argv[2] in r[ki]:
        vals.setdefault(r[mi], []).append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1))
out = {"kernel": sys.argv[2], "launches": len(vals.get("dram__bytes_read.sum", [])),
       "dram_bytes_read_per_launch": sum(vals["dram__bytes_read.sum"]) / len(vals["dram__bytes_read.sum"]),
       "dram_bytes_write_per_launch": sum(vals["dram__bytes_write.sum"]) / len(vals["dram__bytes_write.sum"]),
       "source": sys.argv[1], "note": sys.argv[3] if len(sys.argv) > 3 else ""}
out["dram_bytes_per_launch"] = out["dram_bytes_read_per_launch"] + out["dram_bytes_write_per_launch"]
if "gpu__time_duration.sum" in vals:
    out["ncu_duration_s_per_launch"] = sum(vals["gpu__time_duration.sum"]) / len(vals["gpu__time_duration.sum"])
json.dump(out, open(sys.argv[4] if len(sys.argv) > 4 else "profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
