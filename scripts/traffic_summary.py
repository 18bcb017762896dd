"""Per-kernel time and DRAM bytes of the LAST local multiply in an ncu CSV
(`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv`) of `bench.py --steps 1`: writes profiles/traffic.json and prints the
launch summary.  usage: python scripts/traffic_summary.py <csv> <key> <summary.txt>"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ID, K, M, V = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
ker = {}
for r in rows[hi + 1:]:
    if len(r) != len(h):
        continue
    k = ker.setdefault(int(r[ID]), {"name": r[K]})
    k[r[M]] = float(r[V].replace(",", ""))
ids = sorted(ker)
first = [i for i in ids if "analyse_rows_kernel" in ker[i]["name"]][-1]
agg = {}
for i in ids[ids.index(first):]:
    name = ker[i]["name"].split("(")[0].replace("void ", "")
    a = agg.setdefault(name, {"bytes": 0, "ms": 0.0})
    a["bytes"] += int(ker[i].get("dram__bytes_read.sum", 0) + ker[i].get("dram__bytes_write.sum", 0))
    a["ms"] += ker[i].get("gpu__time_duration.sum", 0) / 1e6
tot_b = sum(a["bytes"] for a in agg.values())
tot_ms = sum(a["ms"] for a in agg.values())
json.dump({sys.argv[2]: tot_b, "_note": "dram__bytes_read.sum + dram__bytes_write.sum over every kernel of one "
           f"config-2 local multiply (ncu; {sys.argv[1].split('/')[-1]})",
           "per_kernel": {k: {"bytes": a["bytes"], "ms": round(a["ms"], 3)} for k, a in agg.items()}},
          open("profiles/traffic.json", "w"), indent=1)
with open(sys.argv[3], "w") as f:
    f.write("# config-2 local multiply (R-MAT s18 permuted, tropical int32), one call under ncu\n"
            "# (serialised launches; --clock-control none): kernel time and DRAM bytes\n\n")
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["ms"]):
        f.write(f"{a['ms']:8.3f} ms {100 * a['ms'] / tot_ms:6.1f}% {a['bytes'] / 1e9:9.3f} GB  {k}\n")
    f.write(f"\n{tot_ms:8.3f} ms total, {tot_b / 1e9:.2f} GB DRAM\n")
print(open(sys.argv[3]).read())
