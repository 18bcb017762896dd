"""Stall samples and instructions per CUDA source line from an ncu report (needs -lineinfo + --import-source)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows, fname, hdr = [], None, None
for line in raw:
    r = next(csv.reader([line]))
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            st = int(d["Warp Stall Sampling (All Samples)"]); ie = int(d["Instructions Executed"])
        except ValueError:
            continue
        try:
            xs = int(d.get("L1 Wavefronts Shared Excessive", "0") or 0)
        except ValueError:
            xs = 0
        rows.append((st, ie, fname, int(r[0]), r[1].strip()[:90], xs))
tot_s = sum(x[0] for x in rows) or 1; tot_i = sum(x[1] for x in rows) or 1
tot_x = sum(x[5] for x in rows) or 1
key = 1 if len(sys.argv) > 3 and sys.argv[3] == "inst" else 0
rows.sort(key=lambda x: x[key], reverse=True)
for st, ie, f, ln, src, xs in rows[:top]:
    print(f"{st / tot_s * 100:5.1f}% stall {ie / tot_i * 100:5.1f}% inst {xs / tot_x * 100:5.1f}% smem-excess  {f}:{ln}  {src}")
