import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
for r in rows[hi + 1:][-n:]:
    print(f"{float(r[vi].replace(',', '')) / 1e6:9.3f} ms  {r[ki][:110]}")
