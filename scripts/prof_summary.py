import csv, sys, subprocess, collections
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h = r[0]
for row in r[2:]:
    d = dict(zip(h, row))
    print(d.get('Kernel Name', '')[:80])
    keys = [k for k in h if 'smsp__pcsamp_warps_issue_stalled' in k and not k.endswith('_not_issued')]
    vals = sorted([(float(d[k].replace(',', '')), k) for k in keys if d[k]], reverse=True)
    tot = sum(v for v, _ in vals) or 1
    print("  stalls:", ", ".join(f"{k[33:]} {v/tot*100:.0f}%" for v, k in vals[:8]))
    for k in ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
              'sm__warps_active.avg.pct_of_peak_sustained_active', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
              'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'lts__t_sector_hit_rate.pct',
              'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
              'l1tex__throughput.avg.pct_of_peak_sustained_active']:
        print("   ", k, d.get(k))
if len(sys.argv) > 2:
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + ([] if sys.argv[2] == "-" else ["-k", sys.argv[2]]),
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(sass.splitlines()))
    hdr = rows[1]
    ii = hdr.index('Instructions Executed'); si = hdr.index('Source'); ws = hdr.index('Warp Stall Sampling (All Samples)')
    seen = set(); seq = []
    for rr in rows[2:]:
        if len(rr) != len(hdr) or rr[0] in seen: continue
        seen.add(rr[0])
        try: seq.append((int(rr[0], 16), int(rr[ii]), int(rr[ws]), rr[si].strip()))
        except ValueError: pass
    seq.sort()
    tot = sum(s[1] for s in seq) or 1; tots = sum(s[2] for s in seq) or 1
    blocks = []; cur = None
    for a, n, s, src in seq:
        if cur and cur['n'] == n: cur['k'] += 1; cur['s'] += s; cur['last'] = src
        else:
            cur = {'a': a, 'n': n, 'k': 1, 's': s, 'first': src, 'last': src}; blocks.append(cur)
    for b in blocks:
        w = b['n'] * b['k']
        if w / tot > 0.015 or b['s'] / tots > 0.03:
            print(f"{hex(b['a'])[-5:]} x{b['k']:3d} cnt={b['n']:11d} {w/tot*100:5.1f}% inst {b['s']/tots*100:5.1f}% stall | {b['first'][:42]} ... {b['last'][:38]}")
