#!/usr/bin/env python
"""Benchmark: semiring SpGEMM Gflop/s and time-to-C on B200 (BASELINE.json).

N = 1  : BASELINE config 2 — C = A.A, A = R-MAT scale 18 / edge factor 16,
         (min, +) int32 tropical semiring, local multiply on one B200.
N > 1  : the same C = A.A through Sparse SUMMA (2.5D, hybrid broadcasts) on a
         1x2 / 2x2 / 2x4 grid, one process per GPU (torchrun), strong scaling.

A "step" is one full C = A.A (every product formed, every row folded, exact
C materialised in HBM).  value = 2F / step time (semiring Gflop/s, F =
intermediate products); e2e = the same metric through the reference-shaped
host call (host CSR in, host CSR out, all copies timed).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "semiring SpGEMM Gflop/s & time-to-C at 1/2/4/8 B200 vs CPU ref"
GRIDS = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}
# matrix_checksum (checksum.hpp:20-38) of C = A.A from the CPU oracle's streaming
# restatement (oracle/spg_oracle.cpp, pinned to the reference): the bench
# checks its own C against these after the timed loop ("parity" in the line).
# keys: R-MAT (config, scale, edge factor, seed, permuted); stencil (4, N);
# ER (5, log2 n, d, seed) — configs 4 and 5 from tools/golden_checksums.py
GOLDEN_CSUM = {
    (2, 18, 16.0, 1, True): 7149000290918998130,
    (2, 18, 16.0, 1, False): 10351070082044141371,
    (3, 22, 16.0, 1, True): 216229255003959338,
    (4, 252): 16022149531309518969,  # nnz(C) = 1971935064, products = 11512557512
    (5, 22, 64, 1): 3744257256882867897,  # nnz(C) = 17171350284, products = 17179606120
}


def d2h_index_bytes(nnz, procs=1):
    """Column-index bytes of a host download: 2^25-entry chunks, a share
    (SPG_D2H_GPU_WIDEN; library default 0.1 for one process on the host, 1
    when several share it) widened on the GPU and sent as int64, the rest
    sent as int32 and widened on the host."""
    chunk = 1 << 25
    nch = (nnz + chunk - 1) // chunk
    frac = min(max(float(os.environ.get("SPG_D2H_GPU_WIDEN", "0.1" if procs == 1 else "1")), 0.0), 1.0)
    gpu = sum(1 for k in range(nch) if frac > 0 and int(frac * (k + 1) + 1e-9) > int(frac * k + 1e-9))
    wide = sum(min(chunk, nnz - k * chunk) for k in range(nch)
               if frac > 0 and int(frac * (k + 1) + 1e-9) > int(frac * k + 1e-9))
    return 4 * nnz + 4 * wide if gpu else 4 * nnz


def golden_key(args):
    if args.config == 4:
        return (4, args.stencil_n)
    if args.config == 5:
        return (5, args.er_log2, args.er_d, args.seed)
    return (args.config, args.scale, args.ef, args.seed, bool(args.permute))


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j.get("hbm_gbs", 6553.9)), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler running DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        # nvidia-smi's NVML start-up takes driver locks that can stall the GPU
        # for hundreds of ms: wait for its second sample before timing starts
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < 10.0:
            self.f.flush()
            if os.path.getsize(self.path) > 0:
                with open(self.path) as fh:
                    if fh.read().count("\n") >= 2:
                        break
            time.sleep(0.05)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons)}
        busy = sorted(sm)[len(sm) // 4:] or sm
        return {"sm_mhz": float(np.median(busy)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def make_input(scale, ef, seed, sr=4, permute=False):
    from paper_2504_06408_b200 import generators
    from paper_2504_06408_b200.generators import coo_to_csr_fast
    t0 = time.time()
    coo = generators.generate_rmat(sr, scale, ef, seed)
    if permute:
        coo = generators.permute_symmetric(coo, seed)
    a = coo_to_csr_fast(coo)
    log(f"[bench] R-MAT s{scale} ef{ef}: n={a.nrows} nnz={a.nnz} (gen {time.time() - t0:.1f}s)")
    return a


def workload(args):
    """BASELINE.json configs 2-5: generator, semiring,
    sizes and the closed-form / measured totals the run must reproduce."""
    c = args.config
    if c == 2:
        return {"gen": "rmat", "sr": 4, "n": 1 << args.scale, "vs": 4, "dtype": "int32",
                "name": f"rmat{args.scale}_ef{int(args.ef)}_tropical_i32_AxA (BASELINE config 2)",
                "expect": {"products": 2934326978, "nnz_C": 1281547801} if (args.scale, args.ef) == (18, 16.0)
                else None}
    if c == 3:
        return {"gen": "rmat", "sr": 2, "n": 1 << args.scale, "vs": 1, "dtype": "u8",
                "name": f"rmat{args.scale}_ef{int(args.ef)}_boolean_AxA (BASELINE config 3)", "expect": None}
    if c == 4:
        N = args.stencil_n
        return {"gen": "stencil27", "sr": 0, "n": N ** 3, "N": N, "vs": 8, "dtype": "f64",
                "name": f"stencil27_N{N}_fp64_AxA (BASELINE config 4)",
                "expect": {"products": (9 * N - 10) ** 3, "nnz_C": (5 * N - 6) ** 3}}
    if c == 5:
        n = 1 << args.er_log2
        return {"gen": "er", "sr": 5, "n": n, "d": args.er_d, "value_mode": 1, "vs": 16, "dtype": "f64+u64",
                "name": f"er2^{args.er_log2}_d{args.er_d}_maxtimes_struct_AxA (BASELINE config 5)", "expect": None}
    raise SystemExit(f"--config {c}: choose 2, 3, 4 or 5")


def b_alg(nnz_l, nrows, F, nnz_c, vs):
    """nnz(L)(12+V) + F(4+V) + nnz(C)(4+V) + 8(rows+1)."""
    return nnz_l * (12 + vs) + F * (4 + vs) + nnz_c * (4 + vs) + 8 * (nrows + 1)


def cpu_sample(a, target_products, sr):
    """Row-subsample of A (every s-th row) with about target_products products in A_s . A."""
    rowlen = np.diff(a.rowptr)
    prod_row = np.zeros(a.nrows, dtype=np.int64)
    # products of row i = sum over its columns k of len(row k)
    seg = np.repeat(np.arange(a.nrows), rowlen)
    np.add.at(prod_row, seg, rowlen[a.colids])
    total = int(prod_row.sum())
    stride = max(1, int(round(total / max(target_products, 1))))
    rows = np.arange(0, a.nrows, stride)
    lens = rowlen[rows]
    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = np.concatenate([a.colids[a.rowptr[r]:a.rowptr[r + 1]] for r in rows]).astype(np.int64)
    vals = np.concatenate([a.values[a.rowptr[r]:a.rowptr[r + 1]] for r in rows])
    return rows.size, ptr, idx, vals, int(prod_row[rows].sum()), stride


def cpu_reference_gflops(a, sr, target_products, nthreads=None):
    """The unmodified reference esc_multiply (oracle/_ref), all host threads,
    on a bounded row sample of the same C = A.A."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_bind as ob
    nthreads = nthreads or os.cpu_count() or 1
    nrow_s, ptr, idx, vals, F_s, stride = cpu_sample(a, target_products, sr)
    A_s = ob.Mat(sr, nrow_s, a.ncols, ptr, idx, vals)
    A = ob.Mat(sr, a.nrows, a.ncols, a.rowptr, a.colids, a.values)
    if ob.ref is not None:
        sec, nnz, fl, _ = ob.ref_esc_rows_mt(A_s, A, 0, nrow_s, nthreads)
        kind = "reference"
    else:  # prebuilt reference missing: time the oracle restatement instead
        t0 = time.perf_counter()
        _, nnz, fl, _ = ob.orc_stream(A_s, A, nthreads=nthreads)
        sec = time.perf_counter() - t0
        kind = "port"
    return {"value": 2.0 * fl / sec / 1e9, "unit": "Gflop/s", "cores": nthreads, "kind": kind,
            "sample": f"rows i % {stride} == 0 of A ({nrow_s} rows) times A: F={fl} products, "
                      f"nnz={nnz}, {sec:.2f} s, esc_multiply on {nthreads} threads over disjoint row slices",
            "seconds": sec}


def host_info():
    """nproc, CPU model and host RAM of the box (recorded beside the CPU numbers)."""
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    mem_gb = None
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                mem_gb = round(int(line.split()[1]) / 2**20, 1)
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "host_ram_gb": mem_gb}


def reference_input(args):
    """A for the reference arm, built by the REFERENCE itself (oracle/_ref:
    generate_rmat, rmat.hpp:15-60, and coo_to_csr) plus the same seeded
    relabelling in numpy — the reference process never loads this repo's
    library."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_bind as ob
    _, _, r, c, v = ob.ref_generate_rmat(4, args.scale, args.ef, args.seed)
    n = 1 << args.scale
    if args.permute:  # generators.permute_symmetric: entry (i, j) -> (p[i], p[j])
        perm = np.random.default_rng(args.seed).permutation(n).astype(np.int64)
        r, c = perm[r], perm[c]
    m = ob.ref_coo_to_csr(4, n, n, r, c, v)

    class _Csr:  # the fields cpu_reference_gflops reads
        nrows, ncols = m.nrows, m.ncols
        rowptr, colids, values = m.ptr, m.idx, m.vals
        nnz = int(m.ptr[-1])
    return _Csr


def run_reference_arm(args):
    """`--impl reference`: the reference CPU implementation on the host cores:
    its esc_multiply (local_spgemm.hpp:83-156, compiled unmodified into
    oracle/_ref) over disjoint row slices of the same C = A.A on every host
    thread, each step a bounded row sample (the full product needs ~24 B per
    product = ~70 GB of expand-sort-compress tuples)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_bind as ob
    if ob.ref is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libspsumma_ref.so not built"}), flush=True)
        return
    a = reference_input(args)
    times = []
    res = None
    for i in range(args.warmup + args.steps):
        res = cpu_reference_gflops(a, 4, args.cpu_products)
        if i >= args.warmup:
            times.append(res["seconds"])
    gflops = [2.0 * float(res["sample"].split("F=")[1].split(" ")[0]) / t / 1e9 for t in times]
    val = float(np.median(gflops))
    hi = host_info()
    F_full = 2934326978 if (args.scale, args.ef) == (18, 16.0) else None
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "Gflop/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.median(times)) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "config": {"workload": f"rmat{args.scale}_ef{int(args.ef)}_tropical_i32_AxA (BASELINE config 2)",
                                            "permuted": bool(args.permute), "sample": res["sample"],
                                            "input": "generated and compressed by the reference (oracle/_ref)",
                                            "summa25_multiply_full": "infeasible here: ~24 B x F = "
                                            + (f"{24 * F_full / 1e9:.0f} GB" if F_full else "24 B x F")
                                            + " of expand-sort-compress tuples vs host RAM " + str(hi["host_ram_gb"]) + " GB",
                                            **hi},
            "cpu_baseline": {"value": val, "unit": "Gflop/s", "cores": res["cores"], "kind": res["kind"],
                             "sample": res["sample"]},
            "e2e": {"value": val, "unit": "Gflop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_single(args):
    import torch

    from paper_2504_06408_b200 import Context, DeviceCsr, esc_multiply, local_multiply
    from paper_2504_06408_b200._lib import DCsr, MultStats, check, lib

    sr = 4
    vs = 4
    a = make_input(args.scale, args.ef, args.seed, permute=args.permute)
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    ctx = Context(0)
    check(lib.spg_ctx_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)), ctx.handle)
    d = DeviceCsr.upload(ctx, a)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    st = {}
    for _ in range(args.warmup):
        c = local_multiply(d, d, stats=st)
        c.free()
    torch.cuda.synchronize()
    F, nnz_c = st["products"], st["nnz_out"]
    log(f"[bench] F={F} nnz(C)={nnz_c} bins={st['rows_per_bin']} phases: analyse {st['ms_analyse']:.2f} "
        f"numeric {st['ms_numeric']:.2f} compact {st['ms_compact']:.2f} ms")

    times = []
    launches0 = ctx.kernel_launches()
    with Clocks(0) as clk:
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            c = local_multiply(d, d)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            if len(times) < args.steps:
                c.free()
    launches = ctx.kernel_launches() - launches0
    # parity: the last timed C against the oracle's checksum of the same product
    csum = c.checksum()
    c.free()
    # the dominant kernel's share: one untimed call with per-phase CUDA events
    st2 = {}
    local_multiply(d, d, stats=st2).free()
    golden = GOLDEN_CSUM.get((2, args.scale, args.ef, args.seed, bool(args.permute)))
    parity = None if golden is None else bool(csum == golden)
    ms = float(np.mean(times))
    gflops = 2.0 * F / (ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    balg = b_alg(a.nnz, a.nrows, F, nnz_c, vs)
    achieved = balg / (ms * 1e-3) / 1e9

    # e2e: reference-shaped host call esc_multiply(A, A): H2D, multiply, D2H of C
    from paper_2504_06408_b200.device import pin
    unpin = pin(a.rowptr, a.colids, a.values)  # inputs in pinned host memory
    e2e_times = []
    h2d = 2 * (8 * (a.nrows + 1) + 8 * a.nnz + vs * a.nnz)
    d2h = 8 * (a.nrows + 1) + vs * nnz_c + d2h_index_bytes(nnz_c)  # rowptr + values + column indices
    for k in range(args.e2e_steps + (1 if args.e2e_steps > 0 else 0)):
        t0 = time.perf_counter()
        ch = esc_multiply(a, a, ctx=ctx)
        if k == 0:  # untimed warm-up: first touch of the pinned result buffers
            del ch
            continue
        e2e_times.append(time.perf_counter() - t0)
        assert ch.nnz == nnz_c
        del ch
    e2e_s = float(np.median(e2e_times)) if e2e_times else float("nan")
    unpin()

    # companion measurement on the generator's own vertex order (SURVEY §7:
    # the relabelled input is reported beside the unpermuted one)
    unperm = None
    if args.permute and not args.no_unpermuted:
        del d
        a_u = make_input(args.scale, args.ef, args.seed, permute=False)
        d_u = DeviceCsr.upload(ctx, a_u)
        for _ in range(2):
            local_multiply(d_u, d_u).free()
        t_u = []
        for k in range(3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            c_u = local_multiply(d_u, d_u)
            e1.record(stream)
            torch.cuda.synchronize()
            t_u.append(e0.elapsed_time(e1))
            if k < 2:
                c_u.free()
        cs_u = c_u.checksum()
        c_u.free()
        g_u = GOLDEN_CSUM.get((2, args.scale, args.ef, args.seed, False))
        ms_u = float(np.mean(t_u))
        unperm = {"ms_per_step": ms_u, "value": 2.0 * F / (ms_u * 1e-3) / 1e9, "unit": "Gflop/s",
                  "roofline_frac": b_alg(a_u.nnz, a_u.nrows, F, nnz_c, vs) / (ms_u * 1e-3) / 1e9 / peak,
                  "parity": None if g_u is None else bool(cs_u == g_u), "steps": 3, "warmup": 2}
        del d_u

    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_reference_gflops(a, sr, args.cpu_products)
        cpu.pop("seconds", None)
        cpu.update(host_info())

    traffic, fold_dram = None, None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            traffic = tj.get(f"rmat{args.scale}")
            fold_dram = next((v["bytes"] for k, v in tj.get("per_kernel", {}).items() if "br_numeric" in k), None)
        except Exception:
            traffic = None
    dominant = None
    if st2.get("output_mode") == 3 and st2.get("ms_fold", 0) > 0:
        # rank-space fold (br_numeric_kernel): gathers of R's (col, value) per product,
        # C written once, the window bitmaps read back (SURVEY §8d terms)
        fb = F * (4 + vs) + nnz_c * (4 + vs) + int(st2["bitmap_bytes"])
        ach = fb / (st2["ms_fold"] * 1e-3) / 1e9
        dominant = {"kernel": "br_numeric_kernel (rank-space fold into C)", "ms": st2["ms_fold"],
                    "share_of_multiply": st2["ms_fold"] / st2["ms_total"], "algorithmic_bytes": fb,
                    "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": fold_dram,
                    "work_items": st2["fold_items"],
                    "note": "phase time by CUDA events on the context stream around the fold (short-row "
                            "compaction runs beside it); F and nnz(C) of the whole multiply (the long rows hold "
                            "~99% of F); traffic = ncu dram bytes of the kernel (profiles/traffic.json)"}
    line = {
        "metric": METRIC, "value": gflops, "unit": "Gflop/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"rmat{args.scale}_ef{int(args.ef)}_tropical_i32_AxA (BASELINE config 2)",
                   "grid": "1x1", "permuted": bool(args.permute), "products": F, "nnz_A": a.nnz, "nnz_C": nnz_c,
                   "local_multiply_ms": ms,
                   "local_multiply_ms_note": "device-resident A, C materialised in HBM; the host round trip is e2e",
                   "steps_ms": [round(float(x), 3) for x in times],
                   "unpermuted": unperm,
                   "phases_ms_untimed_warmup_call": {k: round(st[k], 3) for k in ("ms_analyse", "ms_numeric",
                                                                                    "ms_compact")},
                   "rows_per_bin": st["rows_per_bin"], "output_mode": st["output_mode"],
                   "l2": "flushed between steps (512 MB write)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "note": f"B_alg of the whole local multiply (SURVEY §8d) / its event time; peak {peak_kind}",
                     "dominant_kernel": dominant},
        "parity": parity,
        "parity_check": {"checksum_C": csum, "golden": golden,
                         "how": "matrix_checksum (checksum.hpp:20-38) of the last timed C vs the CPU oracle's"},
        "cpu_baseline": cpu,
        "e2e": (None if args.e2e_steps <= 0 else
                {"value": 2.0 * F / e2e_s / 1e9, "unit": "Gflop/s", "h2d_bytes_per_step": h2d,
                 "d2h_bytes_per_step": d2h, "seconds": e2e_s}),
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def run_summa(args):
    """N GPUs, one process each (torchrun): C = A.A through summa25_multiply on
    a 1x2 / 2x2 / 2x4 grid.  Time-to-C per step = host-resident distributed
    blocks -> device-resident merged C blocks (prepare H2D, size exchanges,
    broadcasts, local multiplies, merge), device-timed, max over ranks."""
    import uuid

    import torch
    import torch.distributed as dist

    from paper_2504_06408_b200 import Context, generators
    from paper_2504_06408_b200._lib import check, lib
    from paper_2504_06408_b200.summa import (DEVICE_ONLY, HOST_ONLY, HYBRID, Comm, checksum_part, checksum_seed,
                                             distribute, grid_for, summa25_multiply)

    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29511")
    torch.cuda.set_device(local)
    import datetime
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=600))
    job = [uuid.uuid4().hex[:12] if rank == 0 else None]
    dist.broadcast_object_list(job, src=0)
    wl = workload(args)
    if args.grid:
        pr, pc = (int(x) for x in args.grid.split("x"))
    elif wl["gen"] == "stencil27":  # banded: 1 x N keeps every rank's block column equally loaded
        pr, pc = 1, world
    else:
        pr, pc = grid_for(world)
    if pr * pc != world:
        raise SystemExit(f"--grid {args.grid} does not hold {world} ranks")
    i, j = rank // pc, rank % pc
    mode = {"host": HOST_ONLY, "device": DEVICE_ONLY, "hybrid": HYBRID}[args.comm]

    t_gen = time.time()
    ctx = Context(local)
    sr, n = wl["sr"], wl["n"]
    from paper_2504_06408_b200.summa import block_from_piece, block_range
    rr, cr = block_range(n, pr, i), block_range(n, pc, j)
    if wl["gen"] == "rmat":
        coo = generators.generate_rmat(sr, args.scale, args.ef, args.seed)
        if args.permute:
            coo = generators.permute_symmetric(coo, args.seed)
        blk = distribute(ctx, coo, pr, pc, only_rank=rank)  # on the GPU: this rank's block only
        del coo
    elif wl["gen"] == "stencil27":
        blk = block_from_piece(generators.generate_stencil27_block(sr, wl["N"], rr, cr), rr, cr)
    else:
        blk = block_from_piece(generators.generate_er_block(sr, n, wl["d"], args.seed, rr, cr,
                                                            value_mode=wl["value_mode"]), rr, cr)
    log(f"[bench] rank {rank}: block {rr}x{cr} nnz={blk.storage.nnz} (gen {time.time() - t_gen:.1f}s)")
    # the distributed input blocks live in page-locked host memory (the
    # library's pinned allocator), as a production caller would keep them
    from paper_2504_06408_b200.device import pinned_copy
    st = blk.storage
    for k in ("colptr", "jc", "cp", "rowids", "values"):
        if hasattr(st, k):
            setattr(st, k, pinned_copy(getattr(st, k)))
    stream = torch.cuda.current_stream()
    check(lib.spg_ctx_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream)), ctx.handle)
    comm = Comm(job[0], world, rank, pr, pc, local, staging_bytes=64 << 20)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    # hybrid thresholds measured on THIS box at start-up (untimed), per scope
    if args.threshold >= 0:
        thr, thr_col, thr_info = args.threshold, args.threshold, {"source": "--threshold"}
    else:
        from paper_2504_06408_b200.summa import calibrated_thresholds

        def _rmax(x):
            tt = torch.tensor([x], dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            return float(tt[0])
        thr, thr_col, thr_info = calibrated_thresholds(comm, local, dist.barrier, _rmax)

    # C blocks larger than HBM (config 3 / 5 on 1-2 GPUs: 90-360 GB per rank)
    # are streamed: column batches, each checksummed and released (§8f-2)
    output = args.output
    if output == "auto":
        output = "checksum" if (args.config in (3, 5) and world <= 2) else "block"

    def step():
        c, led = summa25_multiply(comm, ctx, blk, blk, n, n, n, two_round=not args.one_round, mode=mode,
                                  threshold=thr, threshold_col=thr_col, fuse_stages=not args.no_fuse, output=output)
        return c, led

    for _ in range(args.warmup):
        c, led = step()
        c.free()
    times, leds = [], []
    launches0 = ctx.kernel_launches()
    with Clocks(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            c, led = step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            leds.append(led)
            if len(times) < args.steps:
                c.free()
    launches = ctx.kernel_launches() - launches0
    part = checksum_part(c, blk.rows[0], blk.cols[0]) if output == "block" else leds[-1]["checksum_part"]
    nnz_blk = c.nnz if output == "block" else leds[-1]["nnz_out"]
    c.free()
    # e2e: the same call plus the D2H read of this rank's C block (host
    # result); skipped (--e2e-steps 0) when C blocks exceed host RAM
    e2e_local, d2h = float("nan"), 0
    if args.e2e_steps > 0 and output == "block":
        for k in range(2):  # k == 0: untimed warm-up of the pinned result buffers
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            c2, _ = step()
            host_c = c2.download()
            e2e_local = time.perf_counter() - t0
            if k == 0:
                del host_c
                c2.free()
        d2h = 8 * (host_c.ncols + 1) + wl["vs"] * host_c.nnz + d2h_index_bytes(host_c.nnz, world)
        del host_c
        c2.free()

    t = torch.tensor(times, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # this rank's algorithmic bytes of its local multiply
    balg_r = b_alg(leds[-1]["left_nnz"], blk.cols[1] - blk.cols[0], leds[-1]["products"], nnz_blk, wl["vs"])
    agg = torch.tensor([float(leds[-1]["products"]), float(nnz_blk), float(part & 0xFFFFFFFF), float(part >> 32),
                        float(launches), float(d2h), float(balg_r)], dtype=torch.float64)
    dist.all_reduce(agg, op=dist.ReduceOp.SUM)
    e2e_t = torch.tensor([e2e_local], dtype=torch.float64)
    dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    mine = torch.tensor([times[-1], leds[-1]["ms_total"]] + [leds[-1]["ms"][k] for k in
                        ("prepare", "broadcast", "local_multiply", "merge")] + [float(leds[-1]["products"])],
                        dtype=torch.float64)
    allr = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allr, mine)
    ms = float(t.mean())
    F = int(agg[0])
    if rank == 0:
        led0 = leds[-1]
        csum = (checksum_seed(n, n) + int(agg[2]) + (int(agg[3]) << 32)) % (1 << 64)
        peak, peak_kind = peaks()
        h2d = 8 * (blk.storage.ncols + 1) + (8 + wl["vs"]) * blk.storage.nnz
        nnz_c = int(agg[1])
        golden = GOLDEN_CSUM.get(golden_key(args))
        achieved = float(agg[6]) / (ms * 1e-3) / 1e9
        line = {
            "metric": METRIC, "value": 2.0 * F / (ms * 1e-3) / 1e9, "unit": "Gflop/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": wl["dtype"], "data": "synthetic",
            "config": {"workload": wl["name"] + " via summa25_multiply", "baseline_config": args.config,
                       "grid": f"{pr}x{pc}", "permuted": bool(args.permute and wl["gen"] == "rmat"),
                       "two_round": not args.one_round,
                       "fuse_stages": not args.no_fuse,
                       "comm": args.comm,
                       "threshold_bytes": {"row_scope": thr, "col_scope": thr_col,
                                           "calibration": thr_info},
                       "products": F, "nnz_C": nnz_c, "checksum_C": csum,
                       "expected": wl.get("expect"),
                       "matches_expected": (None if not wl.get("expect") else
                                            all({"products": F, "nnz_C": nnz_c}[k] == v
                                                for k, v in wl["expect"].items())),
                       "time_to_C_ms": ms, "steps_ms_max_over_ranks": [round(float(x), 2) for x in t],
                       "rank0_ledger": led0,
                       "per_rank_ms": [{"event": round(float(x[0]), 2), "ledger_total": round(float(x[1]), 2),
                                        "prepare": round(float(x[2]), 2), "bcast": round(float(x[3]), 2),
                                        "multiply": round(float(x[4]), 2), "merge": round(float(x[5]), 2),
                                        "products": int(x[6])} for x in allr],
                       "l2": "flushed between steps (512 MB write)", "parallelism": f"summa{pr}x{pc}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * world, "unit": "GB/s",
                         "frac": achieved / (peak * world), "traffic": None,
                         "note": f"sum over ranks of each rank's local-multiply B_alg (SURVEY §8d) / time-to-C (max over "
                                 f"ranks, broadcasts included) vs {world} x the {peak_kind} HBM peak"},
            "parity": None if golden is None else bool(csum == golden),
            "parity_check": {"checksum_C": csum, "golden": golden,
                             "how": "sum over ranks of matrix_checksum terms (checksum.hpp:20-38) vs the CPU oracle's"},
            "output": output,
            "cpu_baseline": None,
            "e2e": (None if args.e2e_steps <= 0 else
                    {"value": 2.0 * F / float(e2e_t[0]) / 1e9, "unit": "Gflop/s", "h2d_bytes_per_step": 2 * h2d,
                     "d2h_bytes_per_step": int(agg[5]), "seconds": float(e2e_t[0])}),
            "gpu_launches": int(agg[4]), "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


def main():
    if os.environ.get("SPG_DEBUG_HANG"):
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["SPG_DEBUG_HANG"]), exit=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, help="BASELINE.json config (2 = default N=1 line; 3, 4, 5 "
                    "run through summa25_multiply)")
    ap.add_argument("--scale", type=int, default=0, help="R-MAT scale (default 18 for config 2, 22 for config 3)")
    ap.add_argument("--stencil-n", type=int, default=252)
    ap.add_argument("--er-log2", type=int, default=22)
    ap.add_argument("--er-d", type=int, default=64)
    ap.add_argument("--ef", type=float, default=16.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-products", type=float, default=0.0,
                    help="products in the CPU sample (default: 3e7 per host core, at most 1e9)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-unpermuted", action="store_true", help="skip the companion unpermuted N=1 measurement")
    ap.add_argument("--summa", action="store_true", help="use the SUMMA path even on one GPU (1x1 grid)")
    ap.add_argument("--one-round", action="store_true", help="SummaOptions::two_round = false")
    ap.add_argument("--no-fuse", action="store_true", help="per-stage multiplies + merge_partials (reference structure)")
    ap.add_argument("--no-permute", dest="permute", action="store_false",
                    help="use the generator's vertex order (default: relabel vertices by a seeded random "
                         "permutation, as CombBLAS does, so grid blocks carry equal work; F and nnz(C) unchanged)")
    ap.add_argument("--comm", default="hybrid", choices=["host", "device", "hybrid"])
    ap.add_argument("--output", default="auto", choices=["auto", "block", "checksum"],
                    help="SUMMA C block: materialised in HBM, or streamed in checksummed column batches (auto: "
                         "streamed for configs 3 and 5 on 1-2 GPUs, whose C blocks exceed HBM)")
    ap.add_argument("--grid", default="", help="PRxPC process grid (default 1x1/1x2/2x2/2x4 by GPU count)")
    ap.add_argument("--threshold", type=int, default=-1, help="hybrid threshold bytes (-1: measured default)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.scale <= 0:
        args.scale = 22 if args.config == 3 else 18
    if args.cpu_products <= 0:
        args.cpu_products = min(1e9, 3e7 * (os.cpu_count() or 1))
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if args.gpus == 1 and int(os.environ.get("WORLD_SIZE", "1")) == 1 and not args.summa and args.config == 2:
        run_single(args)
    else:
        run_summa(args)


if __name__ == "__main__":
    main()
