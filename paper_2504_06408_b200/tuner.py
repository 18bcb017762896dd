"""Measured hybrid-communication tuning (replaces the reference's modelled
tuner: tuner.hpp:17-117 and latency_model.hpp:21-185).

The reference prices the host and device broadcast paths with synthetic
log-log latency curves; here the curves are MEASURED on the box through the
real transports (`spg_bcast`: pinned shared-memory staging vs NCCL over
NVLink), stored in the reference's JSON curve format, and the threshold is
the measured crossover (`find_crossover`, same bisection contract).
"""
from __future__ import annotations

import json
import math
import time
from typing import Dict, List, Optional, Sequence, Tuple

Curve = List[Tuple[float, float]]  # (bytes, seconds), strictly increasing bytes


def curve_at(curve: Curve, nbytes: float) -> float:
    """LatencyCurve::at (latency_model.hpp:44-55): piecewise-linear in log-log,
    extrapolated by the end segments."""
    if len(curve) < 2:
        raise ValueError("latency curve needs at least two sample points")
    x = math.log(max(nbytes, 1.0))
    hi = 1
    while hi + 1 < len(curve) and math.log(curve[hi][0]) < x:
        hi += 1
    x0, x1 = math.log(curve[hi - 1][0]), math.log(curve[hi][0])
    y0, y1 = math.log(curve[hi - 1][1]), math.log(curve[hi][1])
    return math.exp(y0 + (x - x0) / (x1 - x0) * (y1 - y0))


def find_crossover(host, device, lo: int = 1, hi: int = 1 << 30) -> Optional[int]:
    """find_crossover (tuner.hpp:17-39): smallest size in [lo, hi] where the
    host path stops being cheaper than the device path (1-byte bisection);
    None when there is no sign change in range.  `host`/`device` are curves
    or callables bytes -> seconds (the model's *_path_total)."""
    if lo >= hi:
        raise ValueError("find_crossover needs lo < hi")
    hf = host if callable(host) else (lambda b: curve_at(host, b))
    df = device if callable(device) else (lambda b: curve_at(device, b))

    def host_minus_device(b):
        return hf(b) - df(b)

    if host_minus_device(lo) >= 0.0 or host_minus_device(hi) < 0.0:
        return None
    while hi - lo > 1:
        mid = lo + (hi - lo) // 2
        if host_minus_device(mid) >= 0.0:
            hi = mid
        else:
            lo = mid
    return hi


def default_threshold_ladder(crossover: Optional[int]) -> List[int]:
    """default_threshold_ladder (tuner.hpp:101-117): 0, s*/32..s*/2, s*..16 s*, inf."""
    star = crossover if crossover else 1 << 16
    ladder = [0]
    for shift in range(5, 0, -1):
        t = star >> shift
        if t > 0 and t != ladder[-1]:
            ladder.append(t)
    for shift in range(0, 5):
        t = star << shift
        if t != ladder[-1]:
            ladder.append(t)
    ladder.append((1 << 64) - 1)
    return ladder


def broadcast_stages(fanout: int) -> int:
    """broadcast_stages (latency_model.hpp:66-71): ceil(log2(f)) curve evaluations."""
    if fanout < 1:
        raise ValueError("broadcast fanout must be >= 1")
    return int(fanout - 1).bit_length()


def to_reference_json(curves: Dict[str, Curve]) -> dict:
    """The reference's model file layout (latency_model.hpp:135-148)."""
    return {"curves": {k: [[float(b), float(t)] for b, t in v] for k, v in curves.items()}}


def measure_bcast_curves(comm, sizes: Sequence[int], reps: int = 10, scope: int = 0,
                         barrier=None, reduce_max=None, device: int = 0, fanout: int = 2) -> Dict[str, Curve]:
    """Times spg_bcast on this rank's `scope` (0 = grid row, 1 = grid column)
    for every size through each path: the host path (root D2H into pinned
    shared memory, peers H2D, pipelined) and the device path (NCCL broadcast
    over NVLink).  Each sample is the max over ranks of the median of `reps`
    runs (reduce_max combines across ranks).  Also times plain pinned D2H/H2D
    copies (the model's copy curves).  Returns curves keyed like the reference
    model plus `host_path_total` / `device_path_total`."""
    import torch

    from .summa import DEVICE_ONLY, HOST_ONLY

    buf = torch.empty(max(sizes), dtype=torch.uint8, device=f"cuda:{device}")
    pinned = torch.empty(max(sizes), dtype=torch.uint8, pin_memory=True)
    out: Dict[str, Curve] = {"host_path_total": [], "device_path_total": [], "copy_d2h": [], "copy_h2d": []}
    for nbytes in sizes:
        for key, mode in (("host_path_total", HOST_ONLY), ("device_path_total", DEVICE_ONLY)):
            ts = []
            for r in range(reps + 2):
                torch.cuda.synchronize()
                if barrier:
                    barrier()
                t0 = time.perf_counter()
                comm.bcast(scope, 0, buf.data_ptr(), nbytes, mode=mode, threshold=0)
                torch.cuda.synchronize()
                if r >= 2:
                    ts.append(time.perf_counter() - t0)
            med = sorted(ts)[len(ts) // 2]
            out[key].append((float(nbytes), reduce_max(med) if reduce_max else med))
        for key, fn in (("copy_d2h", lambda n: pinned[:n].copy_(buf[:n], non_blocking=True)),
                        ("copy_h2d", lambda n: buf[:n].copy_(pinned[:n], non_blocking=True))):
            ts = []
            for r in range(reps + 2):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                fn(nbytes)
                torch.cuda.synchronize()
                if r >= 2:
                    ts.append(time.perf_counter() - t0)
            out[key].append((float(nbytes), sorted(ts)[len(ts) // 2]))
    # reference-format curves are PER BROADCAST STAGE: the reference prices a
    # scope of f ranks as broadcast_stages(f) curve evaluations
    # (latency_model.hpp:88-106), so the measured fanout-f totals are divided
    # by that count; host_bcast is what remains of the host path after the
    # two staging copies, floored at 1 ns
    st = max(broadcast_stages(fanout), 1)
    out["host_bcast"] = [(b, max(t - d - h, 1e-9) / st) for (b, t), (_, d), (_, h) in
                         zip(out["host_path_total"], out["copy_d2h"], out["copy_h2d"])]
    out["device_bcast"] = [(b, t / st) for b, t in out["device_path_total"]]
    for k in out:  # the reference requires non-decreasing latencies
        pts, best = [], 0.0
        for b, t in out[k]:
            best = max(best, t)
            pts.append((b, best))
        out[k] = pts
    return out


def save_model(path: str, curves: Dict[str, Curve], extra: dict | None = None, fanout: int | None = None):
    doc = to_reference_json({k: curves[k] for k in ("host_bcast", "device_bcast", "copy_h2d", "copy_d2h")})
    if fanout is not None:
        doc["fanout"] = int(fanout)
    doc["measured"] = {k: [[b, t] for b, t in curves[k]] for k in ("host_path_total", "device_path_total")}
    if extra:
        doc.update(extra)
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)


INFINITE_THRESHOLD = (1 << 64) - 1  # kInfiniteThreshold: every payload on the host path


def model_path_totals(doc: dict, fanout: int):
    """The reference's host_path_total / device_path_total (latency_model.hpp:
    104-109) of a model file, as callables bytes -> seconds."""
    cv = {k: [(float(b), float(t)) for b, t in v] for k, v in doc["curves"].items()}
    st = broadcast_stages(fanout)

    def host(b):
        return curve_at(cv["copy_d2h"], b) + st * curve_at(cv["host_bcast"], b) + curve_at(cv["copy_h2d"], b)

    def device(b):
        return st * curve_at(cv["device_bcast"], b)
    return host, device


def calibrate_threshold(comm, scope: int, fanout: int, device: int, barrier, reduce_max, reps: int = 5,
                        min_log2: int = 10, max_log2: int = 26, cache_key: str | None = None) -> dict:
    """The hybrid threshold MEASURED on this box (north star: not hard-coded):
    host and device broadcast paths timed through the real transports on the
    `scope` communicator (fanout ranks) for 2^min_log2 .. 2^max_log2 bytes,
    crossover by the reference's bisection.  Collective over the scope's
    ranks.  Cached per GPU model/UUID set and fanout when `cache_key` is given
    (SPG_CALIB_DIR, default ~/.cache/paper_2504_06408_b200): a fresh box
    measures, a repeat run reuses.  Ranks sharing a GPU have no device path:
    every payload takes the host path."""
    import os
    if not comm.has_device_path:
        return {"threshold": INFINITE_THRESHOLD, "crossover": None, "source": "host path only (ranks share a GPU)"}
    path = None
    if cache_key:
        d = os.environ.get("SPG_CALIB_DIR", os.path.join(os.path.expanduser("~"), ".cache", "paper_2504_06408_b200"))
        path = os.path.join(d, f"calib_{cache_key}_f{fanout}_s{scope}.json")
        if os.path.exists(path):
            try:
                with open(path) as f:
                    doc = json.load(f)
                return {**doc["calibration"], "source": f"cached measurement {path}"}
            except (OSError, KeyError, ValueError):
                pass
    sizes = [1 << k for k in range(min_log2, max_log2 + 1)]
    curves = measure_bcast_curves(comm, sizes, reps=reps, scope=scope, barrier=barrier, reduce_max=reduce_max,
                                  device=device, fanout=fanout)
    host, dev = curves["host_path_total"], curves["device_path_total"]
    xo = find_crossover(host, dev, sizes[0], sizes[-1])
    if xo is None:  # one path wins everywhere in range
        thr = INFINITE_THRESHOLD if curve_at(host, sizes[-1]) < curve_at(dev, sizes[-1]) else 0
    else:
        thr = xo
    cal = {"threshold": int(thr), "crossover": xo, "fanout": fanout, "sizes": [sizes[0], sizes[-1]], "reps": reps}
    if path and comm.rank == 0:
        os.makedirs(os.path.dirname(path), exist_ok=True)
        save_model(path, curves, extra={"calibration": cal}, fanout=fanout)
    return {**cal, "source": "measured on this box at start-up"}


def crossover_warning(host, device, lo: int = 1, hi: int = 1 << 30) -> Optional[str]:
    """crossover_warning (tuner.hpp:43-53): text when the measured curves have
    no host/device crossover in range (hybrid routing then degenerates)."""
    if find_crossover(host, device, lo, hi) is not None:
        return None
    return ("latency model has no host/device crossover in its sampled range; "
            "hybrid routing will degenerate to a single path")


def sweep_thresholds(comm, ctx, a_block, n: int, thresholds: Sequence[int], allsum, allmax,
                     two_round: bool = True) -> List[dict]:
    """sweep_thresholds (tuner.hpp:64-99): runs C = A (x) A once per threshold
    under hybrid routing on this rank's block (every rank calls it with the
    same thresholds) and tabulates the host-handled broadcast percentage, the
    MEASURED broadcast time (the reference reports its simulated cost) and the
    local-multiply time, both max over ranks, plus the checksum of C.  Every
    run must produce the identical product: diverging checksums raise
    InternalError.  `allsum(int) -> int` / `allmax(float) -> float` reduce a
    value over all ranks (e.g. torch.distributed)."""
    from . import errors
    from .summa import HYBRID, checksum_part, checksum_seed, summa25_multiply

    rows: List[dict] = []
    for t in thresholds:
        c, led = summa25_multiply(comm, ctx, a_block, a_block, n, n, n, two_round=two_round, mode=HYBRID,
                                  threshold=int(t), threshold_col=int(t))
        part = checksum_part(c, a_block.rows[0], a_block.cols[0])
        c.free()
        lo, hi = allsum(part & 0xFFFFFFFF), allsum(part >> 32)
        checksum = (checksum_seed(n, n) + lo + (hi << 32)) % (1 << 64)
        host, dev = allsum(led["host_bcasts"]), allsum(led["device_bcasts"])
        if rows and checksum != rows[0]["result_checksum"]:
            raise errors.InternalError("threshold sweep runs produced different products; routing must "
                                       "not affect results")
        rows.append({"threshold_bytes": int(t),
                     "pct_host_bcasts": 0.0 if host + dev == 0 else 100.0 * host / (host + dev),
                     "comm_seconds": allmax(led["ms"]["broadcast"]) / 1e3,
                     "wall_local_seconds": allmax(led["ms"]["local_multiply"]) / 1e3,
                     "time_to_c_seconds": allmax(led["ms_total"]) / 1e3,
                     "result_checksum": checksum})
    return rows
