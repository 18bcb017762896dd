"""GPU: distributed summa25_multiply through the C-ABI, one process per GPU
(torchrun), checked block-by-block against the CPU oracle.  Uses every GPU
the box exposes (1x1 on one GPU; 1x2 / 2x2 / 2x4 grids when more exist)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    import torch
    return torch.cuda.device_count()


def run_worker(nproc, *args, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", str(nproc),
           os.path.join(ROOT, "tests", "summa_worker.py"), *map(str, args)]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    return p.stdout


@pytest.mark.parametrize("sr,mode,two_round,fuse", [(4, 2, 1, 1), (4, 2, 1, 0), (2, 0, 1, 1), (1, 1, 0, 0),
                                                     (0, 2, 1, 1), (5, 2, 0, 1), (2, 2, 0, 0)])
def test_summa_all_gpus(sr, mode, two_round, fuse):
    n = ngpus()
    nproc = 8 if n >= 8 else 4 if n >= 4 else 2 if n >= 2 else 1
    out = run_worker(nproc, "--sr", sr, "--scale", 10, "--mode", mode, "--two-round", two_round, "--fuse", fuse)
    assert "blocks_ok=True checksum_ok=True" in out


def test_summa_host_path_chunked_staging():
    # tiny staging buffer forces the pipelined multi-chunk host-path broadcast
    n = ngpus()
    nproc = 2 if n >= 2 else 1
    out = run_worker(nproc, "--sr", 4, "--scale", 11, "--mode", 0, "--staging", 8192)
    assert "blocks_ok=True checksum_ok=True" in out


@pytest.mark.parametrize("grid", ["1x2", "2x2", "2x4", "1x4"])
@pytest.mark.parametrize("fuse", [1, 0])
def test_summa_grids_on_one_gpu_host_path(grid, fuse):
    """Every BASELINE grid shape, its ranks sharing the box's GPU(s) when
    there are fewer GPUs than ranks (no NCCL then: host-path broadcasts
    through the pinned shared-memory staging): schedule, panel slicing, size
    exchanges, broadcasts, fused or per-stage multiplies + merge, checked
    block by block against the oracle."""
    pr, pc = (int(x) for x in grid.split("x"))
    out = run_worker(pr * pc, "--sr", 4, "--scale", 10, "--grid", grid, "--fuse", fuse, "--mode", 0)
    assert "blocks_ok=True checksum_ok=True" in out


@pytest.mark.parametrize("grid", ["1x2", "2x2", "2x4"])
def test_summa_per_round_fusion_bounds_panel_memory(grid):
    """fuse_stages = 2 (one fused multiply per 2.5D round, the two round
    products folded by the GPU merge, merge_partials summa.hpp:122-172): C is
    exact, and the peak broadcast-buffer bytes per rank in two-round mode
    are at most the one-round peak (SPEC acceptance 9) — about half."""
    pr, pc = (int(x) for x in grid.split("x"))
    peaks = {}
    for two in (1, 0):
        out = run_worker(pr * pc, "--sr", 4, "--scale", 11, "--grid", grid, "--fuse", 2, "--mode", 0,
                         "--two-round", two)
        assert "blocks_ok=True checksum_ok=True" in out
        peaks[two] = int(out.split("peak_bcast_buffer_bytes_max=")[1].split()[0])
    assert 0 < peaks[1] <= peaks[0] and peaks[1] < 0.75 * peaks[0], peaks


@pytest.mark.parametrize("grid", ["1x1", "1x2", "2x2"])
def test_summa_streamed_checksum_output(grid):
    """output = checksum (SURVEY §8f-2, C larger than HBM): the fused product
    in many small column batches, each checksummed and released; the sum of
    the ranks' shares equals the oracle's matrix_checksum of C."""
    pr, pc = (int(x) for x in grid.split("x"))
    for sr in (2, 4):
        out = run_worker(pr * pc, "--sr", sr, "--scale", 11, "--grid", grid, "--mode", 0, "--output", "checksum",
                         "--batch-bytes", 1 << 16)
        assert "blocks_ok=True checksum_ok=True" in out


@pytest.mark.parametrize("sr", [1, 2, 4])
@pytest.mark.parametrize("two_round", [1, 0])
def test_summa_2x2_ledger_matches_reference(sr, two_round):
    """p = 4 (2 x 2) summa25_multiply of the golden R-MAT (scale 9, edge factor
    8, seed 3) in the reference structure (per-stage multiplies + merge): the
    distributed counters — broadcasts, size exchanges, local multiplies,
    skipped stages — and the checksum of C equal the reference's
    (tests/golden/make_golden.py section 6)."""
    out = run_worker(4, "--sr", sr, "--scale", 9, "--ef", 8, "--seed", 3, "--grid", "2x2", "--fuse", 0,
                     "--mode", 0, "--two-round", two_round, "--golden-ledger", f"summa_{sr}_p4_r{two_round}")
    assert "ledger_ok=True" in out and "blocks_ok=True checksum_ok=True" in out


@pytest.mark.parametrize("grid", ["1x4", "4x1", "1x2", "2x1"])
def test_summa_rectangular_grids(grid):
    """Non-square grids use the common-refinement stage schedule."""
    pr, pc = (int(x) for x in grid.split("x"))
    if pr * pc > ngpus():
        pytest.skip(f"needs {pr * pc} GPUs")
    for fuse in (1, 0):
        out = run_worker(pr * pc, "--sr", 4, "--scale", 10, "--grid", grid, "--fuse", fuse, "--mode", 2)
        assert "blocks_ok=True checksum_ok=True" in out


@pytest.mark.slow
@pytest.mark.skipif(os.environ.get("SPG_FULLSIZE") != "1", reason="full-size BASELINE configs: set SPG_FULLSIZE=1")
@pytest.mark.parametrize("config", [2, 4, 5, 3])
def test_fullsize_config_against_streaming_oracle(config):
    """BASELINE configs at full size on all GPUs vs the oracle's streaming
    checksum of the full C (tests/fullsize_worker.py)."""
    n = ngpus()
    nproc = 8 if n >= 8 else 4 if n >= 4 else 2 if n >= 2 else 1
    if config in (3, 5) and nproc < 4:
        pytest.skip("needs 4 GPUs (C does not fit fewer)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", str(nproc),
           os.path.join(ROOT, "tests", "fullsize_worker.py"), "--config", str(config)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=3000, cwd=ROOT,
                       env=dict(os.environ, MASTER_ADDR="127.0.0.1"))
    assert p.returncode == 0 and '"match": true' in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]


def test_threshold_sweep_same_product_every_threshold():
    """sweep_thresholds (tuner.hpp:64-99): every threshold of the ladder, from
    all-device to all-host, yields the identical C (checksums compared)."""
    n = ngpus()
    nproc = 4 if n >= 4 else 2 if n >= 2 else 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", str(nproc),
           os.path.join(ROOT, "tools", "threshold_sweep.py"), "--scale", "11", "--reps", "1"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env=dict(os.environ, MASTER_ADDR="127.0.0.1"))
    assert p.returncode == 0 and '"same_product_every_threshold": true' in p.stdout, p.stdout[-2000:] + p.stderr[-3000:]
    if nproc > 1:
        import json
        doc = json.loads(p.stdout.strip().splitlines()[-1])
        pct = [r["pct_host_bcasts"] for r in doc["rows"]]
        assert pct[0] == 0.0 and pct[-1] == 100.0  # threshold 0: all device; infinity: all host


@pytest.mark.parametrize("sr", [4, 0, 5])
def test_gather_full_c_on_root(sr):
    """gather: the blocks of C assembled on rank 0's GPU equal
    the oracle's full C (tropical / max-times bit-exact, fp64 within 1e-12)."""
    n = ngpus()
    nproc = 8 if n >= 8 else 4 if n >= 4 else 2 if n >= 2 else 1
    out = run_worker(nproc, "--sr", sr, "--scale", 10, "--gather", 1)
    assert "gather_ok=True" in out and "blocks_ok=True" in out
