"""CPU (no GPU): the SUMMA data flow of summa25_multiply across real
processes (gloo, world size 2, 4 and 8) — block distribution (local_block /
block_range, dist_matrix.hpp:23-111), the stage schedule (spg_summa_schedule:
the reference's q stages on square grids, the common refinement on
rectangular ones, summa.hpp:248-330), panel slicing at a_off / b_off, the
row-scope A and column-scope B broadcasts, and the stage-ordered fold — with
the per-stage local products computed densely on the host (tropical min-plus,
exact), so the assembled C must equal A (x) A bit for bit.  The device path
runs the same schedule with CUDA kernels (tests/test_gpu_summa.py)."""
import ctypes as C
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

INF = np.iinfo(np.int32).max


def _dense(block, nrows, ncols):
    """Tropical dense matrix of a CSC / DCSC block (zero = INT32_MAX)."""
    from paper_2504_06408_b200.formats import DcscMatrix
    d = np.full((nrows, ncols), INF, dtype=np.int64)
    s = block.storage
    if isinstance(s, DcscMatrix):
        for q, col in enumerate(s.jc):
            for e in range(s.cp[q], s.cp[q + 1]):
                d[s.rowids[e], col] = s.values[e]
    else:
        for col in range(s.ncols):
            for e in range(s.colptr[col], s.colptr[col + 1]):
                d[s.rowids[e], col] = s.values[e]
    return d


def _minplus(a, b):
    """(min, +) product with saturation at INT32_MAX (semiring.hpp TropicalI32)."""
    out = np.full((a.shape[0], b.shape[1]), INF, dtype=np.int64)
    for k in range(a.shape[1]):
        s = np.minimum(a[:, k:k + 1] + b[k:k + 1, :], INF)
        s[(a[:, k:k + 1] == INF) | (b[k:k + 1, :] == INF)] = INF
        out = np.minimum(out, s)
    return out


def _worker(rank, world, pr, pc, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_06408_b200 import generators
        from paper_2504_06408_b200._lib import Stage, lib
        from paper_2504_06408_b200.summa import local_block

        i, j = rank // pc, rank % pc
        coo = generators.generate_rmat(4, 7, 8.0, 3)
        n = coo.nrows
        blk = local_block(coo, pr, pc, i, j)
        a_loc = _dense(blk, blk.rows[1] - blk.rows[0], blk.cols[1] - blk.cols[0])
        row_groups = [dist.new_group([r * pc + c for c in range(pc)]) for r in range(pr)]
        col_groups = [dist.new_group([r * pc + c for r in range(pr)]) for c in range(pc)]
        stages = (Stage * 64)()
        ns = lib.spg_summa_schedule(n, pr, pc, stages, 64)
        assert 0 < ns <= 64
        c_loc = np.full(a_loc.shape[0:1] + (blk.cols[1] - blk.cols[0],), INF, dtype=np.int64)
        for st in stages[:ns]:
            width = st.hi - st.lo
            # A panel: block row i, inner columns [lo, hi) from grid column a_col_block
            apan = [a_loc[:, st.a_off:st.a_off + width] if j == st.a_col_block else None]
            dist.broadcast_object_list(apan, src=i * pc + st.a_col_block, group=row_groups[i])
            # B panel (B = A): inner rows [lo, hi), block column j, from grid row b_row_block
            bpan = [a_loc[st.b_off:st.b_off + width, :] if i == st.b_row_block else None]
            dist.broadcast_object_list(bpan, src=st.b_row_block * pc + j, group=col_groups[j])
            c_loc = np.minimum(c_loc, _minplus(apan[0], bpan[0]))  # fold in stage order
        blocks = [None] * world if rank == 0 else None
        dist.gather_object((blk.rows, blk.cols, c_loc), blocks, dst=0)
        if rank == 0:
            full = np.full((n, n), INF, dtype=np.int64)
            for (r0, r1), (c0, c1), cb in blocks:
                full[r0:r1, c0:c1] = cb
            a = np.full((n, n), INF, dtype=np.int64)
            a[coo.rows, coo.cols] = coo.values
            want = _minplus(a, a)
            assert np.array_equal(full, want)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported through the queue
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,pr,pc", [(2, 1, 2), (2, 2, 1), (4, 2, 2), (8, 2, 4)])
def test_summa_dataflow_multiprocess(world, pr, pc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + (os.getpid() % 1000) + 7 * world + pr
    procs = [ctx.Process(target=_worker, args=(r, world, pr, pc, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
