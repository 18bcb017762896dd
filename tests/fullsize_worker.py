"""torchrun worker: a BASELINE configuration at FULL size through
summa25_multiply, checked against the CPU oracle's streaming restatement
(row-parallel SPA over all host cores; the reference itself
cannot hold these products in RAM).  Every rank builds only its own block,
multiplies, and contributes its checksum part; rank 0 rebuilds the full A,
streams A (x) A through the oracle on all host threads and compares the
order-free checksum, nnz(C) and the product count.

    torchrun --nproc-per-node 4 tests/fullsize_worker.py --config 4
"""
import argparse
import datetime
import json
import os
import sys
import time
import uuid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--scale", type=int, default=0)
    ap.add_argument("--stencil-n", type=int, default=252)
    ap.add_argument("--er-log2", type=int, default=22)
    ap.add_argument("--er-d", type=int, default=64)
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    import oracle_bind as ob
    from paper_2504_06408_b200 import Context, generators
    from paper_2504_06408_b200.generators import coo_to_csr_fast
    from paper_2504_06408_b200.summa import (HYBRID, Comm, block_from_piece, block_range, checksum_part,
                                             checksum_seed, grid_for, local_block, measured_threshold,
                                             summa25_multiply)

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=3000))
    job = [uuid.uuid4().hex[:12] if rank == 0 else None]
    dist.broadcast_object_list(job, src=0)
    c = args.config
    seed = 1

    def full_coo():
        if c in (2, 3):
            scale = args.scale or (18 if c == 2 else 22)
            m = generators.generate_rmat(4 if c == 2 else 2, scale, 16.0, seed)
            return generators.permute_symmetric(m, seed)
        if c == 4:
            return generators.generate_stencil27(0, args.stencil_n)
        return generators.generate_er(5, 1 << args.er_log2, args.er_d, seed, value_mode=1)

    if c == 4:
        pr, pc = 1, world
    else:
        pr, pc = grid_for(world)
    i, j = rank // pc, rank % pc
    if c in (2, 3):
        m = full_coo()
        n = m.nrows
        blk = local_block(m, pr, pc, i, j)
        del m
    elif c == 4:
        n = args.stencil_n ** 3
        rr, cr = block_range(n, pr, i), block_range(n, pc, j)
        blk = block_from_piece(generators.generate_stencil27_block(0, args.stencil_n, rr, cr), rr, cr)
    else:
        n = 1 << args.er_log2
        rr, cr = block_range(n, pr, i), block_range(n, pc, j)
        blk = block_from_piece(generators.generate_er_block(5, n, args.er_d, seed, rr, cr, value_mode=1), rr, cr)
    ctx = Context(local)
    comm = Comm(job[0], world, rank, pr, pc, local, staging_bytes=64 << 20)
    t0 = time.time()
    cm, led = summa25_multiply(comm, ctx, blk, blk, n, n, n, two_round=True, mode=HYBRID,
                               threshold=measured_threshold(pc), threshold_col=measured_threshold(pr))
    t_gpu = time.time() - t0
    part = checksum_part(cm, blk.rows[0], blk.cols[0])
    t = torch.tensor([part & 0xFFFFFFFF, part >> 32, cm.nnz, led["products"]], dtype=torch.int64)
    cm.free()
    parts = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    if rank == 0:
        got = checksum_seed(n, n)
        for p in parts:
            got = (got + int(p[0]) + (int(p[1]) << 32)) % (1 << 64)
        nnz = sum(int(p[2]) for p in parts)
        prods = sum(int(p[3]) for p in parts)
        t1 = time.time()
        a = coo_to_csr_fast(full_coo())
        am = ob.Mat.of(a)
        s, z, f, _ = ob.orc_stream(am, am, nthreads=os.cpu_count() or 1)
        want = (ob.orc_seed(n, n) + s) % (1 << 64)
        res = {"config": c, "grid": f"{pr}x{pc}", "n": n, "products": prods, "oracle_products": f, "nnz_C": nnz,
               "oracle_nnz_C": z, "checksum_C": got, "oracle_checksum_C": want,
               "match": got == want and nnz == z and prods == f, "gpu_call_s": round(t_gpu, 2),
               "oracle_s": round(time.time() - t1, 1), "oracle_threads": os.cpu_count()}
        print("[fullsize] " + json.dumps(res), flush=True)
        if not res["match"]:
            sys.exit(1)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
