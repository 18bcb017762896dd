"""CPU (no GPU): the shared-memory fabric under real multi-process ranks
(gloo rendezvous, world size 2 and 4): barriers, exchange_sizes over row and
column scopes, host-path broadcasts (chunked through the staging ring),
protocol errors and peer-abort propagation (fabric.hpp:141-149, :287-290)."""
import os
import uuid

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, pr, pc, job, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_06408_b200 import errors
        from paper_2504_06408_b200.summa import Comm
        comm = Comm(job, world, rank, pr, pc, device=-1, staging_bytes=16384)
        i, j = rank // pc, rank % pc
        comm.barrier()
        # exchange_sizes: root of row scope i is column (i % pc); of column scope j is row (j % pr)
        t = comm.exchange_sizes(0, i % pc, (100 + i, 7, 3) if j == i % pc else (0, 0, 0))
        assert t == (100 + i, 7, 3), t
        t = comm.exchange_sizes(1, j % pr, (200 + j, 1, 2) if i == j % pr else (0, 0, 0))
        assert t == (200 + j, 1, 2), t
        # host-path broadcasts of host buffers: small and multi-chunk
        for nbytes in (1, 1000, 16384, 100003):
            buf = np.zeros(nbytes, dtype=np.uint8)
            root = (nbytes % pc)
            if j == root:
                buf[:] = (np.arange(nbytes) * (i + 3)) % 251
            path = comm.bcast(0, root, buf.ctypes.data, nbytes, mode=2, threshold=1 << 40)
            assert path == 0
            assert np.array_equal(buf, (np.arange(nbytes) * (i + 3)) % 251)
        comm.barrier()  # every rank is done broadcasting before rank 0 raises the abort below
        # a root outside the scope is a ProtocolError on the offending rank
        if world > 1:
            if rank == 0:
                with pytest.raises(errors.ProtocolError):
                    comm.exchange_sizes(0, 99, (0, 0, 0))
            else:
                # rank 0's failure tears the peers down instead of deadlocking them
                with pytest.raises(errors.AbortedError):
                    comm.barrier()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported through the queue
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,pr,pc", [(2, 1, 2), (4, 2, 2), (8, 2, 4)])
def test_fabric_multiprocess(world, pr, pc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    job = "t" + uuid.uuid4().hex[:10]
    port = 29500 + (os.getpid() % 1000) + world
    procs = [ctx.Process(target=_worker, args=(r, world, pr, pc, job, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
