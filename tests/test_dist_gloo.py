"""Host logic of the multi-GPU layer on CPU: world_size 2 (and 3) with the gloo
backend.  The per-rank compute is the CPU oracle injected through
``compute_fn`` (the product path always calls the CUDA library); what is under
test is the partition, the count allgather, the global offsets and the
assembly, which must reproduce the single-process result exactly."""
import os
import socket
import types

import numpy as np
import pytest
import torch.multiprocessing as mp

import gen
import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_compute(rowptr, colidx, row_begin, row_end, chunk_size=128):
    r = oracle.symbolic(rowptr, colidx, chunk_size=chunk_size, row_begin=row_begin,
                        row_end=row_end, nthreads=1)
    ns = types.SimpleNamespace(**{k: r[k] for k in ("nnz_L", "nnz_U", "fill_count", "nsuper",
                                                     "nnz_A_offdiag")})
    ns.arrays = {k: r[k] for k in ("L_rowptr", "L_colidx", "U_rowptr", "U_colidx", "sn_start")}
    return ns


def _worker(rank, world, port, name, scale, chunk, q):
    import torch.distributed as dist

    import paper_2007_00840_b200 as g
    from paper_2007_00840_b200 import dist as gd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rp, ci = gen.config(name, scale)
        bounds = gd.partition(rp, ci, world, chunk, partition_fn=g.partition_rows)
        sl = gd.symbolic_distributed(rp, ci, bounds, rank=rank, compute_fn=_oracle_compute,
                                     chunk_size=chunk)
        q.put((rank, bounds.tolist(), sl.row_begin, sl.row_end, sl.counts.tolist(), sl.L_base,
               sl.U_base, sl.sn_base, sl.result.arrays if sl.result is not None else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name,scale,chunk", [(2, "C5", 12, 128), (3, "C4", 40, 64),
                                                    (2, "C1", None, 128)])
def test_distributed_host_logic_gloo(world, name, scale, chunk):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, scale, chunk, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort(key=lambda t: t[0])
    rp, ci = gen.config(name, scale)
    n = rp.size - 1
    full = oracle.symbolic(rp, ci, chunk_size=chunk)
    bounds = outs[0][1]
    assert all(o[1] == bounds for o in outs)            # identical partition on every rank
    assert bounds[0] == 0 and bounds[-1] == n
    assert all(b % chunk == 0 for b in bounds[:-1])
    counts = np.array(outs[0][4])
    assert all(np.array_equal(np.array(o[4]), counts) for o in outs)
    tot = counts.sum(axis=0)
    assert tot[0] == full["nnz_L"] and tot[1] == full["nnz_U"]
    assert tot[2] == full["fill_count"] and tot[3] == full["nsuper"]
    # each rank's global offsets point at its slice of the single-process CSR
    for o in outs:
        rank, _, rb, re, _, Lb, Ub, snb, arr = o
        assert Lb == full["L_rowptr"][rb] and Ub == full["U_rowptr"][rb]
        if arr is not None:
            assert np.array_equal(arr["L_colidx"], full["L_colidx"][full["L_rowptr"][rb]:full["L_rowptr"][re]])
            assert full["sn_start"][snb] == rb
    from paper_2007_00840_b200 import dist as gd
    asm = gd.assemble([o[8] for o in outs], n)
    for k in ("L_rowptr", "L_colidx", "U_rowptr", "U_colidx", "sn_start"):
        assert np.array_equal(asm[k], full[k]), k
