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
    ns.row_begin, ns.row_end = row_begin, row_end
    return ns


def _oracle_stitch(res, prev, chunk=128):
    """Plain Def. def:T3 scan of the head rows of a range whose
    first block was computed as if row_begin started one: test-side stand-in
    for gsofa_supernode_stitch on oracle results.  Returns the range's tail."""
    a = res.arrays
    rb, re = res.row_begin, res.row_end
    Lp, Li, Up = a["L_rowptr"], a["L_colidx"], a["U_rowptr"]
    sn = [int(x) for x in a["sn_start"]]
    if prev is not None and rb % chunk:
        he = min(re, (rb // chunk + 1) * chunk)
        r, pn, new = prev[2], prev[1], []
        for s in range(rb, he):
            k = s - rb
            nu = int(Up[k + 1] - Up[k])
            if not (nu == pn - 1 and r in set(Li[Lp[k]:Lp[k + 1]].tolist())):
                r = s
                new.append(s)
            pn = nu
        old = sum(1 for x in sn[:-1] if x < he)
        sn = new + sn[old:]
        a["sn_start"] = np.array(sn, np.int32)
        res.nsuper = len(sn) - 1
    leader = sn[-2] if len(sn) > 1 else prev[2]
    return (re - 1, int(Up[-1] - Up[-2]), leader)


def _worker(rank, world, port, name, scale, chunk, q, fixed_bounds=None):
    import torch.distributed as dist

    import paper_2007_00840_b200 as g
    from paper_2007_00840_b200 import dist as gd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rp, ci = gen.config(name, scale)
        bounds = (np.array(fixed_bounds, np.int64) if fixed_bounds is not None
                  else gd.partition(rp, ci, world, partition_fn=g.partition_rows))
        sl = gd.symbolic_distributed(rp, ci, bounds, rank=rank, compute_fn=_oracle_compute,
                                     stitch_fn=lambda r, p: _oracle_stitch(r, p, chunk),
                                     chunk_size=chunk)
        q.put((rank, bounds.tolist(), sl.row_begin, sl.row_end, sl.counts.tolist(), sl.L_base,
               sl.U_base, sl.sn_base, sl.result.arrays if sl.result is not None else None))
    finally:
        dist.destroy_process_group()


def _inside_supernodes(name, scale, chunk, world):
    """Range starts strictly inside multi-row supernodes (not at chunk
    multiples): every boundary must be stitched."""
    rp, ci = gen.config(name, scale)
    sn = oracle.symbolic(rp, ci, chunk_size=chunk)["sn_start"]
    cand = [int(a) + 1 for a, b in zip(sn[:-1], sn[1:]) if b - a >= 3 and (a + 1) % chunk]
    pick = [cand[(i + 1) * len(cand) // world] for i in range(world - 1)]
    return [0] + sorted(pick) + [rp.size - 1]


@pytest.mark.parametrize("world,name,scale,chunk,inside", [
    (2, "C5", 12, 128, False), (3, "C4", 40, 64, False), (2, "C1", None, 128, False),
    (3, "C3", 1500, 128, True), (2, "C2", 10, 16, True)])
def test_distributed_host_logic_gloo(world, name, scale, chunk, inside):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    fb = _inside_supernodes(name, scale, chunk, world) if inside else None
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, scale, chunk, q, fb))
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
    if inside:
        assert all(b % chunk for b in bounds[1:-1])  # every boundary needs the stitch
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
            lead = full["sn_start"][(full["sn_start"] >= rb) & (full["sn_start"] < re)]
            assert np.array_equal(arr["sn_start"][:-1], lead)          # stitched supernodes
            assert snb == int((full["sn_start"][:-1] < rb).sum())
    from paper_2007_00840_b200 import dist as gd
    asm = gd.assemble([o[8] for o in outs], n)
    for k in ("L_rowptr", "L_colidx", "U_rowptr", "U_colidx", "sn_start"):
        assert np.array_equal(asm[k], full[k]), k


@pytest.mark.parametrize("name,scale,chunk", [("C1", None, 128), ("C3", 1500, 128), ("C2", 10, 16),
                                              ("C4", 40, 64)])
def test_stitch_chain_oracle(name, scale, chunk):
    """Many ranges, cut everywhere (inside supernodes, at chunk multiples, one
    row long): per-range oracle results stitched in order reproduce the
    whole-matrix supernodes (the reading of Def. def:T3 the GPU stitch uses)."""
    rp, ci = gen.config(name, scale)
    n = rp.size - 1
    full = oracle.symbolic(rp, ci, chunk_size=chunk)
    rng = np.random.default_rng(7)
    cuts = sorted(set(rng.integers(1, n, 12).tolist()) | {chunk, chunk + 1, chunk + 2, n // 2, n // 2 + 1})
    bounds = [0] + [c for c in cuts if 0 < c < n] + [n]
    prev, parts = None, []
    for rb, re in zip(bounds[:-1], bounds[1:]):
        res = _oracle_compute(rp, ci, rb, re, chunk)
        res.row_begin, res.row_end = rb, re
        prev = _oracle_stitch(res, prev, chunk)
        parts.append(res.arrays)
    from paper_2007_00840_b200 import dist as gd
    asm = gd.assemble(parts, n)
    assert np.array_equal(asm["sn_start"], full["sn_start"])


# ------------------------------------------------------------ row interleave
# dist.symbolic_interleaved: round-robin units of rows,
# and for finer-than-chunk units the all_gather of per-row Def. def:T3 data.
# Compute, rowinfo and the per-chunk scan are injected CPU stand-ins (the
# product path calls the CUDA library); under test are the deal, the padding
# and part-major layout of the gathered rows, and the count allgather.

def _il_compute(rowptr, colidx, interleave, chunk_size, row_begin, row_end):
    from paper_2007_00840_b200 import dist as gd
    N, q, U = interleave
    rows = gd.interleave_rows(row_begin, row_end, N, q, U)
    r = oracle.rows(rowptr, colidx, rows, 1)
    ns = types.SimpleNamespace(rows=rows.size, glob=rows, chunk=chunk_size, il=interleave)
    ns.arrays = {k: r[k] for k in ("L_rowptr", "L_colidx", "U_rowptr", "U_colidx")}
    ns.nnz_L, ns.nnz_U = int(r["L_rowptr"][-1]), int(r["U_rowptr"][-1])
    offd = sum(int(np.count_nonzero(colidx[rowptr[s]:rowptr[s + 1]] != s)) for s in rows)
    ns.nnz_A_offdiag = offd
    ns.fill_count = ns.nnz_L + ns.nnz_U - rows.size - offd
    if U % chunk_size == 0:  # unit-local supernodes: the oracle scan per unit
        lead = []
        for u0 in range(0, rows.size, U):
            sl = slice(u0, min(rows.size, u0 + U))
            Lp = r["L_rowptr"][sl.start:sl.stop + 1] - r["L_rowptr"][sl.start]
            Up = r["U_rowptr"][sl.start:sl.stop + 1] - r["U_rowptr"][sl.start]
            Li = r["L_colidx"][r["L_rowptr"][sl.start]:r["L_rowptr"][sl.stop]]
            lead += oracle.supernodes(int(rows[u0]), Lp, Li, Up, chunk_size)[:-1].tolist()
        ns.arrays["sn_start"] = np.array(lead + [int(rows[-1]) + 1], np.int32)
        ns.nsuper = len(lead)
    else:
        ns.nsuper = -1
    return ns


def _il_rowinfo(res):
    import torch
    a, W = res.arrays, (res.chunk + 31) // 32
    nnzU = torch.tensor(np.diff(a["U_rowptr"]), dtype=torch.int32)
    mask = np.zeros((res.rows, W), np.uint32)
    for k, s in enumerate(res.glob):
        for c in a["L_colidx"][a["L_rowptr"][k]:a["L_rowptr"][k + 1]]:
            d = int(s - c)
            if d <= s % res.chunk:
                mask[k, d // 32] |= np.uint32(1 << (d % 32))
    return nnzU, torch.tensor(mask.view(np.int32))


def _il_gathered(res, all_n, all_m, stride):
    """Per chunk, the greedy Def. def:T3 scan over the gathered rows; this
    part keeps its own leaders."""
    N, q, U = res.il
    nn, mm = all_n.numpy(), all_m.numpy().view(np.uint32)
    end = int(res.glob[-1]) + 1
    n_rows = max(end, 0)
    mine, lead = set(res.glob.tolist()), []

    def at(s):
        u = s // U
        return (u % N) * stride + (u // N) * U + s % U

    total_rows = res.total_rows
    for cs in range(0, total_rows, res.chunk):
        r, pn = cs, 0
        for s in range(cs, min(total_rows, cs + res.chunk)):
            i = at(s)
            nu, d = int(nn[i]), s - r
            join = s != cs and nu == pn - 1 and (int(mm[i, d // 32]) >> (d % 32)) & 1
            if not join:
                r = s
                if s in mine:
                    lead.append(s)
            pn = nu
    res.arrays["sn_start"] = np.array(lead + [n_rows], np.int32)
    res.nsuper = len(lead)


def _il_worker(rank, world, port, name, scale, chunk, U, q):
    import torch.distributed as dist

    from paper_2007_00840_b200 import dist as gd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rp, ci = gen.config(name, scale)

        def compute(rowptr, colidx, **kw):
            r = _il_compute(rowptr, colidx, **kw)
            r.total_rows = rowptr.size - 1
            return r
        res, counts = gd.symbolic_interleaved(rp, ci, rank=rank, unit_rows=U, chunk_size=chunk,
                                              compute_fn=compute, rowinfo_fn=_il_rowinfo,
                                              gathered_fn=_il_gathered)
        q.put((rank, counts.tolist(), res.arrays))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name,scale,chunk,U", [
    (2, "C1", None, 128, 32), (3, "C2", 10, 64, 96), (2, "C3", 1500, 128, 256), (3, "C4", 40, 64, 64)])
def test_interleave_host_logic_gloo(world, name, scale, chunk, U):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_il_worker, args=(r, world, port, name, scale, chunk, U, q))
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
    counts = np.array(outs[0][1])
    assert all(np.array_equal(np.array(o[1]), counts) for o in outs)
    tot = counts.sum(axis=0)
    assert tot[0] == full["nnz_L"] and tot[1] == full["nnz_U"] and tot[2] == full["fill_count"]
    assert tot[3] == full["nsuper"] and tot[5] == n
    from paper_2007_00840_b200 import dist as gd
    asm = gd.assemble_interleaved([o[2] for o in outs], 0, n, U, n)
    for k in ("L_rowptr", "L_colidx", "U_rowptr", "U_colidx", "sn_start"):
        assert np.array_equal(asm[k], full[k]), k


# ---------------------------------------------------- dynamic block stealing

def _steal_worker(rank, world, port, name, scale, chunk, q):
    import torch.distributed as dist

    from paper_2007_00840_b200 import dist as gd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rp, ci = gen.config(name, scale)

        def compute(rowptr, colidx, row_begin, row_end, chunk_size):
            return _oracle_compute(rowptr, colidx, row_begin, row_end, chunk_size)
        import paper_2007_00840_b200 as g
        for rep in range(2):  # the counter is reset between calls
            mine, counts, blocks = gd.symbolic_stealing(rp, ci, rank=rank, chunk_size=chunk,
                                                        compute_fn=compute)
        q.put((rank, [(k, rb, re, r.arrays) for k, rb, re, r in mine], counts.tolist(), blocks))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name,scale,chunk", [(2, "C2", 10, 16), (3, "C4", 40, 64), (2, "C3", 1500, 128)])
def test_stealing_host_logic_gloo(world, name, scale, chunk):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_steal_worker, args=(r, world, port, name, scale, chunk, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rp, ci = gen.config(name, scale)
    n = rp.size - 1
    full = oracle.symbolic(rp, ci, chunk_size=chunk)
    blocks = outs[0][3]
    assert all(o[3] == blocks for o in outs)
    assert all(rb % chunk == 0 for rb, _ in blocks) and sorted(blocks)[0][0] == 0
    got = {}
    for o in outs:
        for k, rb, re, arr in o[1]:
            assert k not in got  # claimed exactly once
            got[k] = (rb, re, arr)
    assert sorted(got) == list(range(len(blocks)))
    counts = np.array(outs[0][2])
    assert counts[:, 2].sum() == full["fill_count"] and counts[:, 3].sum() == full["nsuper"]
    from paper_2007_00840_b200 import dist as gd
    parts = [got[k][2] for k in sorted(got, key=lambda k: got[k][0])]
    asm = gd.assemble(parts, n)
    for key in ("L_rowptr", "L_colidx", "U_rowptr", "U_colidx", "sn_start"):
        assert np.array_equal(asm[key], full[key]), key
