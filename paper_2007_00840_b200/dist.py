"""Multi-GPU layer: one process per GPU (torch.distributed), graph replicated,
source rows split into contiguous work-balanced ranges.

Rows are independent given the static G(A); only supernode detection
couples consecutive rows.  Ranges are row-granular (equal shares
of an elimination-tree work estimate, P:264, P:454-459 -- aligning them to
chunk_size would cost balance: the heavy top-separator rows are few).  A range
that starts inside a chunk has provisional head supernodes, so the ranks run
the supernode-boundary exchange: a chain r -> r+1 of 24-byte tail records
{last row, its nnz(U), leader of its block}; each rank re-runs Def. def:T3
over its head rows with the incoming tail (gsofa_supernode_stitch, a CUDA
kernel) and forwards its own tail.  Then one allgather of per-rank counts
(nnz_L, nnz_U, fill, nsuper, nnz_A_offdiag) gives every rank the global CSR
offsets of its slice.  Both are tiny messages over NCCL (NVLink/NVSwitch on a
B200 box); nothing else crosses GPUs.

Row interleave (the paper's source scheduling,
P:632-647): instead of contiguous ranges, units of U rows are dealt
round-robin to the ranks (symbolic_interleaved).  With U a multiple of
chunk_size every unit starts a chunk, supernodes are unit-local and no
exchange is needed; with a finer U each rank exports 4 + 4 W bytes per row
(nnz(U(s,:)) and the candidate-leader L mask, gsofa_result_rowinfo), one
all_gather over NCCL moves them, and every rank runs the per-chunk Def. T3
scan over the gathered rows (gsofa_supernodes_gathered) -- the B200 analogue
of the paper's unified-memory remote reads.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

COUNT_FIELDS = ("nnz_L", "nnz_U", "fill_count", "nsuper", "nnz_A_offdiag", "rows")


@dataclass
class RankSlice:
    rank: int
    world: int
    row_begin: int
    row_end: int
    counts: np.ndarray        # [world, len(COUNT_FIELDS)] int64, all ranks
    L_base: int               # global offset of this slice in L_colidx
    U_base: int               # global offset of this slice in U_colidx
    sn_base: int              # global index of this slice's first supernode
    result: object = None     # local Result (None if the range is empty)

    @property
    def totals(self):
        t = self.counts.sum(axis=0)
        return dict(zip(COUNT_FIELDS, (int(x) for x in t)))


def partition(rowptr, colidx, world: int, align: int = 1, partition_fn=None):
    """Contiguous row ranges, one per rank (row-granular unless align > 1)."""
    if partition_fn is None:
        from . import partition_rows as partition_fn
    return partition_fn(rowptr, colidx, world, align)


def global_offsets(counts: np.ndarray, rank: int):
    """Exclusive prefix over ranks of the gathered counts -> (L_base, U_base, sn_base)."""
    before = counts[:rank].sum(axis=0) if rank else np.zeros(counts.shape[1], np.int64)
    return int(before[0]), int(before[1]), int(before[3])


def allgather_counts(local: np.ndarray, group=None, device=None) -> np.ndarray:
    """all_gather of a small int64 vector (NCCL on GPU tensors, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.as_tensor(local, dtype=torch.int64)
    if device is not None:
        t = t.to(device)
    out = torch.empty(world * t.numel(), dtype=torch.int64, device=t.device)
    dist.all_gather_into_tensor(out, t, group=group)
    return out.cpu().numpy().reshape(world, -1)


NO_TAIL = (-1, -1, -1)


def exchange_tail(tail, rank: int, world: int, recv: bool, group=None, device=None):
    """One hop of the supernode-boundary chain: receive the predecessor's tail
    (recv=True, from rank-1) or send ours to rank+1.  A tail is (row, nnzU,
    leader); NO_TAIL stands for "none" (rank 0, or empty ranges before)."""
    import torch
    import torch.distributed as dist
    if recv:
        t = torch.empty(3, dtype=torch.int64, device=device)
        dist.recv(t, src=rank - 1, group=group)
        v = tuple(int(x) for x in t.cpu().tolist())
        return None if v == NO_TAIL else v
    t = torch.tensor(NO_TAIL if tail is None else tail, dtype=torch.int64, device=device)
    dist.send(t, dst=rank + 1, group=group)
    return None


def _stitch_gpu(res, prev):
    return res.stitch(prev).as_tuple()


def symbolic_distributed(rowptr, colidx, bounds, *, rank: int, compute_fn=None, stitch_fn=None,
                         group=None, device=None, **kw) -> RankSlice:
    """Run this rank's row range, stitch supernodes with the neighbours and
    exchange counts.

    compute_fn(rowptr, colidx, row_begin=..., row_end=..., **kw) -> object with
    nnz_L, nnz_U, fill_count, nsuper, nnz_A_offdiag (default: the CUDA
    library's :func:`symbolic`); stitch_fn(result, prev_tail) -> tail fixes the
    head supernodes in place (default: gsofa_supernode_stitch).  Tests inject
    the CPU oracle and a plain Def. def:T3 scan here to check the host logic
    with the gloo backend; the product path always uses the GPU library.
    """
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if compute_fn is None:
        from . import symbolic as compute_fn
    if stitch_fn is None:
        stitch_fn = _stitch_gpu
    rb, re = int(bounds[rank]), int(bounds[rank + 1])
    res = None
    local = np.zeros(len(COUNT_FIELDS), np.int64)
    if re > rb:
        res = compute_fn(rowptr, colidx, row_begin=rb, row_end=re, **kw)
    # supernode-boundary exchange: chain rank-1 -> rank -> rank+1
    prev = exchange_tail(None, rank, world, True, group, device) if rank > 0 else None
    tail = stitch_fn(res, prev) if res is not None else prev
    if rank + 1 < world:
        exchange_tail(tail, rank, world, False, group, device)
    if res is not None:
        local[:] = [res.nnz_L, res.nnz_U, res.fill_count, res.nsuper, res.nnz_A_offdiag, re - rb]
    counts = allgather_counts(local, group=group, device=device)
    assert counts.shape == (world, len(COUNT_FIELDS))
    L_base, U_base, sn_base = global_offsets(counts, rank)
    return RankSlice(rank, world, rb, re, counts, L_base, U_base, sn_base, res)


def assemble(slices_arrays, n: int):
    """Concatenate per-rank host arrays into the global result (verification
    helper; not on the timed path).  slices_arrays: list over ranks of dicts
    with L_rowptr, L_colidx, U_rowptr, U_colidx, sn_start (local, row-range
    based) -- empty ranges may be None."""
    Lp, Li, Up, Ui, sn = [np.zeros(1, np.int64)], [], [np.zeros(1, np.int64)], [], []
    lb = ub = 0
    for a in slices_arrays:
        if a is None:
            continue
        Lp.append(a["L_rowptr"][1:] + lb)
        Up.append(a["U_rowptr"][1:] + ub)
        Li.append(a["L_colidx"])
        Ui.append(a["U_colidx"])
        sn.append(a["sn_start"][:-1])
        lb += int(a["L_rowptr"][-1])
        ub += int(a["U_rowptr"][-1])
    sn.append(np.array([n], np.int32))
    return dict(L_rowptr=np.concatenate(Lp), L_colidx=np.concatenate(Li).astype(np.int32),
                U_rowptr=np.concatenate(Up), U_colidx=np.concatenate(Ui).astype(np.int32),
                sn_start=np.concatenate(sn).astype(np.int32))


# ------------------------------------------------------------ row interleave

def interleave_rows(row_begin: int, row_end: int, nparts: int, part: int, unit_rows: int) -> np.ndarray:
    """Global rows of `part` under the round-robin unit deal (ascending)."""
    u = np.arange(part, (row_end - row_begin + unit_rows - 1) // unit_rows, nparts, dtype=np.int64)
    rows = (row_begin + u[:, None] * unit_rows + np.arange(unit_rows, dtype=np.int64)[None, :]).ravel()
    return rows[rows < row_end]


def _rowinfo_gpu(res):
    return res.rowinfo()


def _gathered_gpu(res, nnzU_all, mask_all, stride):
    res.supernodes_gathered(nnzU_all, mask_all, stride)


def symbolic_interleaved(rowptr, colidx, *, rank: int, unit_rows: int = 128, chunk_size: int = 128,
                         row_begin: int = 0, row_end: int | None = None, compute_fn=None,
                         rowinfo_fn=None, gathered_fn=None, group=None, device=None, **kw):
    """This rank's units of rows (round-robin deal of unit_rows-row units,
    SURVEY §8(f) NEXT-2); supernodes completed by the rowinfo all_gather when
    unit_rows is not a multiple of chunk_size; then the count allgather.

    compute_fn(rowptr, colidx, interleave=(N, q, U), chunk_size=..., ...) ->
    result with rows/nsuper/counts; rowinfo_fn(result) -> (nnzU [rows],
    mask [rows, W]) tensors; gathered_fn(result, nnzU_all, mask_all, stride)
    completes its supernodes.  Defaults: the CUDA library; tests inject CPU
    versions to check the host logic on gloo.  Returns (result, counts)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = (rowptr.size if isinstance(rowptr, np.ndarray) else rowptr.numel()) - 1
    row_end = n if row_end is None else row_end
    if compute_fn is None:
        from . import symbolic as compute_fn
    rowinfo_fn = rowinfo_fn or _rowinfo_gpu
    gathered_fn = gathered_fn or _gathered_gpu
    res = compute_fn(rowptr, colidx, interleave=(world, rank, unit_rows), chunk_size=chunk_size,
                     row_begin=row_begin, row_end=row_end, **kw)
    if res.nsuper < 0:
        # Def. def:T3 data of every row, part-major, padded to the largest part
        stride = max(interleave_rows(row_begin, row_end, world, p, unit_rows).size for p in range(world))
        nnzU, mask = rowinfo_fn(res)
        W = mask.shape[1]
        pad_n = torch.zeros(stride, dtype=torch.int32, device=nnzU.device)
        pad_m = torch.zeros((stride, W), dtype=torch.int32, device=mask.device)
        pad_n[: nnzU.numel()] = nnzU
        pad_m[: mask.shape[0]] = mask
        # NCCL gathers device tensors in place; gloo (tests, shared-GPU
        # smoke runs) goes through host memory
        cdev = pad_n.device if dist.get_backend(group) != "gloo" else torch.device("cpu")
        all_n = torch.empty(world * stride, dtype=torch.int32, device=cdev)
        all_m = torch.empty((world * stride, W), dtype=torch.int32, device=cdev)
        dist.all_gather_into_tensor(all_n, pad_n.to(cdev), group=group)
        dist.all_gather_into_tensor(all_m, pad_m.to(cdev), group=group)
        gathered_fn(res, all_n.to(nnzU.device), all_m.to(mask.device), stride)
    local = np.array([res.nnz_L, res.nnz_U, res.fill_count, res.nsuper, res.nnz_A_offdiag, res.rows],
                     np.int64)
    counts = allgather_counts(local, group=group, device=device)
    return res, counts


def assemble_interleaved(parts, row_begin: int, row_end: int, unit_rows: int, n: int):
    """Global CSR + supernodes from the parts' host arrays (verification
    helper): rows dealt back in order, sn_start = union of the parts'
    leaders."""
    N = len(parts)
    rows_of = [interleave_rows(row_begin, row_end, N, q, unit_rows) for q in range(N)]
    m = row_end - row_begin
    nL = np.zeros(m, np.int64)
    nU = np.zeros(m, np.int64)
    for q, a in enumerate(parts):
        nL[rows_of[q] - row_begin] = np.diff(a["L_rowptr"])
        nU[rows_of[q] - row_begin] = np.diff(a["U_rowptr"])
    Lp = np.concatenate([[0], np.cumsum(nL)]).astype(np.int64)
    Up = np.concatenate([[0], np.cumsum(nU)]).astype(np.int64)
    Li = np.empty(int(Lp[-1]), np.int32)
    Ui = np.empty(int(Up[-1]), np.int32)
    for q, a in enumerate(parts):
        for k, s in enumerate(rows_of[q] - row_begin):
            Li[Lp[s]:Lp[s + 1]] = a["L_colidx"][a["L_rowptr"][k]:a["L_rowptr"][k + 1]]
            Ui[Up[s]:Up[s + 1]] = a["U_colidx"][a["U_rowptr"][k]:a["U_rowptr"][k + 1]]
    sn = np.sort(np.concatenate([a["sn_start"][:-1] for a in parts] + [np.array([row_end])]))
    return dict(L_rowptr=Lp, L_colidx=Li, U_rowptr=Up, U_colidx=Ui, sn_start=sn.astype(np.int32))


# ---------------------------------------------------- dynamic block stealing
# SURVEY §8(f) NEXT-2, the third variant: instead of a fixed assignment, the
# ranks claim chunk-aligned row blocks (equal estimated work, heaviest --
# highest rows -- first) from one shared atomic counter until none is left.
# Blocks start at multiples of chunk_size, so their supernodes are complete
# and nothing is stitched; one all_gather of per-block counts gives
# every rank the global CSR offsets.  The counter here is the process group's
# store (an atomic add over TCP); a device-side counter in one GPU's memory
# mapped by its peers (CUDA IPC over NVLink) would make a claim ~10 us instead
# of ~50-100 us -- at a few dozen claims per call either is noise.

def steal_blocks(rowptr, colidx, nblocks: int, chunk_size: int = 128, partition_fn=None):
    """Chunk-aligned blocks of equal estimated work, in claim order
    (descending rows): list of (row_begin, row_end)."""
    b = partition(rowptr, colidx, nblocks, align=chunk_size, partition_fn=partition_fn)
    blocks = [(int(b[i]), int(b[i + 1])) for i in range(len(b) - 1) if b[i + 1] > b[i]]
    return blocks[::-1]


def symbolic_stealing(rowptr, colidx, *, rank: int, blocks_per_rank: int = 4, chunk_size: int = 128,
                      compute_fn=None, store=None, key: str = "gsofa_steal", group=None, device=None,
                      **kw):
    """Claim blocks from the shared counter until they run out; returns
    (list of (block index, row_begin, row_end, result), counts [nblocks, 6]
    gathered from all ranks: each block's counts come from the rank that
    computed it)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if compute_fn is None:
        from . import symbolic as compute_fn
    if store is None:
        from torch.distributed import distributed_c10d as c10d
        store = c10d._get_default_store()
    blocks = steal_blocks(rowptr, colidx, world * blocks_per_rank, chunk_size)
    dist.barrier(group=group)
    mine = []
    local = np.zeros((len(blocks), len(COUNT_FIELDS)), np.int64)
    while True:
        k = int(store.add(key, 1)) - 1  # atomic fetch-and-add: this rank's next block
        if k >= len(blocks):
            break
        rb, re = blocks[k]
        res = compute_fn(rowptr, colidx, row_begin=rb, row_end=re, chunk_size=chunk_size, **kw)
        local[k] = [res.nnz_L, res.nnz_U, res.fill_count, res.nsuper, res.nnz_A_offdiag, re - rb]
        mine.append((k, rb, re, res))
    # every block was computed by exactly one rank: the element-wise sum over
    # ranks is the full table
    counts = allgather_counts(local.ravel(), group=group, device=device)
    counts = counts.reshape(world, len(blocks), len(COUNT_FIELDS)).sum(axis=0)
    dist.barrier(group=group)
    if rank == 0:
        store.add(key, -int(store.add(key, 0)))  # reset for the next call
    dist.barrier(group=group)
    return mine, counts, blocks
