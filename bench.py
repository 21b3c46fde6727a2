#!/usr/bin/env python
"""Benchmark of the gSoFa symbolic-factorization hot path on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

A step = one full symbolic factorization (seed -> traversal -> extraction ->
supernodes, plus for N > 1 the NCCL count allgather) of the synthetic
BASELINE config (default C5 = configs[4], 3D 7-point 128^3, ND order: the
largest matrix, on which north_star's 1/2/4/8-GPU strong scaling is quoted).
``--gpus N`` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one GPU each, NCCL).
value = fill-ins found per second over the whole job (max over ranks of the
device time); e2e = the same through the public API with host (pinned)
buffers, uploads and result downloads inside the timed region.

Rank 0 prints ONE JSON line on stdout; diagnostics go to stderr.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gen  # noqa: E402

METRIC = "symbolic-factorization fill-ins/s"
UNIT = "fill-ins/s"
CONFIG_DESC = {
    "C1": "C1: 2D 5-point 32x32, natural order, p=0.25 dropout (n=1,024)",
    "C2": "C2: 3D 7-point 64^3, nested-dissection order, p=0.25 dropout (n=262,144)",
    "C3": "C3: BBMAT-shaped banded+scatter (n=38,744, nnz=1.77M), natural order",
    "C4": "C4: G3_circuit-shaped ND mesh + hubs (n=1,585,478, nnz=7.66M)",
    "C5": "C5: 3D 7-point 128^3, nested-dissection order, p=0.25 dropout (n=2,097,152)",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def fills_of_rows(rp, ci, r):
    """Per-sample fill-in count from oracle rows (for the CPU baselines)."""
    rows = r["rows"]
    deg = rp[rows + 1] - rp[rows]
    # off-diagonal A entries in those rows
    offd = 0
    for s in rows:
        seg = ci[rp[s]:rp[s + 1]]
        offd += int(np.count_nonzero(seg != s))
    return int(r["L_rowptr"][-1] + r["U_rowptr"][-1] - rows.size - offd), int(deg.sum())


def cpu_oracle_sample(rp, ci, target_s: float, seed: int = 0):
    """Run the (untuned) oracle on every k-th row of the workload, halving k
    until one run takes at least ~target_s/2 seconds on this host (or all rows
    are covered).  Returns (fill-ins/s, description, threads, seconds)."""
    import oracle
    n = rp.size - 1
    threads = oracle.default_threads()
    stride = max(1, n // 256)
    while True:
        rows = np.arange(stride // 2, n, stride, dtype=np.int64)
        t = time.perf_counter()
        r = oracle.rows(rp, ci, rows, threads)
        dt = time.perf_counter() - t
        if dt >= target_s / 2 or stride == 1:
            break
        stride = max(1, int(stride / max(2.0, min(16.0, target_s / 2 / max(dt, 1e-3)))))
    r["rows"] = rows
    fills, _ = fills_of_rows(rp, ci, r)
    desc = (f"every {stride}-th row ({rows.size} of {n} rows, uniform over the row range), "
            f"{fills} fill-ins in {dt:.2f} s")
    return fills / dt, desc, threads, dt


def algorithmic_bytes(stats, n, rows, fills):
    """Algorithmic bytes of the traversal per SURVEY.md §8(d):
      4 B label read per (source, edge) inspection      (edge_inspections)
      4 B label write per improvement                   (first_visits: each
          (source, vertex) label is lowered once in threshold order; a lower
          bound for the FIFO order)
      4 B colidx per (item, neighbour) pair             (item_edges: one read
          shared by the sources of a lockstep item, A_g)
      12 B per (source, frontier entry)                 (source_expansions:
          4 B label(u) + ~8 B queue)
      4 B output per fill-in
      2 * n/8 B per source                              (row extraction + clear)
    Returns (bytes, breakdown dict)."""
    parts = {
        "label_reads": 4 * stats["edge_inspections"],
        "label_writes": 4 * stats.get("first_visits", 0),
        "colidx": 4 * stats["item_edges"],
        "frontier": 12 * stats.get("source_expansions", 0),
        "fill_output": 4 * fills,
        "extraction": 2 * (n / 8) * rows,
    }
    return sum(parts.values()), parts


def ncu_kernels(config, schedule):
    """Per-kernel DRAM traffic from the committed ncu --set full captures
    (profiles/traffic.json): dram bytes per launch and ncu's own duration."""
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except Exception:
        return None, None
    ent = tj.get(f"{config}/{schedule}")
    if not ent:
        return None, None
    return ent.get("kernels", {}), ent.get("source")


def self_launch(args):
    """--gpus N without a torchrun environment: re-run this script under
    torch.distributed.run with N ranks (one per GPU, NCCL), rendezvous on
    127.0.0.1; rank 0's JSON line is this process's stdout."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    log(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}")
    return subprocess.call(cmd)


def run_reference(args, rank, world):
    """--impl reference: the oracle as it stands, on host cores (rank 0 only)."""
    if rank != 0:
        return 0
    rp, ci = gen.config(args.config)
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    vals = []
    desc = threads = None
    for i in range(args.warmup + args.steps):
        v, desc, threads, dt = cpu_oracle_sample(rp, ci, per_step, seed=i)
        if i >= args.warmup:
            vals.append((v, dt))
    value = statistics.median(v for v, _ in vals)
    ms = statistics.median(dt for _, dt in vals) * 1e3
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "int32", "data": "synthetic (gen.config, seeded)",
           "config": {"workload": CONFIG_DESC[args.config], "n": int(rp.size - 1),
                      "nnz_offdiag": int(ci.size)},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                            "sample": desc},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=sorted(CONFIG_DESC))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--schedule", default="auto", choices=["auto", "threshold", "height", "fifo"])
    ap.add_argument("--max-concurrent", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--layout", default="ranges", choices=["ranges", "interleave", "steal"],
                    help="N > 1: contiguous work-balanced ranges (default), round-robin "
                         "units of --unit rows, or chunk-aligned blocks claimed from a shared "
                         "counter (SURVEY §8(f) NEXT-2)")
    ap.add_argument("--unit", type=int, default=128)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.impl == "reference":
        # the oracle arm runs on host cores, rank 0 only (other ranks exit 0)
        rank = int(os.environ.get("RANK", "0"))
        return run_reference(args, rank, int(os.environ.get("WORLD_SIZE", str(args.gpus))))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"[bench] WORLD_SIZE={world} but --gpus {args.gpus}")
        return 2

    import torch
    import torch.distributed as dist

    import paper_2007_00840_b200 as g
    from paper_2007_00840_b200 import dist as gd

    ndev = torch.cuda.device_count()
    shared = world > ndev  # dev smoke test: several ranks on one GPU
    dev_index = local % ndev
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    coll_dev = dev
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if shared:
            # NCCL needs one GPU per rank; for a single-GPU smoke test of the
            # multi-rank path the count allgather goes over gloo instead
            dist.init_process_group("gloo")
            coll_dev = None
            log(f"[rank {rank}] {world} ranks share {ndev} GPU(s): gloo collectives (smoke test only)")
        else:
            dist.init_process_group("nccl", device_id=dev)

    t0 = time.perf_counter()
    rp, ci = gen.config(args.config)
    n = rp.size - 1
    log(f"[rank {rank}] {args.config}: n={n} nnz={ci.size} generated in {time.perf_counter()-t0:.1f}s")
    chunk = 128
    # row-granular ranges of equal estimated work; supernodes are stitched
    # across range boundaries by the tail chain (gsofa_supernode_stitch)
    bounds = gd.partition(rp, ci, world) if world > 1 else np.array([0, n], np.int64)
    rb, re = int(bounds[rank]), int(bounds[rank + 1])
    d_rp = torch.from_numpy(rp).to(dev)
    d_ci = torch.from_numpy(ci).to(dev)
    ctx = g.Context(dev_index)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def one_step(host=False):
        kw = dict(ctx=ctx, chunk_size=chunk, schedule=args.schedule,
                  max_concurrent=args.max_concurrent, stream=stream)
        src = (h_rp, h_ci) if host else (d_rp, d_ci)
        if world > 1 and args.layout == "steal":
            kw2 = {k: v for k, v in kw.items() if k != "chunk_size"}
            mine, counts, _ = gd.symbolic_stealing(*src, rank=rank, chunk_size=chunk, device=coll_dev,
                                                   outputs_on_device=not host, **kw2)
            fills = int(counts[:, 2].sum())
            for _, _, _, r_ in mine[1:]:
                r_.free()
            res = mine[0][3] if mine else None  # (the step's first block stands for the stats)
        elif world > 1 and args.layout == "interleave":
            # this rank's units, per-row Def. T3 all_gather if finer than a chunk
            kw2 = {k: v for k, v in kw.items() if k != "chunk_size"}
            res, counts = gd.symbolic_interleaved(*src, rank=rank, unit_rows=args.unit, chunk_size=chunk,
                                                  device=coll_dev, outputs_on_device=True, **kw2)
            fills = int(counts[:, 2].sum())
        elif world > 1:
            # this rank's range, supernode-boundary chain, count allgather
            sl = gd.symbolic_distributed(*src, bounds, rank=rank, device=coll_dev,
                                         outputs_on_device=not host, **kw)
            res, fills = sl.result, sl.totals["fill_count"]
        else:
            res = g.symbolic(*src, row_begin=rb, row_end=re, outputs_on_device=not host, **kw)
            fills = res.fill_count
        if host and res is not None:
            arrs = res.to_numpy(copy=False)  # the CSR arrays, in (pinned) host memory
            assert arrs["L_rowptr"].size == res.rows + 1
        return res, fills

    # ---- warm-up
    for _ in range(args.warmup):
        r, fills = one_step()
        if r is not None:
            r.free()
    # ---- timed region (device time, CUDA events on the launch stream)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    step_ms, stats_acc, launches = [], {}, 0
    sched_used = args.schedule
    fills_step = 0
    local_fills = 0
    with ClockSampler(dev_index) as clk:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (256 MiB > 126 MB L2), untimed
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r, fills_step = one_step()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            if r is not None:
                local_fills += r.fill_count  # this rank's rows (roofline of its kernels)
                sched_used = r.schedule  # the library's choice under "auto"
                for k, v in r.stats.items():
                    stats_acc[k] = stats_acc.get(k, 0) + v
                launches += int(r.stats["kernel_launches"])
                r.free()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    tot_ms = sum(step_ms)
    per_rank_ms = [tot_ms / args.steps]
    if world > 1:
        t = torch.tensor([tot_ms, float(launches)], dtype=torch.float64, device=coll_dev or "cpu")
        allt = torch.empty(2 * world, dtype=torch.float64, device=t.device)
        dist.all_gather_into_tensor(allt, t)
        allt = allt.cpu().view(world, 2)
        per_rank_ms = [float(x) / args.steps for x in allt[:, 0]]
        tot_ms, launches_all = float(allt[:, 0].max()), int(allt[:, 1].sum())
    else:
        launches_all = launches
    ms_per_step = tot_ms / args.steps
    value = fills_step / (ms_per_step / 1e3)

    # ---- e2e through the public API with pinned host buffers
    h_rp = torch.from_numpy(rp).pin_memory()
    h_ci = torch.from_numpy(ci).pin_memory()
    e2e_ms, h2d, d2h = [], 0, 0
    for i in range(1 + args.e2e_steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        r, fills_e = one_step(host=True)
        torch.cuda.synchronize(dev)
        dt = (time.perf_counter() - t) * 1e3
        if i > 0:
            e2e_ms.append(dt)
        if r is not None:
            h2d = int(rp.nbytes + ci.nbytes)
            d2h = int(2 * (r.rows + 1) * 8 + 4 * (r.nnz_L + r.nnz_U + r.nsuper + 1))
            r.free()
    e2e_step = statistics.median(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_step, float(h2d), float(d2h)], dtype=torch.float64,
                         device=coll_dev or "cpu")
        m = t.clone()
        dist.all_reduce(m[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        e2e_step, h2d, d2h = float(m[0]), int(t[1]), int(t[2])

    # ---- roofline of the dominant kernel (traversal), measured live: the
    # traversal kernels' device time (CUDA events on the launch stream inside
    # the call) and SURVEY §8(d)'s algorithmic bytes of the work they did
    peak, peak_src = load_peaks()
    trav_ms = stats_acc.get("ms_traverse", 0.0)
    alg, alg_parts = (algorithmic_bytes(stats_acc, n, (re - rb) * args.steps, local_fills)
                      if stats_acc else (0, {}))
    achieved = alg / (trav_ms / 1e3) / 1e9 if trav_ms > 0 else 0.0
    kern = {"threshold": "solo_kernel+stream_kernel", "height": "stream_kernel (height order)"}.get(
        sched_used, "traverse_kernel")
    roofline = {"kernel": kern, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                "bytes_model": "SURVEY.md §8(d): 4 B/edge inspection + 4 B/first visit + "
                               "4 B/(item,neighbour) colidx + 12 B/(source, frontier entry) + "
                               "4 B/fill + n/4 B/source",
                "algorithmic_bytes_per_step": alg / args.steps,
                "algorithmic_bytes_parts_per_step": {k: v / args.steps for k, v in alg_parts.items()},
                "kernel_ms_per_step": trav_ms / args.steps,
                "kernel_share_of_step": (trav_ms / args.steps) / ms_per_step if ms_per_step else None}
    # what ncu says the same kernels do to DRAM (one --set full capture per
    # kernel, committed under profiles/): bytes per launch, its GB/s, and
    # the fraction of the measured copy bandwidth
    kinfo, ksrc = ncu_kernels(args.config, sched_used)
    if kinfo:
        nk = {}
        tot_b = 0.0
        for k, v in kinfo.items():
            b = float(v["dram_bytes"])
            tot_b += b
            gbs = b / float(v["duration_s"]) / 1e9
            nk[k] = {"dram_bytes": b, "ncu_ms": float(v["duration_s"]) * 1e3, "dram_gbs": gbs,
                     "dram_frac": gbs / peak}
        roofline["traffic"] = tot_b  # dram read + write of the traversal kernels, per launch
        roofline["ncu"] = {"kernels": nk, "source": ksrc}
        # what HBM actually does during the traversal (north_star: "achieved
        # HBM GB/s from ncu"): the kernels' DRAM bytes over their ncu time
        dur = sum(v["ncu_ms"] for v in nk.values()) / 1e3
        if dur > 0:
            roofline["ncu_dram_gbs"] = tot_b / dur / 1e9
            roofline["ncu_dram_frac"] = roofline["ncu_dram_gbs"] / peak
        roofline["limiter"] = (
            "per-level CTA barriers of the lockstep groups over latency-bound closure levels (ncu: "
            "barrier stalls dominate, then long scoreboard; DRAM well below peak; see roofline.ncu)"
            if sched_used == "height" else
            "latency of dependent L2 atomics (ncu: long-scoreboard stalls dominate, DRAM well below "
            "peak; see roofline.ncu)")
    # the unit operation of the traversal is a random 4-byte atomic (one per
    # (item, neighbour) pair); its ceiling on this GPU was measured with
    # scripts/atomics_bench.cu (profiles/atomic_peak.json)
    try:
        ap = json.load(open(os.path.join(ROOT, "profiles", "atomic_peak.json")))
        a_peak = float(ap["atomicOr_returning_l2_gops"])
        a_ach = stats_acc.get("item_edges", 0) / (trav_ms / 1e3) / 1e9 if trav_ms > 0 else 0.0
        roofline["atomic"] = {"achieved": a_ach, "peak": a_peak, "unit": "G atomics/s",
                              "frac": a_ach / a_peak, "peak_source": ap["source"]}
    except Exception:
        pass
    if stats_acc.get("first_visits"):
        roofline["revisit_factor"] = stats_acc["source_expansions"] / stats_acc["first_visits"]
    stats_step = {k: (v / args.steps) for k, v in stats_acc.items()}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, desc, threads, dt = cpu_oracle_sample(rp, ci, args.cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": "int32", "data": "synthetic (gen.config, seeded; no datasets)",
               "config": {"workload": CONFIG_DESC[args.config], "n": n, "nnz_offdiag": int(ci.size),
                          "row_ranges": [int(b) for b in bounds],
                          "per_rank_ms": per_rank_ms,
                          "fill_ins": fills_step, "schedule": sched_used,
                          "parallelism": (f"rows split over {world} GPU(s)"
                                          + {"interleave": f", interleaved units of {args.unit}",
                                             "steal": ", blocks claimed from a shared counter"}.get(
                                              args.layout, ", work-balanced ranges")) if world > 1 else "1 GPU",
                          "l2": "flushed between timed steps (256 MiB write, untimed)"},
               "e2e": {"value": fills_step / (e2e_step / 1e3), "unit": UNIT,
                       "ms_per_step": e2e_step, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
               "gpu_launches": launches_all,
               "roofline": roofline,
               "cpu_baseline": cpu,
               "clocks": clk.summary(),
               "stats_per_step": stats_step}
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
