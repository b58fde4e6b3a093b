#!/usr/bin/env python
"""ALTO B200 hot-path benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], the config its metric is quoted on):
c2 = 12000 x 9000 x 28000, 76M unique Zipf(1.2) nonzeros, U(0,1) values,
R = 16, fp64, 64-bit ALTO keys; synthetic and seeded (no dataset exists).
A step is one CP-ALS sweep on the device: for every mode an MTTKRP (the hot
path) + the normal-equation solve + column normalisation + new Gram.
``value`` = MTTKRP nonzeros/s of the sweep = N_modes * M / step time, for
the whole job (all ranks). Multi-GPU: each rank owns a balanced ALTO-ordered
slice of the same tensor and the factor-sized partials are summed with one
NCCL all-reduce per mode (strong scaling).

Also reported: the MTTKRP kernel's roofline (algorithmic bytes per launch /
CUDA-event launch time vs the measured HBM copy bandwidth), the end-to-end
number through the public API with host buffers, the encoder (linearise +
sort) throughput, CP-APR seconds per outer iteration on c4 (BASELINE
configs[3]) with the Phi kernel's roofline, and the CPU baseline (the C/OpenMP
port of the reference kernels in oracle/, on a bounded sample).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

HBM_FALLBACK_GBS = 6650.0


def measured_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[4:8]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# CPU side: the oracle port (test infrastructure) as the reported baseline


def cpu_sweep_rate(cfg, nnz, steps, warmup, threads, seed=0):
    """MTTKRP nnz/s of a CP-ALS sweep by the C/OpenMP port of the reference
    kernels (recursive strategy, L = threads, like `alto bench mttkrp`
    with workers = threads) on a bounded sample with the config's shape and
    distributions."""
    from oracle import alto_oracle as orc
    from paper_2403_06348_b200 import synthetic

    coords, vals = synthetic.generate_numpy(cfg, nnz, seed=seed)
    keys, svals, scoords = orc.from_coo(cfg.dims, coords, vals)
    R = cfg.rank
    w, factors = orc.normalized(*orc.init_factors(cfg.dims, R, 0), ord=2)
    grams = [f.T @ f for f in factors]
    N = len(cfg.dims)

    seg_cache = {}  # the reference caches segments on the tensor (partition.py:87-89)
    orc.segments(scoords, threads)  # warm numpy paths
    orc.mttkrp(scoords, svals, factors, 0, "recursive", threads, threads, seg_cache=seg_cache)

    def sweep():
        nonlocal w
        for n in range(N):
            v = orc._hadamard(grams, skip=n)
            mt = orc.mttkrp(scoords, svals, factors, n, "recursive", threads, threads, seg_cache=seg_cache)
            a = orc._solve_pseudo(mt, v)
            norms = np.linalg.norm(a, axis=0)
            factors[n] = a / np.where(norms == 0.0, 1.0, norms)
            w = norms
            grams[n] = factors[n].T @ factors[n]

    for _ in range(warmup):
        sweep()
    t0 = time.perf_counter()
    for _ in range(steps):
        sweep()
    dt = (time.perf_counter() - t0) / steps
    return N * len(svals) / dt, dt, len(svals)


def cpu_apr_rate(cfg, nnz, threads, outers=2, seed=0):
    """CP-APR outer iterations by the C/OpenMP port of the reference kernels
    (cp_apr_mu's Phi loop + log-likelihood, recursive strategy, L = threads)
    on a bounded sample with the config's shape and distributions ->
    (nnz x outer iterations per s, s per outer, sample nnz, outers)."""
    from oracle import alto_oracle as orc
    from paper_2403_06348_b200 import synthetic

    coords, vals = synthetic.generate_numpy(cfg, nnz, seed=seed)
    _keys, svals, scoords = orc.from_coo(cfg.dims, coords, vals)
    seg_cache = {}  # the reference caches segments on the tensor (partition.py:87-89)
    orc.cp_apr(cfg.dims, scoords, svals, cfg.rank, 1, max_inner=1, strategy="recursive", L=threads,
               threads=threads, seg_cache=seg_cache)  # warm the library, numpy paths and segments
    t0 = time.perf_counter()
    orc.cp_apr(cfg.dims, scoords, svals, cfg.rank, outers, max_inner=10, strategy="recursive", L=threads,
               threads=threads, seg_cache=seg_cache)
    dt = (time.perf_counter() - t0) / outers
    return len(svals) / dt, dt, len(svals), outers


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2403_06348_b200 import synthetic

    cfg = synthetic.CONFIGS[args.config]
    threads = len(os.sched_getaffinity(0))
    rate, dt, m = cpu_sweep_rate(cfg, args.cpu_sample_nnz, args.steps, args.warmup, threads)
    sample = (f"{m} nnz drawn from the {cfg.name} distribution (shape {cfg.dims}, R={cfg.rank}); "
              f"CP-ALS sweep = {len(cfg.dims)} MTTKRPs (recursive strategy, L={threads}) + solves")
    line = {
        "impl": "reference",
        "metric": "MTTKRP nonzeros/sec (CP-ALS sweep)",
        "value": rate,
        "unit": "nnz/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dt * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded; BASELINE names no public dataset)",
        "config": {"workload": cfg.description, "sample_nnz": m, "threads": threads},
        "cpu_baseline": {"value": rate, "unit": "nnz/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": rate, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm


def _traffic(key: str, full_entry: bool = False, world: int = 1):
    """ncu-measured DRAM bytes per launch of the dominant kernel
    (profiles/traffic.json, from a 1-GPU ncu capture), or None. With
    ``world`` ranks each rank streams its 1/world shard: the per-launch
    bytes are scaled (a 1-GPU measurement, not a per-rank capture)."""
    prof = ROOT / "profiles" / "traffic.json"
    try:
        tr = json.loads(prof.read_text()).get(key)
    except Exception:
        return None
    if not tr:
        return None
    if world > 1:
        tr = dict(tr, dram_bytes_per_launch=tr["dram_bytes_per_launch"] / world,
                  note=(tr.get("note", "") + f" (1-GPU bytes / {world} ranks)").strip())
    return tr if full_entry else tr["dram_bytes_per_launch"]


def _timed(fn):
    import gc

    import torch

    gc.collect()  # free the previous driver state's device buffers before timing
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t0


def drivers_e2e(args, cfg, t):
    """Wall time of the public drivers on the BASELINE configurations, cold
    (fresh tensor object sharing the device arrays: decoded views, memo piece
    indices and Pi layouts are built inside the call) and warm (second call,
    caches reused): cp_als(c2, rank 16, 10 iterations) with and without the
    memoised sweep, and cp_apr_mu(c4, rank 10, 5 x 10)."""
    import torch

    import paper_2403_06348_b200 as alto
    from paper_2403_06348_b200 import synthetic
    from paper_2403_06348_b200.cpd import als as ALS

    def fresh(x):
        return alto.AltoTensor(x.layout, x._keys, x._vals, _validate=False)

    out = {}
    als_cfg = alto.CpAlsConfig(rank=cfg.rank, max_iters=10, fit_tol=1e-300, seed=0)
    rows = {}
    for memo in (True, False):
        os.environ["ALTO_B200_MEMO"] = "1" if memo else "0"
        try:
            tt = fresh(t)
            res, cold = _timed(lambda: alto.cp_als(tt, als_cfg))
            _, warm = _timed(lambda: alto.cp_als(tt, als_cfg))
        finally:
            os.environ.pop("ALTO_B200_MEMO", None)
        rows["memo" if memo else "plain"] = {"cold_s": cold, "warm_s": warm, "build_s": cold - warm,
                                             "fit": res.fit_trace[-1], "iters": res.n_iters}
        del tt
        torch.cuda.empty_cache()
    out["cp_als"] = {"workload": cfg.description, "call": "cp_als(alto, CpAlsConfig(rank=16, max_iters=10))",
                     **rows,
                     "default": "plain: cp_als builds the memoised layouts only when max_iters >= "
                                f"{ALS.AlsState.MEMO_MIN_ITERS} or they are cached on the tensor (cpd/als.py)"}
    if not args.no_apr:
        acfg = synthetic.CONFIGS[args.apr_config]
        ac, av = synthetic.generate(acfg, seed=0, nnz=args.apr_nnz or acfg.nnz)
        (at, enc) = _timed(lambda: alto.AltoTensor.from_device_coo(acfg.dims, ac, av))
        del ac, av
        apr_cfg = alto.CpAprConfig(rank=acfg.rank, max_outer=5, max_inner=10, eps=1e-10, seed=0)
        res, cold = _timed(lambda: alto.cp_apr_mu(at, apr_cfg))
        _, warm = _timed(lambda: alto.cp_apr_mu(at, apr_cfg))
        out["cp_apr"] = {"workload": acfg.description,
                         "call": "cp_apr_mu(alto, CpAprConfig(rank=10, max_outer=5, max_inner=10, eps=1e-10))",
                         "construction_s": enc, "cold_s": cold, "warm_s": warm, "build_s": cold - warm,
                         "s_per_outer_cold": cold / res.n_outer, "s_per_outer_warm": warm / res.n_outer,
                         "inner_iters": res.inner_iters, "loglik_last": res.loglik_trace[-1]}
        del at
        torch.cuda.empty_cache()
    return out


def _call_memo_stats(t, R):
    cm = t._cache.get(("callmemo", R))
    if cm is None:
        return None
    return {"produce_calls": cm.stats["produce"], "consume_calls": cm.stats["consume"],
            "note": "public mttkrp() calls served by the fused producer (stores T for the next mode) / by the "
                    "streaming consumer of the previous call's T (its A_k bitwise unchanged, checked on the "
                    "device); memo.CallMemo"}


def run_native(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    # ALTO_B200_DIST_BACKEND=gloo lets several ranks share one GPU (plumbing
    # checks on a 1-GPU box; such timings mean nothing). Production: NCCL.
    backend = os.environ.get("ALTO_B200_DIST_BACKEND", "nccl")
    dev_index = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(dev_index)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    import paper_2403_06348_b200 as alto
    from paper_2403_06348_b200 import _native as nat
    from paper_2403_06348_b200 import distributed as D
    from paper_2403_06348_b200 import kernels as K
    from paper_2403_06348_b200 import synthetic
    from paper_2403_06348_b200.cpd import als as ALS
    from paper_2403_06348_b200.cpd import apr as APR

    hbm, hbm_src = measured_hbm()
    cfg = synthetic.CONFIGS[args.config]
    nnz = args.nnz or cfg.nnz

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- build the tensor (seeded: the same COO is generated on every rank) ----
    coords, vals = synthetic.generate(cfg, seed=0, nnz=nnz)
    barrier()
    t0 = time.perf_counter()
    if world > 1:
        # each rank keeps an interleaved 1/W of the COO; the distributed
        # construction (encode, sort, splitter search, all-to-all, sort) cuts
        # exactly the single-GPU balanced ALTO shards
        t, _span = D.build_sharded(cfg.dims, coords[rank::world], vals[rank::world])
    else:
        t = alto.AltoTensor.from_device_coo(cfg.dims, coords, vals)
    barrier()
    encode_s = time.perf_counter() - t0
    del coords, vals
    m_all = torch.tensor([t.nnz], dtype=torch.int64, device="cuda")
    D.allreduce_(m_all)
    M = int(m_all.item())
    key_bytes = 8 if t.layout.word_bits == 64 else 16
    N = len(cfg.dims)
    R = cfg.rank

    norm_sq = torch.tensor([float(t._vals @ t._vals)], dtype=torch.float64, device="cuda")
    D.allreduce_(norm_sq)
    reduce = (lambda x: D.allreduce_(x)) if world > 1 else None
    # N > 1: the MTTKRP partials are reduce-scattered to row owners, each rank
    # solves its rows, the blocks are all-gathered (distributed.RowComm);
    # ALTO_B200_ALS_COMM=allreduce keeps one all-reduce of the partial
    # default with NCCL: the row-owner collectives on an NCCL communicator
    # owned by the C ABI (alto_nccl_*, distributed.NativeComm; CP-APR's Phi
    # all-reduce too), captured inside the sweep / outer-iteration graphs;
    # ALTO_B200_ALS_COMM=rows: torch.distributed's NCCL (eager);
    # =allreduce: one all-reduce of the partial
    als_comm = {}
    comm_kind = os.environ.get("ALTO_B200_ALS_COMM", "native" if backend == "nccl" else "rows")
    if world > 1:
        ncomm = None
        if comm_kind == "native" and backend == "nccl":
            try:
                ncomm = D.NativeComm()
            except RuntimeError as ex:
                print(f"warning: library NCCL communicator unavailable ({ex}); torch.distributed NCCL",
                      file=sys.stderr)
        if comm_kind == "allreduce":
            als_comm = {"reduce": reduce}
        elif ncomm is not None:
            als_comm = {"row_comm": ncomm}
            reduce = ncomm.all_reduce
        else:
            als_comm = {"row_comm": D.RowComm()}
    # the steady-state sweep of a CP-ALS loop: memoised (ALTO_B200_MEMO=0 for
    # the plain sweep); drivers_e2e reports the cold cp_als(10) choice
    st = ALS.AlsState(t, alto.CpAlsConfig(rank=R, max_iters=1, seed=0), norm_x_sq=float(norm_sq.item()), memo=True,
                      **als_comm)

    # warm-up sweeps (the device path captures the sweep as a CUDA graph on
    # the second one; every later sweep is one graph replay)
    for _ in range(args.warmup):
        st.sweep()
    # the memoised sweep alternates two kernel sequences (produce/consume/
    # produce, then consume/produce/consume): start the timed region with the
    # slower one, so an odd step count never reports the faster mix
    if st._memo() is not None and any(p.t_valid for p in st._memo_plans.values()):
        st.sweep()
    barrier()
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("timed")
    ev0.record()
    for _ in range(args.steps):
        st.sweep()
    ev1.record()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    step_ms = ev0.elapsed_time(ev1) / args.steps
    step_ms = D.allreduce_max(step_ms, device="cuda")
    fit, _ = st.fit()
    value = N * M / (step_ms / 1e3)
    device_als = hasattr(st, "_dgrams")
    footprint = _footprint(t, st)
    # our kernels per sweep: the MTTKRP of every mode (memo0 / memo1 / dview3
    # on the memoised path) + the ALS-update kernels per mode on the device
    # path (chol, solve_rows, norm_scale; the row-owner path at N > 1: chol,
    # solve, gram, gram_sum, final_raw, scale -- profiles/r02_launches_bench_c2_fused.csv)
    per_mode = {"dview": 1, "oriented": 1, "atomic": 1, "segment": 1, "exact-output": 3}
    als_k = (6 if world > 1 else 3) if device_als else 0
    launches = [args.steps * sum(per_mode.get(k, 2) + als_k for k in st.kernels)]
    if st._memo() is not None:
        # memoised sweep, averaged over its two patterns: a producing mode
        # launches one kernel, a consuming mode one; + the ALS-update kernels
        launches = [int(args.steps * (N * als_k + 1.5 + 1.5))]

    # MTTKRP launch time: the same launches as inside the sweep, each bracketed
    # by CUDA events on the launching stream (graph replays cannot be split)
    events = []
    for _ in range(3):
        for n in range(N):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            st.mttkrp(n)
            e1.record()
            events.append((n, e0, e1))
    torch.cuda.synchronize()

    per_mode = {n: [] for n in range(N)}
    for n, e0, e1 in events:
        per_mode[n].append(e0.elapsed_time(e1))
    mt_ms = {n: statistics.mean(v) for n, v in per_mode.items()}
    avg_launch_ms = statistics.mean(mt_ms.values())
    avg_launch_ms = D.allreduce_max(avg_launch_ms, device="cuda")
    alg_bytes = synthetic.algorithmic_bytes(cfg, t.nnz, R, key_bytes)
    achieved = alg_bytes / (avg_launch_ms / 1e3) / 1e9
    roofline = {
        "bound": "hbm",
        "kernel": f"MTTKRP ({'/'.join(sorted(set(st.kernels)))} kernel, CUDA events around each "
                  f"launch incl. the output zero-fill, 3 launches per mode after the timed sweeps)",
        "achieved": achieved,
        "peak": hbm,
        "peak_source": hbm_src,
        "unit": "GB/s",
        "frac": achieved / hbm,
        "traffic": None,
        "algorithmic_bytes_per_launch": alg_bytes,
        "bytes_model": "M*(W+8) + 8*R*sum(I_n)  (SURVEY.md 8(d))",
        # the gather-inclusive volume adds the (N-1) factor
        # rows every nonzero reads (served by L1/L2, not HBM)
        "gather_inclusive": {
            "bytes_per_launch": alg_bytes + t.nnz * (N - 1) * R * 8,
            "achieved_GBps": (alg_bytes + t.nnz * (N - 1) * R * 8) / (avg_launch_ms / 1e3) / 1e9,
            "note": "operand bytes delivered to the SMs per launch (factor-row gathers mostly hit L1/L2)",
        },
    }
    memo = st._memo() if hasattr(st, "_memo") else None
    if memo is not None:
        # operand bytes of the memoised kernels, averaged over the two sweep
        # patterns (3 producers + 3 consumers): a producer streams the view,
        # gathers N-1 rows per nonzero and writes one partial-sum row per
        # piece; a consumer reads a partial-sum row, a gathered row and three
        # u32 indices per piece
        rowb = 8 * R
        pieces = [p.P for p in st._memo_plans.values()]
        # factor rows gathered: a producing mode gathers one row per nonzero
        # (A_k) and one per piece (A_j: the fused producers
        # fiber-factored memo0 alike), a consuming mode one per piece; both
        # read or write one T row per piece
        g_prod = [t.nnz + pc for pc in pieces]
        g_cons = list(pieces)
        prod = [alg_bytes + g * rowb + pc * rowb for g, pc in zip(g_prod, pieces)]
        cons = [pc * (2 * rowb + 12) for pc in pieces]
        op = (sum(prod) + sum(cons)) / (len(prod) + len(cons))
        roofline["gather_inclusive"] = {
            "bytes_per_launch": op, "achieved_GBps": op / (avg_launch_ms / 1e3) / 1e9,
            "note": "operand bytes delivered to the SMs per launch, average of the memoised sweep's producer "
                    "and consumer launches (gathers mostly hit L1/L2)"}
        gathered_rows_per_step = (sum(g_prod) + sum(g_cons)) / 2  # the two patterns alternate
        roofline["kernel"] = ("MTTKRP, average launch of the memoised sweep (" + _memo_label(st) + "; producing "
                              "modes: piece sums T = sum_k v A_k[k] and the MTTKRP from them; consuming modes: the "
                              "next mode's MTTKRP from T); CUDA events around each launch incl. the output "
                              "zero-fill, 3 launches per mode after the timed sweeps")
    else:
        gathered_rows_per_step = N * t.nnz * (N - 1)
    # the gather ceiling measured on this box (csrc/probe.cu): random 128-byte
    # rows from an L2-resident table / an L1-resident table, all SMs
    try:
        rps = ctypes.c_double(0.0)
        K.nat.call("alto_gather_probe", 28000, 5, ctypes.byref(rps))
        l2_rows = rps.value
        K.nat.call("alto_gather_probe", 512, 5, ctypes.byref(rps))
        l1_rows = rps.value
        gb = gathered_rows_per_step * 8 * K.nat.padded_ld(R)
        ach = gb / (step_ms / 1e3) / 1e9
        ceil_gbs = l2_rows * 8 * K.nat.padded_ld(R) / 1e9
        roofline["gather"] = {
            "bound": "l1tex gather", "unit": "GB/s", "achieved": ach, "peak": ceil_gbs, "frac": ach / ceil_gbs,
            "peak_l1_resident": l1_rows * 8 * K.nat.padded_ld(R) / 1e9,
            "bytes_per_step": gb,
            "note": "factor-row bytes gathered per CP-ALS sweep / sweep time, against the measured random "
                    "128-byte-row gather rate of this GPU (csrc/probe.cu: L2-resident table; peak_l1_resident: "
                    "L1-resident table); the decoded-view kernels are bound by this path, not by HBM "
                    "(profiles/r02_memo_split.md)"}
    except Exception as ex:  # measurement only
        roofline["gather"] = {"error": str(ex)[:200]}
    tr = _traffic(f"{args.config}_sweep_memo" if memo is not None else args.config, full_entry=True, world=world)
    if tr:
        roofline["traffic"] = tr["dram_bytes_per_launch"]
        roofline["traffic_source"] = tr.get("source")
        roofline["traffic_GBps"] = tr["dram_bytes_per_launch"] / (avg_launch_ms / 1e3) / 1e9

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        # the factors evolve like a user's CP-ALS loop: KV pinned versions of
        # each factor; in sweep s, mode n's call sees the modes before n in
        # their version s + 1 (updated earlier in the sweep), the others in
        # version s (no factor is ever passed unchanged where ALS changes it)
        rng = np.random.default_rng(1)
        KV = 4
        hv = []
        for d in cfg.dims:
            vers = []
            for _v in range(KV):
                buf = torch.empty((d, R), dtype=torch.float64, pin_memory=True)
                buf.copy_(torch.from_numpy(rng.random((d, R))))
                vers.append(buf.numpy())
            hv.append(vers)
        h2d = sum(v[0].nbytes for v in hv) * (N - 1)  # a mode's own factor is checked, not uploaded
        d2h = sum(d * R * 8 for d in cfg.dims)
        sweep_no = [0]

        def e2e_mode(n):
            s = sweep_no[0]
            host = [hv[m][(s + (1 if m < n else 0)) % KV] for m in range(N)]
            out = alto.mttkrp(t, host, n)  # numpy result: synchronised
            if world > 1:  # this rank's shard -> the full result: sum the partials
                part = torch.from_numpy(out).cuda()
                D.allreduce_(part)
                out = part.cpu().numpy()
            return out

        def e2e_sweep():
            for n in range(N):
                e2e_mode(n)
            sweep_no[0] += 1

        for _ in range(3):
            e2e_sweep()
        barrier()
        e2e_steps = max(3, min(args.steps, 10))
        step_s = []
        for _ in range(e2e_steps):
            t0 = time.perf_counter()
            e2e_sweep()
            step_s.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        e2e_s = D.allreduce_max(statistics.mean(step_s), device="cuda")
        e2e = {"value": N * M / e2e_s, "unit": "nnz/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
               "ms_per_step_min": min(step_s) * 1e3, "ms_per_step_median": statistics.median(step_s) * 1e3,
               "api": "paper_2403_06348_b200.mttkrp(alto, numpy factors in pinned host memory, mode) "
                      "per mode -> numpy; the ALTO tensor stays device resident; the factors evolve like a "
                      "CP-ALS loop (4 versions per factor, the modes before n updated when mode n is called)"
                      + ("; N > 1: each rank's shard, partials summed across ranks and read back"
                         if world > 1 else ""),
               "call_memo": _call_memo_stats(t, R)}

    # ---- CP-APR on c4 (BASELINE configs[3]) ----
    apr = None
    if not args.no_apr:
        acfg = synthetic.CONFIGS[args.apr_config]
        ann = args.apr_nnz or acfg.nnz
        ac, av = synthetic.generate(acfg, seed=0, nnz=ann)
        if world > 1:  # distributed construction of this rank's ALTO shard
            at, _span = D.build_sharded(acfg.dims, ac[rank::world], av[rank::world])
            afull = at
        else:
            afull = at = alto.AltoTensor.from_device_coo(acfg.dims, ac, av)
        del ac, av
        ast = APR.AprState(at, alto.CpAprConfig(rank=acfg.rank, max_outer=5, max_inner=10, eps=1e-10, seed=0),
                           reduce=reduce)
        # warm-up: outer 1 (no shift), outer 2 (first shift; lazy module
        # loads), outer 3 (captured as a CUDA graph and replayed); the timed
        # outers are graph replays
        ast.outer()
        ast.outer()
        ast.outer()
        barrier()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record()
        a_steps = args.apr_steps
        for _ in range(a_steps):
            ast.outer()
        a1.record()
        barrier()
        s_outer = D.allreduce_max(a0.elapsed_time(a1) / 1e3 / a_steps, device="cuda")
        # Phi launch times: the same launches as inside the outer iterations,
        # bracketed by CUDA events (graph replays cannot be split): the first
        # inner iteration of a mode gathers factor rows (and stores the
        # Khatri-Rao rows when the later ones stream them), iterations 2..
        # stream Pi (csrc/pstream.cu)
        pil = ast._pstream_buf(0)
        gat_ev, str_ev = [], []
        for m in range(len(acfg.dims)):
            ratio = torch.zeros_like(ast.b[m])
            for _ in range(3):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                APR.launch_phi(at, ast.dfac, m, ast.kernels[m], ast.b[m], 1e-10, out=ratio, pi_il_out=pil)
                e1.record()
                gat_ev.append((m, e0, e1))
            if pil is not None:
                for _ in range(3):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    APR.launch_phi_pstream(at, m, acfg.rank, ast.b[m], 1e-10, pil, ratio)
                    e1.record()
                    str_ev.append((m, e0, e1))
        torch.cuda.synchronize()
        akey = 8 if afull.layout.word_bits == 64 else 16

        def phi_line(evs, kind):
            ms = D.allreduce_max(statistics.mean(e0.elapsed_time(e1) for _, e0, e1 in evs), device="cuda")
            byts = statistics.mean(synthetic.algorithmic_bytes(acfg, at.nnz, acfg.rank, akey, kind, m)
                                   for m, _, _ in evs)
            ach = byts / (ms / 1e3) / 1e9
            return ms, {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                        "algorithmic_bytes_per_launch": byts}

        gat_ms, gat_roof = phi_line(gat_ev, "phi")
        gat_roof["traffic"] = _traffic(f"{args.apr_config}_phi", world=world)
        calls = sum(ast.inner_counts[-1])
        apr = {
            "workload": acfg.description,
            "s_per_outer_iteration": s_outer,
            "outer_iterations_timed": a_steps,
            "phi_calls_per_outer": calls,
            "inner_iters_last": ast.inner_counts[-1],
            "loglik_last": ast.loglik_trace[-1],
            "phi_kernels": ast.kernels,
            "phi_gather_ms": gat_ms,
            "phi_gather_roofline": gat_roof,
        }
        if str_ev:
            str_ms, str_roof = phi_line(str_ev, "phi_pre")
            # the streamed layout's compulsory bytes: per nonzero R doubles of
            # Pi + its row + its value (u16 + u8 in the compact layout of
            # count data, u32 + f64 otherwise), + B and Phi rows
            compact = APR.pstream_view(at, 0, acfg.rank)[2]
            per_nnz = 8 * acfg.rank + (3 if compact else 12)
            lay_b = statistics.mean(at.nnz * per_nnz + 16 * acfg.dims[m] * acfg.rank for m, _, _ in str_ev)
            str_roof.update({
                "achieved": lay_b / (str_ms / 1e3) / 1e9,
                "frac": lay_b / (str_ms / 1e3) / 1e9 / hbm,
                "algorithmic_bytes_per_launch": lay_b,
                "bytes_model": f"streamed Pi layout: M*(8R + {per_nnz - 8 * acfg.rank}) + 16*I_n*R "
                               f"({'u16 row + u8 count' if compact else 'u32 row + f64 value'} per nonzero; Pi stored "
                               "by the gathering Phi); the SURVEY.md 8(d) PRE model M*(W+8) + 8*M*R + 16*I_n*R = "
                               f"{statistics.mean(synthetic.algorithmic_bytes(acfg, at.nnz, acfg.rank, akey, 'phi_pre', m) for m, _, _ in str_ev):.4g} B",
            })
            str_roof["traffic"] = _traffic(f"{args.apr_config}_phi_stream", world=world)
            if str_roof["traffic"]:
                str_roof["traffic_GBps"] = str_roof["traffic"] / (str_ms / 1e3) / 1e9
                str_roof["traffic_frac"] = str_roof["traffic_GBps"] / hbm
            n_str = calls - len(acfg.dims)
            apr.update({
                "phi_stream_ms": str_ms,
                "phi_streamed_calls_per_outer": n_str,
                "phi_ms_avg": (gat_ms * len(acfg.dims) + str_ms * n_str) / max(calls, 1),
                # the dominant kernel of the outer iteration
                "phi_roofline": str_roof,
            })
        else:
            apr.update({"phi_ms_avg": gat_ms, "phi_roofline": gat_roof})
        del ast, at, afull

    # ---- per-mode MTTKRP on the other BASELINE configs (c3: the adaptive
    # privatise-vs-atomic choice per mode; optional c5 shard) ----
    extra = []
    for spec in [x for x in args.mttkrp_configs.split(",") if x]:
        name, _, nn = spec.partition(":")
        xcfg = synthetic.CONFIGS[name]
        xnnz = int(float(nn)) if nn else xcfg.nnz
        xc, xv = synthetic.generate(xcfg, seed=0, nnz=xnnz)
        if world > 1:  # distributed construction of this rank's ALTO shard
            xt, _span = D.build_sharded(xcfg.dims, xc[rank::world], xv[rank::world])
        else:
            xt = alto.AltoTensor.from_device_coo(xcfg.dims, xc, xv)
        del xc, xv
        xm = torch.tensor([xt.nnz], dtype=torch.int64, device="cuda")
        D.allreduce_(xm)
        xnnz_all = int(xm.item())
        xR = xcfg.rank
        g = torch.Generator(device="cuda").manual_seed(0)
        xfac = K.DeviceFactors([torch.rand((d, xR), dtype=torch.float64, device="cuda", generator=g)
                                for d in xcfg.dims], xR)
        xkey = 8 if xt.layout.word_bits == 64 else 16
        modes = []
        for n in range(len(xcfg.dims)):
            kern, why = K.select_gpu_kernel(xt, n, xR, None)
            out = K.launch_mttkrp(xt, xfac, n, kern)  # builds the view (untimed)
            if reduce is not None:
                reduce(out)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                K.launch_mttkrp(xt, xfac, n, kern, out=out)
                if reduce is not None:
                    reduce(out)
            e1.record()
            torch.cuda.synchronize()
            ms = D.allreduce_max(e0.elapsed_time(e1) / 3, device="cuda")
            xb = synthetic.algorithmic_bytes(xcfg, xnnz_all, xR, xkey)
            modes.append({"mode": n, "kernel": kern, "reason": why, "ms": ms,
                          "nnz_per_s": xnnz_all / (ms / 1e3),
                          "roofline_frac": xb / (ms / 1e3) / 1e9 / hbm})
            xt._cache.clear()  # one mode's views at a time (c3: 140M nnz)
        extra.append({"workload": xcfg.description, "nnz": xnnz_all,
                      "key_bits": xt.layout.total_bits,
                      "sample": "full config" if xnnz == xcfg.nnz else f"{xnnz} of {xcfg.nnz} nnz",
                      "modes": modes})
        del xt, xfac
        torch.cuda.empty_cache()

    # ---- drivers end to end through the public API (N = 1): cold runs on a
    # tensor with empty caches include every view / memo / Pi-layout build,
    # warm runs reuse them; the difference is the construction cost ----
    drivers = None
    if not args.no_drivers and world == 1:
        drivers = drivers_e2e(args, cfg, t)

    # ---- CPU baseline (rank 0, N = 1) ----
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        threads = len(os.sched_getaffinity(0))
        rate, dt, m = cpu_sweep_rate(cfg, args.cpu_sample_nnz, args.cpu_steps, 1, threads)
        cpu = {"value": rate, "unit": "nnz/s", "cores": threads, "kind": "port",
               "sample": f"{m} nnz from the {cfg.name} distribution, {args.cpu_steps} CP-ALS sweeps "
                         f"(C/OpenMP port of the reference numba kernels, recursive strategy, "
                         f"L = {threads}), {dt:.2f} s per sweep"}

        if apr is not None:
            acfg = synthetic.CONFIGS[args.apr_config]
            arate, adt, am, aouter = cpu_apr_rate(acfg, args.cpu_apr_sample_nnz, threads)
            full_nnz = args.apr_nnz or acfg.nnz
            apr["cpu_baseline"] = {
                "value": adt * full_nnz / am, "unit": "s/outer iteration (extrapolated per nonzero)",
                "nnz_iterations_per_s": arate, "cores": threads, "kind": "port",
                "sample": f"{am} nnz from the {acfg.name} distribution, {aouter} CP-APR outer iterations "
                          f"(max_inner {10}, C/OpenMP port of the reference numba kernels, recursive strategy, "
                          f"L = {threads}), {adt:.3f} s per outer; value = that time x {full_nnz} / {am}"}

    if rank == 0:
        line = {
            "metric": "MTTKRP nonzeros/sec (CP-ALS sweep)",
            "value": value,
            "unit": "nnz/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": step_ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded stand-in for BASELINE configs; no public dataset named)",
            "config": {
                "workload": cfg.description,
                "dims": list(cfg.dims),
                "nnz": M,
                "rank": R,
                "key_bits": t.layout.total_bits,
                "key_bytes": key_bytes,
                "step": "one CP-ALS sweep on device: per mode MTTKRP + normal-equation solve "
                        "+ normalisation + Gram"
                        + ("; solve/normalise/Gram on the GPU (the Cholesky on a side stream, "
                           "overlapped with the MTTKRP), sweep replayed as a CUDA graph (one per "
                           "memoised-sweep pattern), one host sync per sweep" if device_als else ""),
                "l2": "no flush: the 1.5 GB/mode nonzero stream exceeds the 126 MB L2; the "
                      "factor matrices stay L2-resident as in any CP-ALS loop",
                "parallelism": (f"ALTO-order nonzero shards x{world}, "
                                + ("NCCL via the C ABI (alto_nccl_*) " if isinstance(als_comm.get("row_comm"),
                                                                                 D.NativeComm)
                                   else f"{backend.upper()} ")
                                + ("all-reduce of the MTTKRP partials" if "reduce" in als_comm else
                                   "reduce-scatter of the MTTKRP partials to row owners, owner solve, "
                                   "all-reduce of the R x R Gram, all-gather of the factor"))
                if world > 1 else "single GPU",
                "kernels": ([_memo_label(st)] * N if st._memo() is not None else st.kernels),
                "memo": (None if st._memo() is None else
                         {"pairs": {f"{a}->{b}": p.P for (a, b), p in st._memo_plans.items()},
                          "note": "a producing mode's pass also stores sum over the third mode of v*A[k] per "
                                  "(row, next-mode) piece, at the piece's slot in the next mode's order; the "
                                  "next mode streams them (one gathered row per piece); sweeps alternate "
                                  "produce/consume/produce and consume/produce/consume "
                                  "(paper_2403_06348_b200/memo.py, csrc/memo_sums.cu)"}),
                "fit_after": fit,
            },
            "mttkrp_ms_per_mode": [mt_ms[n] for n in range(N)],
            "roofline": roofline,
            "clocks": clk,
            "e2e": e2e,
            "gpu_launches": launches[0],
            "footprint": footprint,
            "encoder": {"nnz": M, "seconds": encode_s, "nnz_per_s": M / encode_s,
                        "stages": "device linearise + radix sort of (key, value)"
                        + (" + splitter search + all-to-all + sort (distributed construction)"
                           if world > 1 else "")},
            "cp_apr": apr,
            "drivers_e2e": drivers,
            "mttkrp_other_configs": extra,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _footprint(t, st) -> dict:
    """Device bytes behind the timed sweep: the ALTO tensor (keys + values)
    next to the layouts the fast kernels stream (cached on the tensor) and the
    memoised sweep's partial sums -- the memory paid for the speed."""
    import torch

    def nbytes(x, seen):
        if isinstance(x, torch.Tensor):
            if not x.is_cuda:
                return 0
            key = x.untyped_storage().data_ptr()
            if key in seen:
                return 0
            seen.add(key)
            return x.untyped_storage().nbytes()
        if isinstance(x, (tuple, list)):
            return sum(nbytes(y, seen) for y in x)
        if isinstance(x, dict):
            return sum(nbytes(y, seen) for y in x.values())
        return 0

    seen = set()
    alto_b = nbytes([t._keys, t._vals], seen)
    layouts = {}
    for k, v in t._cache.items():
        b = nbytes(v, seen)
        if b:
            name = str(k[0]) if isinstance(k, tuple) else str(k)
            layouts[name] = layouts.get(name, 0) + b
    plans = getattr(st, "_memo_plans", None) or {}
    t_b = sum(nbytes(p.T, seen) for p in plans.values())
    total = sum(layouts.values()) + t_b
    return {"alto_tensor_bytes": alto_b, "layout_bytes": layouts, "memo_partial_sum_bytes": t_b,
            "layouts_over_tensor": total / max(alto_b, 1),
            "note": "fstream: interleaved fiber streams of the fused kernels (24 B per nonzero with consumer slots); "
                    "memo_cons: consumer order of the pieces; memo_partial_sum_bytes: T, one R-row per piece and "
                    "pair; all built from the ALTO tensor on first use and droppable (AltoTensor._cache)"}


def _memo_label(st) -> str:
    kind = next(iter(st._memo_plans.values())).kind
    prod = {"fused": "memo_fused_kernel", "memo0": "memo0_kernel"}.get(kind, kind)
    cons = "memo_consume_kernel" if kind == "fused" else "memo1_kernel"
    return f"{prod} (producing modes) / {cons} (consuming modes)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("native", "reference"), default="native")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--nnz", type=int, default=0)
    ap.add_argument("--apr-config", default="c4")
    ap.add_argument("--apr-nnz", type=int, default=0)
    ap.add_argument("--apr-steps", type=int, default=3)
    ap.add_argument("--no-apr", action="store_true")
    ap.add_argument("--mttkrp-configs", default="c3,c5",
                    help="comma list of configs for per-mode MTTKRP lines, name[:nnz] (e.g. c3,c5:62500000)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-drivers", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-nnz", type=int, default=4_000_000)
    ap.add_argument("--cpu-steps", type=int, default=60)
    ap.add_argument("--cpu-apr-sample-nnz", type=int, default=2_000_000)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "native":
        print("note: warm-up raised to the contract minimum of 3", file=sys.stderr)
        args.warmup = 3
    return run_reference(args) if args.impl == "reference" else run_native(args)


if __name__ == "__main__":
    sys.exit(main())
