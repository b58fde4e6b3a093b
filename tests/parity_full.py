"""Full-size parity on the benchmarked inputs (test infrastructure).

The bench times CP-ALS on BASELINE configs[1] (c2) and CP-APR on configs[3]
(c4), both generated on the GPU by ``synthetic.generate(cfg, seed=0)``. This
module downloads exactly those COO arrays and hands them to the CPU oracle
(``oracle/alto_oracle.py``, pinned to the reference by tests/golden), so the
tensors the bench measures are the ones checked:

* c1, c2, c4, c3: ALTO keys, sort order and values bit-exact at full size
  (reference ``pkg/src/alto/tensor.py:188-210``), c3 with 128-bit keys;
* c2, c4: ``make_segments`` bounds, per-mode intervals and boundary rows for
  L in {16, 148} bit-exact (``pkg/src/alto/partition.py:78-123``);
* c2: per-mode MTTKRP through the public ``mttkrp`` vs the oracle's
  recursive strategy (the reference with ``workers = cores``);
* c2: ``cp_als(rank=16, max_iters=10)`` fit trace, weights and factors vs
  the oracle driver (``pkg/src/alto/cpd/als.py:64-151``);
* c4: ``cp_apr_mu(rank=10, 5 x 10, eps=1e-10)``: inner iteration counts
  identical, KKT / log-likelihood traces, weights and factors vs the oracle
  driver (``pkg/src/alto/cpd/apr.py:210-346``); any flip of the ``kkt < tau``
  break (apr.py:302) is reported;
* c3 / c5: per-mode MTTKRP on ALTO shard 0 of 8 (the first
  ``balanced_bounds(M, 8)`` slice, what rank 0 of an 8-GPU run owns), keys
  round-tripped through the oracle's encoder.

``python tests/parity_full.py [names...] --json out.json`` writes the report;
``tests/test_gpu_parity_full.py`` asserts on it. Nothing here is product code.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from oracle import alto_oracle as orc  # noqa: E402

REL_FP64 = 1e-9  # north_star: fp64 results within 1e-9 relative


def _threads() -> int:
    return len(os.sched_getaffinity(0))


def _rel(got, want) -> float:
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = max(float(np.abs(want).max(initial=0.0)), 1e-300)
    return float(np.abs(got - want).max(initial=0.0)) / scale


def _generate(name: str):
    import torch

    import paper_2403_06348_b200 as alto
    from paper_2403_06348_b200 import synthetic

    cfg = synthetic.CONFIGS[name]
    coords, vals = synthetic.generate(cfg, seed=0)  # the bench's tensor
    hc = coords.cpu().numpy()
    hv = vals.cpu().numpy()
    t = alto.AltoTensor.from_device_coo(cfg.dims, coords, vals)
    del coords, vals
    torch.cuda.synchronize()
    return cfg, t, hc, hv


def _encoder(cfg, t, hc, hv, rep: dict):
    t0 = time.perf_counter()
    keys, svals, scoords = orc.from_coo(cfg.dims, hc, hv)
    rep["oracle_encode_sort_s"] = time.perf_counter() - t0
    pos = t.positions
    rep["nnz"] = int(len(svals))
    rep["key_bits"] = t.layout.total_bits
    rep["keys_bit_exact"] = bool(pos.shape == keys.shape and np.array_equal(pos, keys))
    rep["values_bit_exact"] = bool(np.array_equal(t.values, svals))
    t._positions = None  # drop the host copy
    return keys, svals, scoords


def _segments(t, scoords, rep: dict, Ls=(16, 148)):
    from paper_2403_06348_b200.partition import make_segments

    out = {}
    for L in Ls:
        bounds, lo, hi, boundary = orc.segments_large(scoords, L)
        seg = make_segments(t, L)
        ok_b = bool(np.array_equal(seg.bounds(), bounds))
        ok_i = all(np.array_equal(np.stack(seg.interval_arrays(n)), np.stack([lo[:, n], hi[:, n]]))
                   for n in range(scoords.shape[1]))
        ok_r = all(np.array_equal(seg.boundary_rows_of(n), boundary[n]) for n in range(scoords.shape[1]))
        out[str(L)] = {"bounds": ok_b, "intervals": ok_i, "boundary_rows": ok_r,
                       "boundary_row_counts": [int(b.size) for b in boundary]}
    rep["segments"] = out


def _mttkrp_modes(t, scoords, svals, factors, rep: dict, threads: int):
    import paper_2403_06348_b200 as alto

    seg_cache = {}
    errs, ms = [], []
    for n in range(len(factors)):
        got = alto.mttkrp(t, factors, n)
        t0 = time.perf_counter()
        want = orc.mttkrp(scoords, svals, factors, n, "recursive", threads, threads, seg_cache=seg_cache)
        ms.append(time.perf_counter() - t0)
        errs.append(_rel(got, want))
    rep["mttkrp_rel_err"] = errs
    rep["oracle_mttkrp_s"] = ms


def check_c1(rep: dict) -> None:
    cfg, t, hc, hv = _generate("c1")
    keys, svals, scoords = _encoder(cfg, t, hc, hv, rep)
    del hc, hv, keys
    _segments(t, scoords, rep)
    _, factors = orc.init_factors(cfg.dims, cfg.rank, 0)
    _mttkrp_modes(t, scoords, svals, factors, rep, _threads())


def check_c2(rep: dict, als_iters: int = 10) -> None:
    import paper_2403_06348_b200 as alto

    threads = _threads()
    cfg, t, hc, hv = _generate("c2")
    keys, svals, scoords = _encoder(cfg, t, hc, hv, rep)
    del hc, hv, keys
    _segments(t, scoords, rep)
    _, factors = orc.init_factors(cfg.dims, cfg.rank, 0)
    _mttkrp_modes(t, scoords, svals, factors, rep, threads)
    # CP-ALS, BASELINE configs[1]: rank 16, 10 iterations, on both sweep paths:
    # memoised (the bench's steady-state sweep: fused producer + streaming
    # consumer, device update, graph replay) and plain (what cp_als(10) picks)
    t0 = time.perf_counter()
    w, fs, fits = orc.cp_als(cfg.dims, scoords, svals, cfg.rank, als_iters, seed=0, strategy="recursive",
                             L=threads, threads=threads, seg_cache={})
    rep["oracle_cp_als_s"] = time.perf_counter() - t0
    for key, memo in (("cp_als", "1"), ("cp_als_plain", "0")):
        os.environ["ALTO_B200_MEMO"] = memo
        try:
            t0 = time.perf_counter()
            res = alto.cp_als(t, alto.CpAlsConfig(rank=cfg.rank, max_iters=als_iters, fit_tol=1e-300, seed=0))
            rep["gpu_" + key + "_s"] = time.perf_counter() - t0
        finally:
            os.environ.pop("ALTO_B200_MEMO", None)
        rep[key] = {
            "iters": len(res.fit_trace),
            "fit_gpu": res.fit_trace,
            "fit_oracle": fits,
            "fit_abs_err": float(np.abs(np.asarray(res.fit_trace) - np.asarray(fits)).max()),
            "weights_rel_err": _rel(res.model.weights, w),
            "factors_rel_err": [_rel(a, b) for a, b in zip(res.model.factors, fs)],
        }


def check_c4(rep: dict, outers: int = 5) -> None:
    import paper_2403_06348_b200 as alto

    threads = _threads()
    cfg, t, hc, hv = _generate("c4")
    keys, svals, scoords = _encoder(cfg, t, hc, hv, rep)
    del hc, hv, keys
    _segments(t, scoords, rep)
    t0 = time.perf_counter()
    res = alto.cp_apr_mu(t, alto.CpAprConfig(rank=cfg.rank, max_outer=outers, max_inner=10, eps=1e-10, seed=0))
    rep["gpu_cp_apr_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    w, fs, kkts, inners, lls = orc.cp_apr(cfg.dims, scoords, svals, cfg.rank, outers, max_inner=10, seed=0,
                                          eps=1e-10, strategy="recursive", L=threads, threads=threads,
                                          seg_cache={})
    rep["oracle_cp_apr_s"] = time.perf_counter() - t0
    gi = [list(map(int, x)) for x in res.inner_iters]
    flips = [(o, n, gi[o][n], inners[o][n]) for o in range(min(len(gi), len(inners)))
             for n in range(len(inners[o])) if gi[o][n] != inners[o][n]]
    rep["cp_apr"] = {
        "n_outer": [res.n_outer, len(inners)],
        "inner_iters_gpu": gi,
        "inner_iters_oracle": inners,
        "inner_iters_identical": gi == [list(map(int, x)) for x in inners],
        "flips": flips,
        "kkt_rel_err": _rel(np.asarray(res.kkt_trace), np.asarray(kkts)) if not flips else None,
        "loglik_gpu": list(map(float, res.loglik_trace)),
        "loglik_oracle": lls,
        "loglik_rel_err": _rel(res.loglik_trace, lls),
        "weights_rel_err": _rel(res.model.weights, w),
        "factors_rel_err": [_rel(a, b) for a, b in zip(res.model.factors, fs)],
    }


def check_c3_keys(rep: dict) -> None:
    """c3 at full size: 140M nonzeros, 71 index bits -> 128-bit keys."""
    cfg, t, hc, hv = _generate("c3")
    keys, svals, scoords = _encoder(cfg, t, hc, hv, rep)


def check_shard(name: str, rep: dict, world: int = 8, rank: int = 0) -> None:
    """Per-mode MTTKRP on ALTO shard ``rank`` of ``world`` of the full config."""
    import paper_2403_06348_b200 as alto
    from paper_2403_06348_b200 import distributed as D
    from paper_2403_06348_b200 import synthetic

    cfg = synthetic.CONFIGS[name]
    coords, vals = synthetic.generate(cfg, seed=0)
    full = alto.AltoTensor.from_device_coo(cfg.dims, coords, vals)
    del coords, vals
    sh = D.shard_tensor(full, world, rank)
    # materialise the shard as its own tensor so the full one can be freed
    t = alto.AltoTensor(full.layout, sh._keys.clone(), sh._vals.clone(), _validate=False)
    rep["full_nnz"] = full.nnz
    del sh, full
    import torch

    torch.cuda.empty_cache()
    rep["shard"] = f"ALTO shard {rank} of {world} (balanced_bounds(M, {world}))"
    pos = t.positions
    scoords = t.coords  # decoded on the device ...
    svals = t.values
    enc = orc.encode(cfg.dims, scoords)  # ... and re-encoded by the oracle
    rep["nnz"] = int(t.nnz)
    rep["keys_roundtrip_bit_exact"] = bool(np.array_equal(enc, pos))
    if pos.ndim == 1:
        rep["keys_strictly_increasing"] = bool((pos[1:] > pos[:-1]).all())
    else:
        hi, lo = pos[:, 1], pos[:, 0]
        rep["keys_strictly_increasing"] = bool(((hi[1:] > hi[:-1]) | ((hi[1:] == hi[:-1]) & (lo[1:] > lo[:-1]))).all())
    del enc, pos
    rng = np.random.default_rng(7)
    factors = [rng.random((d, cfg.rank)) for d in cfg.dims]
    _mttkrp_modes(t, scoords, svals, factors, rep, _threads())


CHECKS = {
    "c1": check_c1,
    "c2": check_c2,
    "c4": check_c4,
    "c3_keys": check_c3_keys,
    "c3_shard": lambda rep: check_shard("c3", rep),
    "c5_shard": lambda rep: check_shard("c5", rep),
}


def run(name: str) -> dict:
    import torch

    rep: dict = {"check": name, "threads": _threads()}
    t0 = time.perf_counter()
    CHECKS[name](rep)
    rep["wall_s"] = time.perf_counter() - t0
    torch.cuda.empty_cache()
    return rep


def failures(rep: dict) -> list[str]:
    """Human-readable list of the parity bars a report misses."""
    bad = []
    for k in ("keys_bit_exact", "values_bit_exact", "keys_roundtrip_bit_exact", "keys_strictly_increasing"):
        if k in rep and not rep[k]:
            bad.append(k)
    for L, s in rep.get("segments", {}).items():
        for k in ("bounds", "intervals", "boundary_rows"):
            if not s[k]:
                bad.append(f"segments L={L} {k}")
    for n, e in enumerate(rep.get("mttkrp_rel_err", [])):
        if not e <= REL_FP64:
            bad.append(f"mttkrp mode {n} rel err {e}")
    for key in ("cp_als", "cp_als_plain"):
        als = rep.get(key)
        if als:
            if not als["fit_abs_err"] <= REL_FP64:
                bad.append(f"{key} fit err {als['fit_abs_err']}")
            if not als["weights_rel_err"] <= REL_FP64:
                bad.append(f"{key} weights err {als['weights_rel_err']}")
            if not max(als["factors_rel_err"]) <= REL_FP64:
                bad.append(f"{key} factors err {als['factors_rel_err']}")
    apr = rep.get("cp_apr")
    if apr:
        if not apr["inner_iters_identical"]:
            bad.append(f"cp_apr inner iteration flips {apr['flips']}")
        for k in ("kkt_rel_err", "loglik_rel_err", "weights_rel_err"):
            if apr[k] is None or not apr[k] <= REL_FP64:
                bad.append(f"cp_apr {k} {apr[k]}")
        if not max(apr["factors_rel_err"]) <= REL_FP64:
            bad.append(f"cp_apr factors err {apr['factors_rel_err']}")
    return bad


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=list(CHECKS))
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    reports = []
    for name in args.names:
        rep = run(name)
        rep["failures"] = failures(rep)
        reports.append(rep)
        print(json.dumps(rep), flush=True)
    if args.json:
        Path(args.json).write_text(json.dumps(reports, indent=1) + "\n")
    return 0 if all(not r["failures"] for r in reports) else 1


if __name__ == "__main__":
    sys.exit(main())
