"""A/B of the interleaved (bulk-copy staged) decoded views against the
per-lane cp.async staging: plain MTTKRP per mode and the memo piece sums.
usage: python tools/il_ab.py c2 [c4 ...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06348_b200 as alto
from paper_2403_06348_b200 import synthetic, kernels as K, _native as nat
from paper_2403_06348_b200.partition import il_build


def timed(f, n=10):
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def rel(a, b):
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-300))


for name in [a for a in sys.argv[1:] if not a.startswith("--")]:
    cfg = synthetic.CONFIGS[name]
    c, v = synthetic.generate(cfg, seed=0)
    t = alto.AltoTensor.from_device_coo(cfg.dims, c, v); del c, v
    R = cfg.rank
    d = K.DeviceFactors([torch.rand((n, R), dtype=torch.float64, device="cuda") for n in cfg.dims], R)
    for mode in ([] if "--sums-only" in sys.argv else range(len(cfg.dims))):
        out = torch.zeros((cfg.dims[mode], nat.padded_ld(R)), dtype=torch.float64, device="cuda")
        os.environ["ALTO_B200_IL"] = "0"
        f0 = lambda: K.launch_mttkrp(t, d, mode, "dview", out=out)
        ref = K.launch_mttkrp(t, d, mode, "dview").clone()
        ms0 = timed(f0)
        os.environ["ALTO_B200_IL"] = "1"
        got = K.launch_mttkrp(t, d, mode, "dview").clone()
        ms1 = timed(f0)
        print(json.dumps({"cfg": name, "mode": mode, "dview_ms": round(ms0, 4), "dview_il_ms": round(ms1, 4),
                          "rel": rel(got, ref)}), flush=True)
        t._cache.clear(); torch.cuda.empty_cache()
    if name == "c2" or (len(cfg.dims) == 3 and "--memo" in sys.argv):
        os.environ["ALTO_B200_MEMO_SPLIT"] = "1"
        from paper_2403_06348_b200.memo import MemoPlan
        for (m0, m1) in ((0, 1), (1, 2), (2, 0)):
            os.environ["ALTO_B200_MEMO_IL"] = "0"
            p = MemoPlan(t, R, m0, m1)
            ak = d.mats[p.k]
            sums = lambda: nat.call("alto_memo_sums", nat.ptr(p.pieceid), nat.ptr(p.crd[1 - p.jplane]),
                                    nat.ptr(p.vals), t.nnz, nat.ptr(ak), ak.stride(0), R, nat.ptr(p.T),
                                    p.T.stride(0), nat.stream_ptr())
            sums(); torch.cuda.synchronize(); T0 = p.T.clone()
            ms0 = timed(sums)
            ipid = il_build(None, p.pieceid, p.vals, t.nnz, R, 1)[1]
            _r, icrd, ivals = il_build(None, p.crd[1 - p.jplane], p.vals, t.nnz, R, 1)
            sums_il = lambda: nat.call("alto_memo_sums_il", nat.ptr(ipid), nat.ptr(icrd), nat.ptr(ivals), t.nnz,
                                       nat.ptr(ak), ak.stride(0), R, nat.ptr(p.T), p.T.stride(0), nat.stream_ptr())
            p.T.zero_(); sums_il(); torch.cuda.synchronize()
            r = rel(p.T[:, :R], T0[:, :R])
            ms1 = timed(sums_il)
            n = __import__("ctypes").c_int64(0)
            nat.call("alto_il_length", t.nnz, R, __import__("ctypes").byref(n))
            kf = torch.empty(n.value, dtype=torch.int32, device="cuda")
            fv = torch.empty(n.value, dtype=torch.float64, device="cuda")
            nat.call("alto_memo_sums_stream", nat.ptr(p.rows), nat.ptr(p.crd[p.jplane]), nat.ptr(p.crd[1 - p.jplane]),
                     nat.ptr(p.vals), t.nnz, R, nat.ptr(kf), nat.ptr(fv), nat.stream_ptr())
            fast = lambda: nat.call("alto_memo_sums_fast", nat.ptr(kf), nat.ptr(fv), t.nnz, nat.ptr(p.pbase),
                                    nat.ptr(ak), ak.stride(0), R, nat.ptr(p.T), p.T.stride(0), nat.stream_ptr())
            p.T.zero_(); fast(); torch.cuda.synchronize()
            r2 = rel(p.T[:, :R], T0[:, :R])
            ms2 = timed(fast)
            print(json.dumps({"cfg": name, "pair": [m0, m1], "P": p.P, "sums_ms": round(ms0, 4),
                              "sums_il_ms": round(ms1, 4), "rel": r, "sums_fast_ms": round(ms2, 4),
                              "rel_fast": r2}), flush=True)
            # split: fast sums + T-order memo1 vs fused (sums + own MTTKRP) vs memo0
            out0 = torch.zeros((cfg.dims[m0], nat.padded_ld(R)), dtype=torch.float64, device="cuda")
            a1 = d.mats[m1]
            def split():
                fast()
                out0.zero_()
                nat.call("alto_mttkrp_memo1", nat.ptr(p.nrow), nat.ptr(p.ncrd), None, nat.ptr(p.T), p.T.stride(0),
                         p.P, nat.ptr(a1), a1.stride(0), R, nat.ptr(out0), out0.stride(0), nat.stream_ptr())
            split(); torch.cuda.synchronize(); O0 = out0.clone()
            ms_split = timed(split)
            fr = torch.empty(n.value, dtype=torch.int32, device="cuda")
            fj_ = torch.empty(n.value, dtype=torch.int32, device="cuda")
            fk_ = torch.empty(n.value, dtype=torch.int32, device="cuda")
            nat.call("alto_memo_fused_stream", nat.ptr(p.rows), nat.ptr(p.crd[p.jplane]), nat.ptr(p.crd[1 - p.jplane]),
                     nat.ptr(p.vals), t.nnz, R, nat.ptr(fr), nat.ptr(fj_), nat.ptr(fk_), nat.ptr(fv), nat.stream_ptr())
            def fused():
                out0.zero_()
                nat.call("alto_memo_fused", nat.ptr(fr), nat.ptr(fj_), nat.ptr(fk_), nat.ptr(fv), t.nnz, nat.ptr(a1),
                         a1.stride(0), nat.ptr(ak), ak.stride(0), R, nat.ptr(p.pbase), nat.ptr(p.T), p.T.stride(0),
                         nat.ptr(out0), out0.stride(0), nat.stream_ptr())
            p.T.zero_(); fused(); torch.cuda.synchronize()
            rf_t, rf_o = rel(p.T[:, :R], T0[:, :R]), rel(out0[:, :R], O0[:, :R])
            ms_fused = timed(fused)
            print(json.dumps({"cfg": name, "pair": [m0, m1], "split_ms": round(ms_split, 4),
                              "fused_ms": round(ms_fused, 4), "rel_T": rf_t, "rel_out": rf_o}), flush=True)
            del fr, fj_, fk_
            if "--no-hot" in sys.argv:
                del kf, fv
                continue
            import ctypes as C
            cap = C.c_int32(0)
            nat.call("alto_memo_hot_capacity", R, C.byref(cap))
            kc = p.crd[1 - p.jplane][: t.nnz].long()
            dk = cfg.dims[p.k]
            cnt = torch.bincount(kc, minlength=dk)
            for H in sorted({min(int(x), cap.value) for x in (0, 256, 512, cap.value)}):
                top = torch.topk(cnt, H).indices if H > 0 else torch.empty(0, dtype=torch.long, device="cuda")
                share = float(cnt[top].sum() / cnt.sum()) if H > 0 else 0.0
                slot = torch.full((dk,), -1, dtype=torch.int32, device="cuda")
                slot[top] = torch.arange(H, dtype=torch.int32, device="cuda")
                hot = top.to(torch.int32).contiguous()
                nat.call("alto_memo_sums_hot_stream", nat.ptr(p.rows), nat.ptr(p.crd[p.jplane]),
                         nat.ptr(p.crd[1 - p.jplane]), nat.ptr(p.vals), nat.ptr(slot), t.nnz, R, nat.ptr(kf),
                         nat.ptr(fv), nat.stream_ptr())
                hotf = lambda: nat.call("alto_memo_sums_hot", nat.ptr(kf), nat.ptr(fv), t.nnz, nat.ptr(p.pbase),
                                        nat.ptr(ak), ak.stride(0), R, nat.ptr(hot) if H else None, H, nat.ptr(p.T),
                                        p.T.stride(0), nat.stream_ptr())
                p.T.zero_(); hotf(); torch.cuda.synchronize()
                r3 = rel(p.T[:, :R], T0[:, :R])
                ms3 = timed(hotf)
                print(json.dumps({"cfg": name, "pair": [m0, m1], "H": H, "hot_share": round(share, 4),
                                  "sums_hot_ms": round(ms3, 4), "rel": r3}), flush=True)
            del kf, fv
            del p, ipid, icrd, ivals; torch.cuda.empty_cache()
