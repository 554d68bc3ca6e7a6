"""C4 prefill timing: K1 append of N prompt tokens + K3 tcgen05 prefill over
the paged cache (Llama-3-8B GQA 32q/8kv x128, bf16, page 16).  Prints one
JSON line per N with device times (CUDA events) and TFLOP/s under the
reference's FLOP convention 4*Hq*D*sum n(n+1)/2 (attention.py:224-226)."""

import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2506_07311_b200 import AttentionConfig, KvStore, MaskMeta, PagePool, _lib  # noqa: E402
from paper_2506_07311_b200.attention import suffix_runs  # noqa: E402
from paper_2506_07311_b200.store import _stream  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="2048,4096,8192")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--out", default="f32", choices=("f32", "bf16"), help="output dtype")
    ap.add_argument("--gathered", action="store_true",
                    help="experiment: contiguous K/V rows without the block table (one TMA box per 128 keys)")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    hq, hkv, d, ps = args.hq, args.hkv, args.d, 16
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    for n in [int(x) for x in args.n.split(",")]:
        B = args.batch
        pool = PagePool(B * (n // ps + 2) + 16, page_size=ps)
        store = KvStore(pool, hkv, d, dtype=torch.bfloat16, device=dev)
        for b in range(B):
            pool.reserve(b, n)
        cfg = AttentionConfig(head_count=hq, head_dim=d, page_size=ps, kv_head_count=hkv)
        k = torch.randn((B * n, hkv, d), device=dev).bfloat16()
        v = torch.randn((B * n, hkv, d), device=dev).bfloat16()
        for b in range(B):
            store.assign(b, np.arange(n), k[b * n:(b + 1) * n], v[b * n:(b + 1) * n])
        meta = MaskMeta.self_attention(store.batch_view(list(range(B))))
        q = torch.randn((B * n, hq, d), device=dev).bfloat16()
        out = torch.empty((B * n, hq, d), device=dev, dtype=torch.float32 if args.out == "f32" else torch.bfloat16)
        runs = suffix_runs(meta)
        rows = np.asarray([pool.table(b).mirror_row for b in range(B)], dtype=np.int32)
        if args.gathered:
            ent = [np.asarray(pool.table(b).entries) for b in range(B)]
            assert all((np.diff(e) == 1).all() for e in ent), "pages not contiguous"
            rows = np.asarray([e[0] * ps for e in ent], dtype=np.int32)
        plan = _lib.prefill_plan(runs[0], runs[1], meta.view.lengths, rows, hq, hkv, True)
        dplan = torch.from_numpy(plan).to(dev)
        mirror = pool.device_table(dev)
        lib = _lib.load()
        a = _lib.PrefillArgs(q=q.data_ptr(), total_q=B * n, k_cache=store.keys.data_ptr(),
                             v_cache=store.values.data_ptr(), kv_dtype=_lib.PKV_BF16,
                             cache_rows=store.keys.shape[0],
                             block_table=None if args.gathered else mirror.data_ptr(),
                             bt_stride=0 if args.gathered else mirror.shape[1], page_size=ps, hq=hq, hkv=hkv, head_dim=d,
                             scale=cfg.scale, causal=1, out=out.data_ptr(),
                             out_dtype=_lib.PKV_F32 if args.out == "f32" else _lib.PKV_BF16,
                             plan=dplan.data_ptr(), n_items=plan.shape[0])
        sp = _stream(dev)
        if os.environ.get("PF_DEBUG"):
            dbg = torch.zeros(512 + 4 * plan.shape[0], dtype=torch.int64, device=dev)
            a.debug = dbg.data_ptr()
            _lib.check(lib.pkv_paged_prefill(C.byref(a), sp))
            torch.cuda.synchronize()
            full = dbg.cpu().numpy()
            cta = full[512:].reshape(-1, 4).astype(np.float64)
            t = full[:512].astype(np.float64)
            t0 = min(t[t > 0].min(), cta[:, 0].min())
            span = (cta[:, 2].max() - cta[:, 0].min()) / 1e3
            dur = (cta[:, 2] - cta[:, 0]) / 1e3
            first = (cta[:, 1] - cta[:, 0]) / 1e3
            ntiles = np.maximum(plan[:, 7], plan[:, 8]).astype(np.float64)
            A = np.stack([np.ones_like(ntiles), ntiles], 1)
            coef = np.linalg.lstsq(A, dur, rcond=None)[0]
            nsm = len(np.unique(cta[:, 3]))
            busy = dur.sum() / (span * nsm)
            # idle gap between consecutive CTAs on the same SM
            gaps = []
            for sm in np.unique(cta[:, 3]):
                rr = cta[cta[:, 3] == sm]
                rr = rr[np.argsort(rr[:, 0])]
                gaps += list((rr[1:, 0] - rr[:-1, 2]) / 1e3)
            print(json.dumps({"span_us": round(span, 1), "sms": int(nsm), "busy_frac": round(float(busy), 3),
                              "per_item_us": round(float(coef[0]), 2), "per_tile_us": round(float(coef[1]), 3),
                              "first_S_us_median": round(float(np.median(first)), 2),
                              "gap_us_median": round(float(np.median(gaps)), 2) if gaps else None,
                              "tail_us": round(float((cta[:, 2].max() - np.percentile(cta[:, 2], 50)) / 1e3), 1)}))
            if full[448:464].any():  # -DPKV_K3_PHASES build: clocks per softmax phase, CTA 0 row 0
                ph = full[448:464].reshape(2, 8)[:, :5]
                nt0 = int(max(plan[0, 7], plan[0, 8]))
                print("softmax phase clk/tile (wait S, tmem ld, max, exp+st, publish):",
                      [[round(x / max(nt0, 1)) for x in row] for row in ph.tolist()])
            rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
            print("item 0:", plan[0].tolist())
            for name, off in (("S_A ready", 0), ("S_B ready", 64), ("P_A done", 128), ("P_B done", 192),
                              ("PV_A issue", 256), ("PV_B issue", 320), ("K ready", 384)):
                print("%-10s" % name, " ".join("%6.2f" % x for x in rel[off:off + 24]))
            a.debug = None
        for _ in range(3):
            _lib.check(lib.pkv_paged_prefill(C.byref(a), sp))
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.iters)]
        for s, e in ev:
            s.record()
            lib.pkv_paged_prefill(C.byref(a), sp)
            e.record()
        torch.cuda.synchronize()
        ms = sorted(s.elapsed_time(e) for s, e in ev)
        med = ms[len(ms) // 2]
        # append timing (K1 over the whole prompt)
        pos = np.arange(n)
        ta = []
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            store.assign(0, pos, k[:n], v[:n])
            e.record()
            torch.cuda.synchronize()
            ta.append(s.elapsed_time(e))
        flops = 4 * hq * d * B * n * (n + 1) // 2
        tf = flops / (med * 1e-3) / 1e12
        print(json.dumps({"n": n, "batch": B, "items": int(plan.shape[0]), "prefill_ms": med,
                          "tflops": round(tf, 1), "frac_of_sustained": round(tf / peaks["bf16_tflops_sustained"], 3),
                          "append_ms": min(ta), "append_gbs": round(4 * n * hkv * d * 2 / (min(ta) * 1e-3) / 1e9, 1)}))
        sys.stdout.flush()


if __name__ == "__main__":
    main()
