"""Benchmark of the paged-attention hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config auto|c2|c3|c5] [--context L] [--batch B]
                    [--fragment] [--sweep]

One step = one decode step of one attention layer: every sequence appends
one token (K1, fused into the decode launch) and attends over its whole
context (K2-TC split-K flash decode, merge in-kernel).

Workload.  `--config auto` (default) is C2 at one GPU — BASELINE.json
configs[1], LLaMA-7B MHA 32x128 bf16, batch 32, contexts 128-2048 (seed-0
draw, sum 36,477), page 16 — and C5 at N > 1 GPUs — configs[4], 512
sequences with log-uniform contexts 128-32k split over the ranks by LPT
(strong scaling, no data-path collective).  The N = 1 line also carries the
C5 point (`c5`) so the C5 scaling series starts at one GPU, and the C4
prefill side measurement (`prefill_c4`).

Keys of the JSON line (rank 0 prints ONE line):
* `value`     whole-job KV-read GB/s, inputs resident in HBM, CUDA events on
              the launching stream per step, L2 flushed between steps, time =
              max over ranks;
* `e2e`       the same metric through the public API (`DecodeBatch.step`):
              pinned host q/k/v in, pinned host output back, page grants of
              the allocator included (tables are NOT pre-grown);
* `roofline`  the dominant kernel (decode_tc_kernel) against MEASURED_PEAKS;
* `parity_checked` the last timed step re-checked on >= 32 sampled
              sequences: appended K/V rows bit-exact, outputs vs float64;
* `cpu_baseline` the reference's CPU implementation (the real `pagedkv`
              package installed in baseline/_ref; the oracle port if absent)
              on a bounded sample of the same workload.

`--gpus N` without WORLD_SIZE re-launches itself under torch.distributed.run
with N ranks (the driver's form); with fewer GPUs than ranks the ranks share
devices and the timing barrier uses gloo (a plumbing check, not a number).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode attn KV-read GB/s (% of 8 TB/s) and tokens/sec vs context 128-32k, 1/2/4/8 GPU"
NOMINAL_HBM_GBS = 8000.0
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="auto", choices=["auto", "c2", "c3", "c5"])
    ap.add_argument("--context", type=int, default=8192, help="c3 context length")
    ap.add_argument("--batch", type=int, default=16, help="c3 batch")
    ap.add_argument("--fragment", action="store_true",
                    help="block tables over a random permutation of the pool's pages (long-running pool)")
    ap.add_argument("--sweep", action="store_true", help="also run the C3 context sweep (JSON lines on stderr)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-prefill", action="store_true", help="skip the C4 prefill (K3) side measurement")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 point of the N=1 line")
    ap.add_argument("--no-check", action="store_true", help="skip the parity check of the last timed step")
    ap.add_argument("--waves", type=int, default=0, help="split planner target waves (0 = default)")
    ap.add_argument("--heads", default="", help="experiment: override query:kv heads, e.g. 32:32")
    return ap.parse_args(argv)


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------

def resolve_config(args, world: int) -> str:
    return ("c5" if world > 1 else "c2") if args.config == "auto" else args.config


def workload(config: str, rank: int, world: int, *, batch=None, context=None, heads=""):
    """(name, lengths of this rank, hq, hkv, d, ps) of a named config."""
    from paper_2506_07311_b200.sharding import lpt_partition
    from paper_2506_07311_b200.workloads import CONFIG_SHAPES, config_lengths

    if config == "c3":
        lengths = config_lengths("c3", batch=batch, context=context)
        name = f"C3 Llama-3-8B GQA 32q/8kv x128 bf16 decode, batch {batch}, context {context}, page 16"
    elif config == "c5":
        all_lens = config_lengths("c5")
        lengths = [all_lens[i] for i in lpt_partition(all_lens, world)[rank]]
        name = ("C5 request-sharded decode, 512 sequences, contexts 128-32k (seed 0, LPT shards), "
                "GQA 32q/8kv x128 bf16, page 16")
    else:
        lengths = config_lengths("c2")
        name = "C2 LLaMA-7B MHA 32x128 bf16 decode, batch 32, mixed contexts 128-2048 (seed 0), page 16"
    hq, hkv, d, ps, _ = CONFIG_SHAPES[config]
    if heads:  # experiment override "HQ:HKV" (not a BASELINE config)
        hq, hkv = (int(x) for x in heads.split(":"))
        name += f" [heads overridden to {hq}q/{hkv}kv]"
    return name, lengths, hq, hkv, d, ps


def algorithmic_bytes(lengths, hq, hkv, d, ps, s=2, out_bytes=4):
    """KV + Q + O + block-table + length bytes of one step."""
    B = len(lengths)
    kv = sum(2 * n * hkv * d * s for n in lengths)
    return kv + B * hq * d * s + B * hq * d * out_bytes + 4 * sum(-(-n // ps) for n in lengths) + 4 * B, kv


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML)
# ---------------------------------------------------------------------------

class ClockSampler:
    REASONS = {
        0x0000000000000002: "applications_clocks_setting", 0x0000000000000004: "sw_power_cap",
        0x0000000000000008: "hw_slowdown", 0x0000000000000010: "sync_boost",
        0x0000000000000020: "sw_thermal_slowdown", 0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown", 0x0000000000000100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _sample(self):
        nv = self._nv
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
            mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            for bit, name in self.REASONS.items():
                if mask & bit:
                    self.reasons.add(name)
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.0005)

    def __enter__(self):
        if self._nv is not None:
            self._sample()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()
            self._sample()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


class L2Flush:
    """Between timed steps: READ 4x L2 of unrelated data so the next step
    starts with a cold, clean L2 (a write flush would leave dirty lines whose
    write-back steals HBM bandwidth from the timed kernel).  4x (~80 us of
    GPU time) also keeps the host's launch of the next step ahead of the GPU,
    so short steps do not time the host's issue latency."""

    def __init__(self, device):
        import torch

        l2 = torch.cuda.get_device_properties(device).L2_cache_size
        self.buf = torch.ones(max(4 * l2, 512 << 20) // 4, dtype=torch.float32, device=device)

    def __call__(self):
        self.buf.sum()


# ---------------------------------------------------------------------------
# our implementation: the exact timed call, reusable by the parity tests
# ---------------------------------------------------------------------------

def build_cache(lengths, hq, hkv, d, ps, extra_tokens, device, seed=0, fragment=False, reserve_extra=0):
    """A bf16 paged cache holding `lengths` tokens per sequence (randn K/V),
    tables reserved for `reserve_extra` more tokens, pool room for
    `extra_tokens` more.  Layout: the reference's scatter recipe
    (verify.py:172-194: throw-away reservations interleaved with the real
    ones, then freed), or with `fragment` every table over a random
    permutation of the live pages (a long-running pool)."""
    import torch

    from paper_2506_07311_b200 import AttentionConfig, KvStore, PagePool

    B = len(lengths)
    need = sum(-(-(n + extra_tokens) // ps) for n in lengths)
    pad = max(B, need // 8)
    pool = PagePool(need + pad + B + 8, page_size=ps)
    store = KvStore(pool, hkv, d, dtype=torch.bfloat16, device=device)
    for b, n in enumerate(lengths):
        pool.reserve(("pad", b), ps * (1 + (b * 7919) % max(1, pad // B)))
        pool.reserve(b, n + reserve_extra)
    for b in range(B):
        pool.free(("pad", b))
    if fragment:
        live = [list(pool.table(b).entries) for b in range(B)]
        flat = np.concatenate([np.asarray(e, dtype=np.int64) for e in live])
        perm = np.random.default_rng(1000 + seed).permutation(flat)
        off = 0
        for b, e in enumerate(live):
            pool.table(b).entries[:] = perm[off:off + len(e)].tolist()
            off += len(e)
    gen = torch.Generator(device=device).manual_seed(seed)
    chunk = 1 << 15
    for b, n in enumerate(lengths):
        pool.table(b).logical_len = 0
        for s0 in range(0, n, chunk):
            m = min(chunk, n - s0)
            k = torch.randn((m, hkv, d), generator=gen, device=device, dtype=torch.bfloat16)
            v = torch.randn((m, hkv, d), generator=gen, device=device, dtype=torch.bfloat16)
            store.assign(b, np.arange(s0, s0 + m), k, v)
    return pool, store, AttentionConfig(head_count=hq, head_dim=d, page_size=ps, kv_head_count=hkv)


class DecodeBench:
    """One rank's decode benchmark: a scattered (or fragmented) bf16 paged
    cache holding `lengths` tokens, per-step q / k_new / v_new resident in
    HBM, the host plan and metadata of every step precomputed, and ONE C-ABI
    call per step (pkv_paged_attention with the fused append).
    tests/test_gpu_bench_parity.py drives this same object."""

    def __init__(self, lengths, hq, hkv, d, ps, *, total_steps, device, seed=0, fragment=False, waves=0,
                 e2e_steps=None):
        import torch

        from paper_2506_07311_b200 import AttentionConfig, _lib
        from paper_2506_07311_b200.attention import _Workspace

        self.lengths, self.hq, self.hkv, self.d, self.ps = list(lengths), hq, hkv, d, ps
        self.B = B = len(lengths)
        self.device, self.total_steps, self.fragment = device, total_steps, fragment
        # tables cover the device phase; the pool keeps room for the e2e
        # phase's page grants
        e2e_steps = total_steps if e2e_steps is None else e2e_steps
        self.pool, self.store, _ = build_cache(lengths, hq, hkv, d, ps, extra_tokens=total_steps + e2e_steps + 2,
                                               device=device, seed=seed, fragment=fragment,
                                               reserve_extra=total_steps + 1)
        pool, store = self.pool, self.store
        self.cfg = AttentionConfig(head_count=hq, head_dim=d, page_size=ps, kv_head_count=hkv)
        self.lib = lib = _lib.load()
        self.mirror = mirror = pool.device_table(device)
        rows = np.asarray([pool.table(b).mirror_row for b in range(B)], dtype=np.int32)
        self.base = base = np.asarray(lengths, dtype=np.int32)
        gen2 = torch.Generator(device=device).manual_seed(1234 + seed)
        T = total_steps
        self.qs = torch.randn((T, B, hq, d), generator=gen2, device=device, dtype=torch.bfloat16)
        self.ks = torch.randn((T, B, hkv, d), generator=gen2, device=device, dtype=torch.bfloat16)
        self.vs = torch.randn((T, B, hkv, d), generator=gen2, device=device, dtype=torch.bfloat16)
        # per-step metadata [q_seq | key counts | mirror rows | host work plan];
        # key counts grow by one per step (the appended token is attended)
        self.plans = [_lib.attention_plan(base + t + 1, rows, ps, hq, hkv, waves, head_dim=d) for t in range(T)]
        width = 3 * B + max(pl.size for pl in self.plans)
        meta_np = np.zeros((T, width), dtype=np.int32)
        for t in range(T):
            row_t = np.concatenate([np.arange(B, dtype=np.int32), base + t + 1, rows, self.plans[t]])
            meta_np[t, :row_t.size] = row_t
        self.meta = torch.from_numpy(meta_np).to(device)
        self.out = torch.empty((B, hq, d), dtype=torch.float32, device=device)
        self.ws = _Workspace.get(device, lib.pkv_attention_workspace_bytes(B, hq, d))
        self.stream = torch.cuda.current_stream(device)
        self._sp = C.c_void_p(self.stream.cuda_stream)
        self._args = [self._make_args(t) for t in range(T)]
        self.last_step = -1
        torch.cuda.synchronize(device)

    def _make_args(self, t):
        from paper_2506_07311_b200 import _lib

        md = self.meta[t].data_ptr()
        B = self.B
        return _lib.AttentionArgs(
            q=self.qs[t].data_ptr(), q_dtype=_lib.PKV_BF16, n_queries=B, q_seq=md, q_nkeys=md + 4 * B,
            k_cache=self.store.k_cache.data_ptr(), v_cache=self.store.v_cache.data_ptr(), kv_dtype=_lib.PKV_BF16,
            block_table=self.mirror.data_ptr(), bt_stride=self.mirror.shape[1], seq_row=md + 8 * B,
            seq_start=None, page_size=self.ps, hq=self.hq, hkv=self.hkv, head_dim=self.d, scale=self.cfg.scale,
            out=self.out.data_ptr(), out_dtype=_lib.PKV_F32, workspace=self.ws.data_ptr(),
            workspace_bytes=self.ws.numel(), num_sms=0, target_waves=0, prof_start=None, prof_stop=None,
            mode=0, k_new=self.ks[t].data_ptr(), v_new=self.vs[t].data_ptr(),
            plan=md + 12 * B, plan_host=self.plans[t].ctypes.data)

    def step(self, t, prof=None):
        """Decode step t: ONE native call (fused K1 append + K2-TC decode)."""
        from paper_2506_07311_b200 import _lib

        a = self._args[t]
        a.prof_start, a.prof_stop = (prof[0].cuda_event, prof[1].cuda_event) if prof else (None, None)
        st = self.lib.pkv_paged_attention(C.byref(a), self._sp)
        if st:
            _lib.check(st, "pkv_paged_attention")
        self.last_step = t

    def run(self, W, K, flush, barrier=None):
        """W untimed + K timed steps (L2 flushed before each), then K more
        steps whose decode launch alone is bracketed by events on the
        launching stream (the roofline's per-launch time; kept out of the
        timed steps, whose events would otherwise nest).  Needs
        total_steps >= W + 2K.  Returns the step and launch times and the
        clock record of the timed steps."""
        import torch

        assert self.total_steps >= W + 2 * K, "DecodeBench needs total_steps >= W + 2K"
        prof = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for a, b in prof:  # materialise the cudaEvent_t handles
            a.record(self.stream)
            b.record(self.stream)
        for t in range(W):
            flush()
            self.step(t)
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        torch.cuda.synchronize(self.device)
        if barrier:
            barrier()
        torch.cuda.synchronize(self.device)
        with ClockSampler(self.device.index) as clocks:
            for i in range(K):
                flush()  # untimed
                starts[i].record(self.stream)
                self.step(W + i)
                ends[i].record(self.stream)
            torch.cuda.synchronize(self.device)
        if barrier:
            barrier()
        for i in range(K):  # launch-only timing pass (same per-step work)
            flush()
            self.step(W + K + i, prof[i])
        torch.cuda.synchronize(self.device)
        step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        kern_ms = [a.elapsed_time(b) for a, b in prof]
        alg = kv = kalg = 0
        for i in range(K):
            a_b, kv_b = algorithmic_bytes([n + W + i + 1 for n in self.lengths], self.hq, self.hkv, self.d, self.ps)
            alg += a_b
            kv += kv_b
            kalg += algorithmic_bytes([n + W + K + i + 1 for n in self.lengths], self.hq, self.hkv, self.d,
                                      self.ps)[0]
        return {"step_ms": step_ms, "kernel_ms": kern_ms, "alg_bytes": alg, "kv_bytes": kv,
                "kernel_alg_bytes": kalg, "tokens": self.B * K, "clocks": clocks.summary(), "launches": K}

    def verify(self, n_sample=32, seed=0):
        """Re-check the last executed step on `n_sample` sequences: every
        appended K/V row (all steps so far) bit-exact in its page, and the
        step's output against a float64 softmax over the sequence's pages
        gathered through the host block table (relative error, the
        reference's metric verify.py:40-43; bar 2e-2 for bf16)."""
        import torch

        t_last = self.last_step
        assert t_last >= 0, "no step executed"
        rng = np.random.default_rng(seed)
        idx = np.arange(self.B) if self.B <= n_sample else np.sort(rng.choice(self.B, n_sample, replace=False))
        g = self.hq // self.hkv
        ps = self.ps
        worst, rows_ok = 0.0, True
        out = self.out
        for b in idx.tolist():
            L = int(self.base[b]) + t_last + 1
            entries = np.asarray(list(self.pool.table(b).entries), dtype=np.int64)
            pos = np.arange(L)
            rows = torch.from_numpy(entries[pos // ps] * ps + pos % ps).to(self.device)
            K = self.store.k_cache.index_select(0, rows)
            V = self.store.v_cache.index_select(0, rows)
            n0 = int(self.base[b])
            rows_ok &= bool(torch.equal(K[n0:L], self.ks[: t_last + 1, b]))
            rows_ok &= bool(torch.equal(V[n0:L], self.vs[: t_last + 1, b]))
            q = self.qs[t_last, b].double()
            kk = K.double().repeat_interleave(g, dim=1)
            vv = V.double().repeat_interleave(g, dim=1)
            s = torch.einsum("hd,khd->hk", q, kk) * self.cfg.scale
            ref = torch.einsum("hk,khd->hd", torch.softmax(s, dim=-1), vv)
            err = float((out[b].double() - ref).abs().max() / ref.abs().max().clamp_min(1e-30))
            worst = max(worst, err)
        return {"sequences": int(idx.size), "max_rel_err": worst, "appended_rows_bit_exact": rows_ok,
                "tol": 2e-2, "ok": bool(rows_ok and worst <= 2e-2), "step": t_last}

    def run_e2e(self, W, K, flush, reduce_max=None):
        """The same metric through the public API: DecodeBatch.step with
        pinned host q/k/v and a pinned host output (one native call per step:
        H2D, allocator grants + copy-on-write + plan, page clears, the fused
        append + decode, the result written into the mapped host output).
        The device phase appended total_steps tokens, so tables continue from
        there and grow through the allocator (page grants are timed)."""
        import torch

        from paper_2506_07311_b200.batch import DecodeBatch

        B, hq, hkv, d = self.B, self.hq, self.hkv, self.d
        for b, n in enumerate(self.lengths):
            self.pool.table(b).logical_len = n + self.total_steps
        # drop capacity beyond the logical length so steps must be granted pages
        batch = DecodeBatch(self.store, list(range(B)), self.cfg)
        rng = np.random.default_rng(7)
        host = [tuple(torch.from_numpy(rng.standard_normal(shape).astype(np.float32)).bfloat16().pin_memory()
                      for shape in ((B, hq, d), (B, hkv, d), (B, hkv, d))) for _ in range(4)]
        out_host = torch.empty((B, hq, d), dtype=torch.float32).pin_memory()
        lens0 = [self.pool.table(b).logical_len for b in range(B)]
        granted0 = self.pool.census().live_pages
        times, launches, h2d, d2h = [], 0, 0, 0
        stream = torch.cuda.current_stream(self.device)
        for i in range(W + K):
            q, k, v = host[i % 4]
            flush()
            torch.cuda.synchronize(self.device)
            t0 = time.perf_counter()
            batch.step(q, k, v, out=out_host)
            stream.synchronize()
            dt = time.perf_counter() - t0
            if os.environ.get("PKV_E2E_STEP_TIMES"):  # diagnostic: per-step wall times
                print(f"e2e step {i}: {dt * 1e6:.1f} us", file=sys.stderr)
            if i >= W:
                times.append(dt)
                launches += batch.last_launches
                h2d += q.nbytes + k.nbytes + v.nbytes + 4 * batch._stage.meta_used
                d2h += out_host.nbytes
        kv = sum(sum(2 * (n + W + i + 1) * hkv * d * 2 for n in lens0) for i in range(K))
        total = sum(times)
        total_max = reduce_max(total) if reduce_max else total
        return {"total_s": total, "total_s_max": total_max, "kv_bytes": kv, "tokens": B * K,
                "h2d_bytes_per_step": h2d // K, "d2h_bytes_per_step": d2h // K,
                "ms_per_step": 1e3 * total_max / K, "gpu_launches": launches,
                "pages_granted": self.pool.census().live_pages - granted0}


# ---------------------------------------------------------------------------
# CPU side: the reference implementation (baseline/_ref) or the oracle port
# ---------------------------------------------------------------------------

def _reference_module():
    """The real reference package installed in baseline/_ref, or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "pagedkv")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import importlib

    try:
        mod = importlib.import_module("pagedkv")
    except Exception:
        return None
    return mod if os.path.abspath(mod.__file__).startswith(os.path.abspath(REF_DIR)) else None


class CpuReference:
    """The reference's CPU decode step (KvStore.assign of one token per
    sequence + paged_attention under a decode meta, store.py:117-150 and
    attention.py:332-354) over `lengths`, fp32 values (bf16-rounded, the
    survey's c-5 restatement; the reference has no bf16).  GQA shapes are
    folded through the reference kernel (SURVEY c-6).  Uses the real package
    from baseline/_ref when installed, else the oracle port (kind 'port')."""

    def __init__(self, lengths, hq, hkv, d, ps, seed=0, steps=64):
        ref = _reference_module()
        self.kind = "reference" if ref is not None else "port"
        self.lengths, self.hq, self.hkv, self.d, self.ps = list(lengths), hq, hkv, d, ps
        rng = np.random.default_rng(seed)
        self.rng = rng

        from oracle.attention import round_bf16

        def bf16(shape):
            return round_bf16(rng.standard_normal(shape).astype(np.float32))

        self.bf16 = bf16
        cap = sum(-(-(n + steps + 1) // ps) for n in lengths) + 8
        if ref is not None:
            self.mod = ref
            self.pool = ref.PagePool(cap, page_size=ps)
            self.store = ref.KvStore(self.pool, hkv, d)
            self.cfg = ref.AttentionConfig(head_count=hkv, head_dim=d, page_size=ps, causal=True)
        else:
            from oracle import OraclePool, OracleStore

            self.mod = None
            self.pool = OraclePool(cap, ps)
            self.store = OracleStore(self.pool, hkv, d)
        for b, n in enumerate(lengths):
            self.pool.reserve(b, n)
            self.store.assign(b, np.arange(n), bf16((n, hkv, d)), bf16((n, hkv, d)))
        self.g = hq // hkv

    def step(self):
        from oracle.attention import fold_gqa_queries

        B, g = len(self.lengths), self.g
        for b in range(B):
            n = self.pool.table(b).logical_len
            self.pool.grow(b, n + 1)
            self.store.assign(b, [n], self.bf16((1, self.hkv, self.d)), self.bf16((1, self.hkv, self.d)))
        q = self.bf16((B, self.hq, self.d))
        qf = fold_gqa_queries(q, self.hkv)  # [B*g, hkv, d]; identity for MHA
        if self.mod is not None:
            view = self.store.batch_view(list(range(B)))
            lens = view.lengths
            meta = self.mod.MaskMeta(view=view, q_seq=np.repeat(np.arange(B), g), q_pos=np.repeat(lens - 1, g))
            return self.mod.paged_attention(qf, self.store, meta, self.cfg)
        from oracle import OracleMeta
        from oracle.attention import fold_gqa_meta, streaming_attention
        from oracle.store import OracleBatchView

        lens = [self.pool.table(b).logical_len for b in range(B)]
        view = OracleBatchView(lens, ids=list(range(B)))
        rows = self.store.view_row_indices(view)
        meta = fold_gqa_meta(OracleMeta.decode(view), g)
        return streaming_attention(qf, self.store.keys[rows], self.store.values[rows], meta,
                                   scale=1.0 / math.sqrt(self.d), causal=True, tile=self.ps)

    def kv_bytes_next(self):
        """bf16-size KV bytes the next step reads (the same numerator as ours)."""
        return sum(2 * (self.pool.table(b).logical_len + 1) * self.hkv * self.d * 2
                   for b in range(len(self.lengths)))


def cpu_baseline(config, args, budget_s=15.0):
    """Bounded CPU reference sample for the N=1 line: whole decode steps of
    the full workload, as many as fit in ~budget_s."""
    name, lengths, hq, hkv, d, ps = workload(config, 0, 1, batch=args.batch, context=args.context)
    ref = CpuReference(lengths, hq, hkv, d, ps)
    ref.step()  # warm-up
    times, kv = [], 0
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < budget_s or not times:
        kv_t = ref.kv_bytes_next()
        t0 = time.perf_counter()
        ref.step()
        times.append(time.perf_counter() - t0)
        kv += kv_t
    total = sum(times)
    return {"value": kv / total / 1e9, "unit": "GB/s", "tokens_per_s": len(lengths) * len(times) / total,
            "cores": _cpu_threads(), "kind": ref.kind, "ms_per_step": 1e3 * total / len(times),
            "sample": (f"{len(times)} whole decode steps of the full {name} ({len(lengths)} sequences): "
                       f"{'the reference pagedkv package (baseline/_ref)' if ref.kind == 'reference' else 'the oracle port of the reference'}"
                       f" KvStore.assign + paged_attention, fp32 values rounded to bf16, numpy/OpenBLAS on "
                       f"{_cpu_threads()} host threads; bytes counted at bf16 size")}


def _cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, world):
    """--impl reference: the reference's CPU path on the host cores, rank 0
    only, on our arm's config and metric."""
    config = resolve_config(args, world)
    name, lengths, hq, hkv, d, ps = workload(config, 0, 1, batch=args.batch, context=args.context)
    sample = "full workload"
    if config == "c5":  # 14 GB of bf16 KV (28 GB fp32): a bounded sample of sequences
        idx = sorted(range(len(lengths)), key=lambda i: lengths[i])[::16]
        lengths = [lengths[i] for i in idx]
        sample = f"every 16th sequence by length ({len(lengths)} of 512)"
    ref = CpuReference(lengths, hq, hkv, d, ps, steps=args.warmup + args.steps + 2)
    times, kv = [], 0
    for i in range(args.warmup + args.steps):
        kv_t = ref.kv_bytes_next()
        t0 = time.perf_counter()
        ref.step()
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            kv += kv_t
    total = sum(times)
    value = kv / total / 1e9
    desc = (f"{sample}; {'reference pagedkv (baseline/_ref)' if ref.kind == 'reference' else 'oracle port'}: "
            f"per step KvStore.assign of one token per sequence + paged_attention (decode meta), fp32 values "
            f"rounded to bf16, {_cpu_threads()} host threads; bytes counted at bf16 size")
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "strong" if config == "c5" else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": name, "sample": sample, "same_config": sample == "full workload"},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": _cpu_threads(), "kind": ref.kind,
                         "sample": desc},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "tokens_per_s": len(lengths) * len(times) / total,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------

def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: copy, read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(config_name, fragment=False):
    """DRAM bytes per decode launch from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_decode_summary.json")
    try:
        with open(path) as f:
            s = json.load(f)
        return s.get(config_name + ("_fragmented" if fragment else ""), {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def read_probe_gbs():
    """Best read-only HBM bandwidth of tools/probes/read_bw.cu on this pool
    (committed JSON lines): context for the read-dominated decode kernel,
    whose roofline denominator stays the driver's read+write copy."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "read_bw.jsonl")) as f:
            vals = [json.loads(x)["read_gbs"] for x in f if x.startswith("{")]
        return max(vals) if vals else None
    except Exception:
        return None


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int:
    """`bench.py --gpus N` outside torchrun: re-run under torch.distributed.run
    with N ranks (one process per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def measure(args, config, rank, world, device, dist_ctx, *, steps, warmup, e2e=True, check=True):
    """Device phase (+ e2e, + parity check) of one config on this rank;
    returns the aggregated numbers (meaningful on rank 0)."""
    import torch

    name, lengths, hq, hkv, d, ps = workload(config, rank, world, batch=args.batch, context=args.context,
                                             heads=args.heads)
    bench = DecodeBench(lengths, hq, hkv, d, ps, total_steps=warmup + 2 * steps, device=device, seed=rank,
                        fragment=args.fragment, waves=args.waves)
    flush = L2Flush(device)
    r = bench.run(warmup, steps, flush, barrier=dist_ctx["barrier"])
    total_ms = sum(r["step_ms"])
    sums = dist_ctx["sum"]([float(r["tokens"]), float(r["kv_bytes"]), float(r["alg_bytes"])])
    res = {"name": name, "B": bench.B, "total_ms_max": dist_ctx["max"](total_ms), "tokens_all": sums[0],
           "kv_all": sums[1], "alg_all": sums[2], "kernel_ms_mean": statistics.mean(r["kernel_ms"]),
           "kernel_alg_bytes_mean": r["kernel_alg_bytes"] / steps, "step_ms_mean": total_ms / steps,
           "clocks": r["clocks"], "launches": r["launches"], "shape": (hq, hkv, d, ps), "lengths": lengths}
    if check:
        v = bench.verify()
        res["check"] = v
        res["check_ok_all"] = dist_ctx["min"](1.0 if v["ok"] else 0.0) > 0.5
    if e2e:
        e = bench.run_e2e(max(3, warmup // 2), steps, flush, reduce_max=dist_ctx["max"])
        esums = dist_ctx["sum"]([float(e["kv_bytes"]), float(e["tokens"])])
        e["value"] = esums[0] / e["total_s_max"] / 1e9
        e["tokens_per_s"] = esums[1] / e["total_s_max"]
        res["e2e"] = e
    del bench
    torch.cuda.empty_cache()
    return res


def line_for(args, config, res, world, peak, peak_src, steps, warmup):
    value = res["kv_all"] / (res["total_ms_max"] / 1e3) / 1e9
    k_ach = res["kernel_alg_bytes_mean"] / (res["kernel_ms_mean"] / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": res["total_ms_max"] / steps, "higher_is_better": True,
        "scaling": "strong" if config == "c5" else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (randn K/V/Q bf16" + (", fragmented pool: random page permutation)" if args.fragment
                                                 else ", scattered pages: reference recipe verify.py:172-194)"),
        "config": {"workload": res["name"], "global_batch": int(res["tokens_all"] / steps),
                   "kv_bytes_per_step": res["kv_all"] / steps, "page_size": res["shape"][3],
                   "parallelism": f"request-sharded x{world}" + (" (LPT, no data-path collective)" if world > 1 else ""),
                   "l2": "flushed between steps (read of 4x L2 of unrelated data)",
                   "fragmented": bool(args.fragment)},
        "pct_of_8TBs": round(100 * value / world / NOMINAL_HBM_GBS, 2),
        "tokens_per_s": res["tokens_all"] / (res["total_ms_max"] / 1e3),
        "roofline": {"bound": "hbm", "kernel": "decode_tc_kernel (K2-TC, K1 append fused)",
                     "achieved": round(k_ach, 1), "peak": peak, "unit": "GB/s", "frac": round(k_ach / peak, 4),
                     "traffic": load_traffic(config, args.fragment), "peak_source": peak_src,
                     "read_probe_gbs": read_probe_gbs(),
                     "frac_of_read_probe": (round(k_ach / read_probe_gbs(), 4) if read_probe_gbs() else None),
                     "kernel_ms_mean": res["kernel_ms_mean"],
                     "kernel_share_of_step": res["kernel_ms_mean"] / res["step_ms_mean"],
                     "algorithmic_bytes_per_launch": res["kernel_alg_bytes_mean"],
                     "algorithmic_bytes": "SURVEY 8 d-2: sum_b 2*L_b*Hkv*D*2 + B*Hq*D*2 (q) + B*Hq*D*4 (out) "
                                          "+ 4*sum_b ceil(L_b/16) (table) + 4*B (lens)"},
        "clocks": res["clocks"],
        "gpu_launches": res["launches"],
    }
    if "check" in res:
        line["parity_checked"] = bool(res["check_ok_all"])
        line["parity"] = res["check"]
    if "e2e" in res:
        e = res["e2e"]
        line["e2e"] = {"value": round(e["value"], 2), "unit": "GB/s",
                       "h2d_bytes_per_step": e["h2d_bytes_per_step"], "d2h_bytes_per_step": e["d2h_bytes_per_step"],
                       "ms_per_step": e["ms_per_step"], "tokens_per_s": e["tokens_per_s"],
                       "gpu_launches": e["gpu_launches"], "pages_granted": e["pages_granted"],
                       "path": "DecodeBatch.step (one pkv_decode_step call): pinned host q/k/v -> H2D, allocator "
                               "grants + plan + metadata upload, page clears, fused append + decode, output into "
                               "pinned host memory; host perf_counter around each step, synchronised"}
    return line


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, world)
        return
    import torch
    import torch.distributed as dist

    ndev = torch.cuda.device_count()
    device = torch.device("cuda", local % max(ndev, 1))
    torch.cuda.set_device(device)
    backend = "nccl" if world > 1 and ndev >= world else "gloo"
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group("gloo")
    import __graft_entry__

    if rank == 0 and not os.path.exists(os.path.join(ROOT, "paper_2506_07311_b200", "libpkv200.so")):
        __graft_entry__.build()

    def _reduce(vals, op):
        if world == 1:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device=device if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=op)
        return t.tolist()

    dist_ctx = {
        "barrier": (lambda: dist.barrier()) if world > 1 else None,
        "max": lambda x: _reduce([x], dist.ReduceOp.MAX)[0] if world > 1 else x,
        "min": lambda x: _reduce([x], dist.ReduceOp.MIN)[0] if world > 1 else x,
        "sum": lambda v: _reduce(v, dist.ReduceOp.SUM) if world > 1 else v,
    }
    if world > 1:
        dist.barrier()
    config = resolve_config(args, world)
    peak, peak_src = load_peaks()
    res = measure(args, config, rank, world, device, dist_ctx, steps=args.steps, warmup=args.warmup,
                  e2e=not args.no_e2e, check=not args.no_check)
    c5 = None
    if world == 1 and config != "c5" and not args.no_c5 and args.config == "auto":
        c5 = measure(args, "c5", rank, world, device, dist_ctx, steps=min(args.steps, 10),
                     warmup=max(3, min(args.warmup, 5)), e2e=not args.no_e2e, check=not args.no_check)
    if rank == 0:
        line = line_for(args, config, res, world, peak, peak_src, args.steps, args.warmup)
        if world > 1:
            line["config"]["backend"] = backend
            line["config"]["devices"] = ndev
            if ndev < world:  # plumbing check only: ranks time-share one device
                line["note"] = (f"{world} ranks on {ndev} device(s): the ranks time-share a GPU, so the "
                                "max-over-ranks time is not a throughput number")
        if c5 is not None:
            line["c5"] = line_for(args, "c5", c5, world, peak, peak_src, min(args.steps, 10),
                                  max(3, min(args.warmup, 5)))
            for k in ("metric", "unit", "higher_is_better", "vs_baseline", "dtype", "data"):
                line["c5"].pop(k, None)
            line["parity_checked"] = bool(line.get("parity_checked", True) and line["c5"].get("parity_checked", True))
        if world == 1 and not args.no_prefill:
            line["prefill_c4"] = prefill_c4(device)
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline(config, args)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            line["cpu_baseline"]["tokens_per_s"] = cb["tokens_per_s"]
            line["cpu_baseline"]["ms_per_step"] = cb["ms_per_step"]
        print(json.dumps(line), flush=True)
        if args.sweep:
            sweep()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def prefill_c4(device, n=8192):
    """Side measurement of BASELINE.json configs[3] (C4): one 8192-token
    Llama-3-8B GQA prompt appended into the paged cache (K1) and attended
    causally by the K3 tcgen05 prefill kernel.  TFLOP/s under the reference
    FLOP convention 4*Hq*D*n(n+1)/2 (attention.py:224-226), CUDA events;
    the fraction is of the measured bf16 BURST peak (an isolated kernel)."""
    import torch

    from paper_2506_07311_b200 import AttentionConfig, KvStore, MaskMeta, PagePool, _lib, paged_attention
    from paper_2506_07311_b200.attention import _launch_prefill, suffix_runs

    hq, hkv, d, ps = 32, 8, 128, 16
    pool = PagePool(n // ps + 8, page_size=ps)
    store = KvStore(pool, hkv, d, dtype=torch.bfloat16, device=device)
    pool.reserve(0, n)
    g = torch.Generator(device=device).manual_seed(4)
    k = torch.randn((n, hkv, d), generator=g, device=device).bfloat16()
    v = torch.randn((n, hkv, d), generator=g, device=device).bfloat16()
    q = torch.randn((n, hq, d), generator=g, device=device).bfloat16()
    cfg = AttentionConfig(head_count=hq, head_dim=d, page_size=ps, kv_head_count=hkv)
    pos = np.arange(n)
    store.assign(0, pos, k, v)
    meta = MaskMeta.self_attention(store.batch_view([0]))
    runs = suffix_runs(meta)
    rows = np.asarray([pool.table(0).mirror_row], dtype=np.int32)
    mirror = pool.device_table(device)

    def kernel_only(ev):
        return _launch_prefill(q, meta, cfg, runs, k=store.k_cache, v=store.v_cache, kv_code=store.dtype_code,
                               bt=mirror, rows=rows, out_dtype=torch.float32, device=device,
                               prof=(ev[0].cuda_event, ev[1].cuda_event) if ev else None)

    for _ in range(3):
        paged_attention(q, store, meta, cfg, precision="prefill")
        kernel_only(None)
    torch.cuda.synchronize(device)
    times, app, kern = [], [], []
    for _ in range(10):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        store.assign(0, pos, k, v)  # K1 over the whole prompt (host validation included)
        e1.record()
        paged_attention(q, store, meta, cfg, precision="prefill")
        e2.record()
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        for x in ev:
            x.record()  # materialise the cudaEvent_t handles
        kernel_only(ev)
        torch.cuda.synchronize(device)
        app.append(e0.elapsed_time(e1))
        times.append(e1.elapsed_time(e2))
        kern.append(ev[0].elapsed_time(ev[1]))
    # K1 alone (the append kernel's roofline): CUDA events around the native
    # range launch only, K and V rows read + written
    from paper_2506_07311_b200.store import _stream as _raw_stream
    lib = _lib.load()
    k1 = []
    row0 = int(pool.table(0).mirror_row)
    for _ in range(10):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        _lib.check(lib.pkv_kv_append_range(k.data_ptr(), v.data_ptr(), n, row0, 0, mirror.data_ptr(),
                                           mirror.shape[1], ps, store.k_cache.data_ptr(), store.v_cache.data_ptr(),
                                           store.row_bytes, _raw_stream(device)), "pkv_kv_append_range")
        ev1.record()
        torch.cuda.synchronize(device)
        k1.append(ev0.elapsed_time(ev1))
    # the same call issued back to back (a model's layers): host planning of
    # call i+1 overlaps kernel i
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(device)
    e0.record()
    for _ in range(10):
        paged_attention(q, store, meta, cfg, precision="prefill")
    e1.record()
    torch.cuda.synchronize(device)
    pipelined_ms = e0.elapsed_time(e1) / 10
    ms = sorted(times)[len(times) // 2]
    kms = sorted(kern)[len(kern) // 2]
    flops = 4 * hq * d * n * (n + 1) // 2
    tf = flops / (kms * 1e-3) / 1e12
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
        burst, sustained = float(peaks["bf16_tflops"]), float(peaks["bf16_tflops_sustained"])
    except Exception:
        burst, sustained = 1590.0, 1400.0
    append_bytes = 2 * 2 * n * hkv * d * 2  # K and V read + written
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm_peak = float(json.load(f)["hbm_gbs"])
    except Exception:
        hbm_peak = 6650.0
    return {"workload": f"C4 causal prefill, 1 x {n} tokens, GQA 32q/8kv x128 bf16, page 16",
            "kernel": "prefill_tc_kernel (K3, tcgen05/TMEM)", "kernel_ms": kms, "tflops": round(tf, 1),
            "frac_of_burst_bf16": round(tf / burst, 3), "frac_of_sustained_bf16": round(tf / sustained, 3),
            "api_ms": ms, "api_tflops": round(flops / (ms * 1e-3) / 1e12, 1),
            "api_pipelined_ms": pipelined_ms, "append_ms": min(app),
            "append_gbs": round(append_bytes / (min(app) * 1e-3) / 1e9, 1),
            "k1_roofline": {"kernel": "kv_append_kernel (K1, contiguous run)", "bound": "hbm",
                            "kernel_ms": sorted(k1)[len(k1) // 2],
                            "algorithmic_bytes": append_bytes,
                            "achieved": round(append_bytes / (sorted(k1)[len(k1) // 2] * 1e-3) / 1e9, 1),
                            "peak": hbm_peak, "unit": "GB/s",
                            "frac": round(append_bytes / (sorted(k1)[len(k1) // 2] * 1e-3) / 1e9 / hbm_peak, 3),
                            "note": "CUDA events around the pkv_kv_append_range launch alone (host launch "
                                    "cost inside the events); bytes = K and V rows read + written"},
            "note": "kernel_ms: CUDA events around the K3 launch; api_ms: one paged_attention() call on an idle "
                    "GPU (host planning + metadata upload + launch + kernel); api_pipelined_ms: the call issued "
                    "10x back to back (host work of a call hidden behind the previous kernel); append: "
                    "KvStore.assign of the prompt (host validation included); FLOPs per the reference convention"}


def sweep():
    """C3 context sweep: one JSON line per (context, batch) on stderr, each
    with its clock record (separate processes, fresh caches)."""
    for ctx in (2048, 4096, 8192, 16384, 32768):
        for b in (1, 4, 8, 16, 32, 64):
            if b * ctx * 4096 > 24 << 30:
                continue
            cmd = [sys.executable, os.path.abspath(__file__), "--config", "c3", "--context", str(ctx),
                   "--batch", str(b), "--steps", "10", "--warmup", "3", "--no-cpu-baseline", "--no-e2e",
                   "--no-prefill", "--no-c5"]
            out = subprocess.run(cmd, capture_output=True, text=True)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else json.dumps(
                {"error": out.stderr[-500:]})
            sys.stderr.write(f"SWEEP {line}\n")


if __name__ == "__main__":
    main()
