"""Oracle restatement of the reference attention path (TEST INFRASTRUCTURE).

* `OracleMeta` — query addressing of attention.py:51-110 (decode / self /
  suffix constructors with the same validation).
* `streaming_attention` — the tile kernel of attention.py:259-329: flat-view
  tiles of `page_size` slots, EMPTY tiles skipped, running-max online softmax
  with the correction/probability update order of attention.py:299-323, so on
  the same BLAS it reproduces the reference bit-for-bit.  Tile
  classification (attention.py:171-210) is restated in vectorised form; it
  only decides which tiles are visited, never the arithmetic.
* `dense_attention_f64` — the two-pass float64 oracle of attention.py:389-447,
  extended with grouped-query heads (q head h reads kv head h // G).
* `fold_gqa_queries` / `unfold_gqa_output` — SURVEY.md §8 c-6: run a GQA
  problem through the unmodified MHA reference kernel by folding the G query
  heads of one kv head into G query rows.
* `round_bf16` — SURVEY.md §8 c-5: numpy has no bf16; inputs are rounded to
  bf16 (round-to-nearest-even) and fed to the fp32/fp64 oracles.
"""

from __future__ import annotations

import math

import numpy as np

from .errors import NoAllowedKeys, OutOfRange, ShapeMismatch


def relative_error(actual, expected) -> float:
    """verify.py:40-43: max |a-e| over max |e| (not elementwise)."""
    expected = np.asarray(expected, dtype=np.float64)
    scale = max(float(np.max(np.abs(expected))) if expected.size else 0.0, 1e-30)
    diff = np.abs(np.asarray(actual, dtype=np.float64) - expected)
    return float(diff.max()) / scale if diff.size else 0.0


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (RNE) and return them as fp32."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    bits = a.view(np.uint32).astype(np.uint64)
    lsb = (bits >> 16) & 1
    rounded = ((bits + 0x7FFF + lsb) >> 16) << 16
    nan = np.isnan(a)
    out = rounded.astype(np.uint32).view(np.float32).copy()
    out[nan] = np.nan
    return out


class OracleMeta:
    """attention.py:51-110."""

    def __init__(self, view, q_seq, q_pos):
        self.view = view
        self.q_seq = np.asarray(q_seq, dtype=np.int64)
        self.q_pos = np.asarray(q_pos, dtype=np.int64)
        if self.q_seq.ndim != 1 or self.q_seq.shape != self.q_pos.shape:
            raise ShapeMismatch("q_seq/q_pos must be equal-length vectors")
        if self.q_seq.size:
            if np.any(np.diff(self.q_seq) < 0):
                raise ValueError("q_seq must be non-decreasing")
            if self.q_seq.min() < 0 or self.q_seq.max() >= view.lengths.size:
                raise OutOfRange("q_seq outside view")
            if np.any(self.q_pos < 0) or np.any(self.q_pos >= view.lengths[self.q_seq]):
                raise OutOfRange("q_pos outside sequence")

    @property
    def query_count(self) -> int:
        return int(self.q_seq.size)

    @classmethod
    def decode(cls, view):
        if np.any(view.lengths <= 0):
            raise OutOfRange("decode needs length >= 1")
        return cls(view, np.arange(view.lengths.size), view.lengths - 1)

    @classmethod
    def self_attention(cls, view):
        return cls(view, view.slot_seq.copy(), view.slot_local.copy())

    @classmethod
    def suffix(cls, view, q_lengths):
        ql = np.asarray(q_lengths, dtype=np.int64)
        if ql.shape != view.lengths.shape:
            raise ShapeMismatch("one q length per sequence")
        if np.any(ql < 0) or np.any(ql > view.lengths):
            raise OutOfRange("q length outside sequence")
        seq = np.repeat(np.arange(ql.size), ql)
        pos = np.concatenate([np.arange(n - q, n) for n, q in zip(view.lengths, ql)]) \
            if ql.sum() else np.zeros(0, np.int64)
        return cls(view, seq, pos)


def key_intervals(meta: OracleMeta, causal: bool) -> tuple[np.ndarray, np.ndarray]:
    """Allowed flat-key interval [lo, hi) of every query.

    mask_allow (attention.py:113-134) admits key k for query q iff k is a slot
    of q's sequence, its local index is < len, and (causal) <= q_pos — i.e. a
    contiguous run starting at the sequence's prefix offset."""
    v = meta.view
    lo = v.prefix_sums[meta.q_seq]
    span = meta.q_pos + 1 if causal else v.lengths[meta.q_seq]
    return lo, lo + span


def classify_tiles(meta: OracleMeta, causal: bool, tile: int):
    """0 = EMPTY, 1 = PARTIAL, 2 = FULL per (q-tile, kv-tile) (attention.py:171-210)."""
    nq, nk = meta.query_count, meta.view.total_slots
    n_qb, n_kb = -(-nq // tile), -(-nk // tile)
    kinds = np.zeros((n_qb, n_kb), dtype=np.int8)
    if not n_qb or not n_kb:
        return kinds
    lo, hi = key_intervals(meta, causal)
    k0 = np.arange(n_kb) * tile
    k1 = np.minimum(k0 + tile, nk)
    for qb in range(n_qb):
        a = lo[qb * tile:(qb + 1) * tile, None]
        b = hi[qb * tile:(qb + 1) * tile, None]
        hit = ((a < k1[None]) & (b > k0[None])).any(axis=0)
        full = ((a <= k0[None]) & (b >= k1[None])).all(axis=0)
        kinds[qb] = np.where(full, 2, np.where(hit, 1, 0))
    return kinds


def _online_update(state, scores, values_h, cd):
    """One tile of the running-max softmax, in the operation order of
    attention.py:315-323."""
    m_run, den, acc = state
    m_new = np.maximum(m_run, scores.max(axis=2))
    starved = np.isneginf(m_new)
    with np.errstate(invalid="ignore"):
        corr = np.where(np.isneginf(m_run), 0.0, np.exp(m_run - m_new)).astype(cd, copy=False)
        prob = np.where(starved[:, :, None], 0.0,
                        np.exp(scores - m_new[:, :, None])).astype(cd, copy=False)
    den = den * corr + prob.sum(axis=2)
    acc = acc * corr[:, :, None] + prob @ values_h
    return m_new, den, acc


def streaming_attention(queries, keys_rows, values_rows, meta: OracleMeta, *, scale: float,
                        causal: bool, tile: int, stats: dict | None = None) -> np.ndarray:
    """attention.py:259-329 over flat K/V rows (the paged gather of
    attention.py:236-245 is done by the caller: `keys_rows[i]` is flat slot i).

    Raises NoAllowedKeys for any query whose allowed set is empty
    (attention.py:324-327; the reference's IndexError bug, is not
    reproduced)."""
    q = np.asarray(queries)
    nq, h, d = q.shape
    cd = np.dtype(np.float32) if q.dtype == np.float16 else q.dtype
    out = np.zeros((nq, h, d), dtype=cd)
    if nq == 0:
        return out
    lo, hi = key_intervals(meta, causal)
    if np.any(hi <= lo):
        bad = np.nonzero(hi <= lo)[0].tolist()
        raise NoAllowedKeys(f"queries {bad} have zero allowed keys")
    kinds = classify_tiles(meta, causal, tile)
    nk = meta.view.total_slots
    sc = cd.type(scale)
    if stats is not None:
        stats.setdefault("visited_blocks", 0)
        stats.setdefault("skipped_blocks", 0)
        stats.setdefault("allowed_pairs", 0)
    for qb in range(kinds.shape[0]):
        q0, q1 = qb * tile, min(qb * tile + tile, nq)
        qh = np.ascontiguousarray(q[q0:q1].astype(cd, copy=False).transpose(1, 0, 2))
        bq = q1 - q0
        state = (np.full((h, bq), -np.inf, dtype=cd), np.zeros((h, bq), cd),
                 np.zeros((h, bq, d), cd))
        for kb in range(kinds.shape[1]):
            kind = kinds[qb, kb]
            if kind == 0:
                if stats is not None:
                    stats["skipped_blocks"] += 1
                continue
            k0, k1 = kb * tile, min(kb * tile + tile, nk)
            kh = keys_rows[k0:k1].astype(cd, copy=False).transpose(1, 2, 0)
            s = (qh @ kh) * sc
            if kind == 2:
                n_pairs = bq * (k1 - k0)
            else:
                ks = np.arange(k0, k1)[None, :]
                allow = (lo[q0:q1, None] <= ks) & (ks < hi[q0:q1, None])
                s = np.where(allow[None], s, -np.inf)
                n_pairs = int(allow.sum())
            if stats is not None:
                stats["visited_blocks"] += 1
                stats["allowed_pairs"] += n_pairs
            vh = values_rows[k0:k1].astype(cd, copy=False).transpose(1, 0, 2)
            state = _online_update(state, s, vh, cd)
        _, den, acc = state
        out[q0:q1] = (acc / den[:, :, None]).transpose(1, 0, 2)
    return out


def dense_attention_f64(queries, keys, values, lengths, *, causal=True, scale=None,
                        q_lengths=None) -> np.ndarray:
    """attention.py:389-447: contiguous per-sequence K/V, two-pass float64.

    Grouped-query extension: keys/values may carry Hkv = Hq / G heads; query
    head h reads kv head h // G."""
    q = np.asarray(queries, dtype=np.float64)
    k = np.asarray(keys, dtype=np.float64)
    v = np.asarray(values, dtype=np.float64)
    if q.ndim != 3 or k.ndim != 3 or k.shape != v.shape or q.shape[2] != k.shape[2]:
        raise ShapeMismatch("bad shapes")
    hq, hkv = q.shape[1], k.shape[1]
    if hq % hkv:
        raise ShapeMismatch("query heads must be a multiple of kv heads")
    g = hq // hkv
    if g > 1:
        k = np.repeat(k, g, axis=1)
        v = np.repeat(v, g, axis=1)
    lens = np.asarray(lengths, dtype=np.int64)
    if lens.sum() != k.shape[0]:
        raise ShapeMismatch("lengths do not cover K/V rows")
    ql = lens.copy() if q_lengths is None else np.asarray(q_lengths, dtype=np.int64)
    if ql.sum() != q.shape[0]:
        raise ShapeMismatch("q_lengths do not cover query rows")
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[2])
    out = np.zeros(q.shape, dtype=np.float64)
    qs = ks = 0
    for n, m in zip(lens.tolist(), ql.tolist()):
        if m:
            qq = q[qs:qs + m].transpose(1, 0, 2)
            kk = k[ks:ks + n].transpose(1, 2, 0)
            vv = v[ks:ks + n].transpose(1, 0, 2)
            s = (qq @ kk) * scale
            if causal:
                ok = np.arange(n)[None, :] <= np.arange(n - m, n)[:, None]
                if not ok.any(axis=1).all():
                    raise NoAllowedKeys("empty query row")
                s = np.where(ok[None], s, -np.inf)
            s = np.exp(s - s.max(axis=2, keepdims=True))
            s /= s.sum(axis=2, keepdims=True)
            out[qs:qs + m] = (s @ vv).transpose(1, 0, 2)
        qs += m
        ks += n
    return out


def fold_gqa_queries(q: np.ndarray, hkv: int) -> np.ndarray:
    """[nq, Hq, D] -> [nq*G, Hkv, D]; row (i*G + g) head j is q head j*G + g."""
    nq, hq, d = q.shape
    g = hq // hkv
    return np.ascontiguousarray(q.reshape(nq, hkv, g, d).transpose(0, 2, 1, 3).reshape(nq * g, hkv, d))


def unfold_gqa_output(o: np.ndarray, hq: int) -> np.ndarray:
    """Inverse of fold_gqa_queries on the attention output."""
    rows, hkv, d = o.shape
    g = hq // hkv
    nq = rows // g
    return np.ascontiguousarray(o.reshape(nq, g, hkv, d).transpose(0, 2, 1, 3).reshape(nq, hq, d))


def fold_gqa_meta(meta: OracleMeta, g: int) -> OracleMeta:
    """Repeat every query G times."""
    return OracleMeta(meta.view, np.repeat(meta.q_seq, g), np.repeat(meta.q_pos, g))
