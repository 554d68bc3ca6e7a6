"""Seeded toy decoder that drives the decode loop in tests (TEST
INFRASTRUCTURE; the model itself is out of scope — SURVEY.md §2.1 row 7).

Restates the reference's desk-scale model (pkg/src/pagedkv/decoder.py:31-194)
so the GPU tests can run the repo's DecodeSession (the hot path's caller,
decoder.py:196-287) on the box, where /root/reference is absent:
  * weights drawn from default_rng(seed) in the reference's order
    (token embedding; per layer ln1, ln2, wq, wk, wv, wo, w1, w2; final norm;
    unembedding — decoder.py:114-141);
  * pre-norm residual blocks, ReLU MLP, sinusoidal positions (decoder.py:72-108,
    143-179), dense causal no-cache forward (decoder.py:79-92, 181-194).
Pinned against tests/golden/decoder_cases.npz (made by the real reference).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class ToyConfig:
    layers: int = 2
    head_count: int = 4
    head_dim: int = 16
    vocab: int = 256
    seed: int = 0
    mlp_ratio: int = 4

    @property
    def d_model(self) -> int:
        return self.head_count * self.head_dim


def layer_norm(x, gain, bias):
    mu = x.mean(axis=-1, keepdims=True)
    var = x.var(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + 1e-5) * gain + bias


def sinusoid(positions, width):
    pos = np.asarray(positions, dtype=np.float64)[:, None]
    freqs = np.exp(-np.log(10000.0) * np.arange(width // 2, dtype=np.float64) * 2.0 / width)
    ang = pos * freqs[None, :]
    out = np.empty((pos.shape[0], width), dtype=np.float32)
    out[:, 0::2] = np.sin(ang)
    out[:, 1::2] = np.cos(ang)
    return out


class ToyDecoder:
    def __init__(self, config: ToyConfig):
        self.config = config
        rng = np.random.default_rng(config.seed)
        d, hid = config.d_model, config.mlp_ratio * config.d_model

        def dense(d_in, d_out):
            return (rng.standard_normal((d_in, d_out)) / np.sqrt(d_in)).astype(np.float32)

        def norm():
            g = (1.0 + 0.05 * rng.standard_normal(d)).astype(np.float32)
            b = (0.05 * rng.standard_normal(d)).astype(np.float32)
            return g, b

        self.tok_embed = rng.standard_normal((config.vocab, d)).astype(np.float32)
        self.blocks = []
        for _ in range(config.layers):
            ln1 = norm()
            ln2 = norm()
            blk = {"ln1": ln1, "ln2": ln2}
            for key in ("wq", "wk", "wv", "wo"):
                blk[key] = dense(d, d)
            blk["w1"] = dense(d, hid)
            blk["w2"] = dense(hid, d)
            self.blocks.append(blk)
        self.ln_f = norm()
        self.unembed = dense(d, config.vocab)

    # -- the interface DecodeSession drives (decoder.py:143-179) --------------
    def embed(self, tokens, positions):
        return self.tok_embed[np.asarray(tokens, dtype=np.int64)] + sinusoid(positions, self.config.d_model)

    def _qkv(self, block, x_norm, counter=None):
        c = self.config
        n = x_norm.shape[0]
        return tuple((x_norm @ block[w]).reshape(n, c.head_count, c.head_dim) for w in ("wq", "wk", "wv"))

    def _finish_block(self, block, x, attn_rows, counter=None):
        n = x.shape[0]
        x = x + np.asarray(attn_rows).reshape(n, self.config.d_model).astype(np.float32) @ block["wo"]
        h = np.maximum(layer_norm(x, *block["ln2"]) @ block["w1"], 0.0)
        return x + h @ block["w2"]

    def _logits(self, x_last, counter=None):
        return (layer_norm(x_last, *self.ln_f) @ self.unembed)[0]

    def forward_nocache(self, tokens):
        """Dense causal recompute of the whole prefix (decoder.py:79-92, 181-194)."""
        n = len(tokens)
        x = self.embed(tokens, np.arange(n))
        scale = np.float32(1.0 / np.sqrt(self.config.head_dim))
        for blk in self.blocks:
            q, k, v = self._qkv(blk, layer_norm(x, *blk["ln1"]))
            s = np.einsum("qhd,khd->hqk", q, k) * scale
            s = s + np.triu(np.full((n, n), -np.inf, dtype=np.float32), 1)
            s = s - s.max(axis=2, keepdims=True)
            p = np.exp(s)
            p /= p.sum(axis=2, keepdims=True)
            x = self._finish_block(blk, x, np.einsum("hqk,khd->qhd", p, v))
        return self._logits(x[-1:])


def load_cases(path):
    data = dict(np.load(path))
    names = sorted({k.rsplit("_", 1)[0] for k in data})
    cases = []
    for name in names:
        layers, heads, hd, vocab, seed, n_prompt, steps, ps = (int(x) for x in data[name + "_meta"])
        cases.append({
            "name": name, "config": ToyConfig(layers=layers, head_count=heads, head_dim=hd, vocab=vocab, seed=seed),
            "tokens": data[name + "_tokens"], "logits": data[name + "_logits"],
            "nocache": data[name + "_nocache"], "n_prompt": n_prompt, "steps": steps, "page_size": ps,
        })
    return cases
