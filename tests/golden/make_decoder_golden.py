"""Golden vectors for the FMS-style decode loop (the hot path's caller) by
running the REAL reference (`pagedkv.decoder`, decoder.py:31-355) in the
build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_decoder_golden.py

Writes tests/golden/decoder_cases.npz: for each case the greedy tokens and
per-step logits of `generate(mode="cached")` (prefill + steps through the
reference DecodeSession / paged_attention) and of the no-cache dense path.
The GPU tests replay the same model (tests/toy_decoder.py restates its
seeded weights and forward) through this repo's DecodeSession.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("PAGEDKV_REF", "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from pagedkv import decoder as D  # noqa: E402  (the reference itself)

CASES = [
    # name, config kwargs, prompt, steps, page_size
    ("toy_l2_h4x16_ps16", dict(layers=2, head_count=4, head_dim=16, vocab=256, seed=0), list(range(3, 23)), 40, 16),
    ("toy_l3_h2x32_ps8", dict(layers=3, head_count=2, head_dim=32, vocab=128, seed=7), [5, 9, 2, 77, 31], 30, 8),
]


def main():
    arrays = {}
    for name, kw, prompt, steps, ps in CASES:
        dec = D.ToyDecoder(D.DecoderConfig(**kw))
        # cached path, recording the logits of the prefill and every step
        pool = D.PagePool(-(-(len(prompt) + steps) // ps) + 1, ps)
        cache = D.PagedDecoderCache(dec, pool)
        sess = D.DecodeSession(dec, cache, seq_id="gen")
        logits = [sess.prefill(prompt)]
        tokens = list(prompt)
        for _ in range(steps):
            tokens.append(int(np.argmax(logits[-1])))
            logits.append(sess.step(tokens[-1]))
        res = D.generate(dec, prompt, steps, mode="cached", page_size=ps)
        assert res.tokens == tokens
        nocache = [dec.forward_nocache(tokens[: len(prompt) + i]) for i in range(0, steps, 10)]
        arrays[name + "_tokens"] = np.asarray(tokens, dtype=np.int64)
        arrays[name + "_logits"] = np.stack(logits).astype(np.float32)
        arrays[name + "_nocache"] = np.stack(nocache).astype(np.float32)
        arrays[name + "_meta"] = np.asarray([kw["layers"], kw["head_count"], kw["head_dim"], kw["vocab"],
                                             kw["seed"], len(prompt), steps, ps], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "decoder_cases.npz"), **arrays)
    print("wrote", sorted(arrays))


if __name__ == "__main__":
    main()
