"""The hot path's caller end to end: this repo's PagedDecoderCache /
DecodeSession (reference decoder.py:196-287) driving the test toy model
(tests/toy_decoder.py) reproduce the real reference's greedy generation —
the same tokens and per-step logits as reference `generate(mode="cached")`
(golden vectors from tests/golden/make_decoder_golden.py)."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import relative_error  # noqa: E402
from paper_2506_07311_b200 import DecodeSession, PagedDecoderCache, PagePool  # noqa: E402
from toy_decoder import ToyDecoder, load_cases  # noqa: E402

pytestmark = pytest.mark.gpu
CASES = load_cases(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "decoder_cases.npz"))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_decode_session_matches_reference_generation(case):
    dec = ToyDecoder(case["config"])
    ps, n_prompt, steps = case["page_size"], case["n_prompt"], case["steps"]
    pool = PagePool(-(-(n_prompt + steps) // ps) + 1, ps)
    cache = PagedDecoderCache(dec, pool)
    sess = DecodeSession(dec, cache, "gen")
    tokens = [int(t) for t in case["tokens"][:n_prompt]]
    logits = sess.prefill(tokens)
    assert relative_error(logits, case["logits"][0]) <= 1e-5
    for i in range(steps):
        tokens.append(int(np.argmax(logits)))
        logits = sess.step(tokens[-1])
        assert relative_error(logits, case["logits"][i + 1]) <= 1e-5, i
    assert tokens == [int(t) for t in case["tokens"]]
    assert sess.context_len == n_prompt + steps
    assert sess.free() == -(-(n_prompt + steps) // ps)


def test_decode_session_bf16_cache_stays_close():
    case = CASES[0]
    dec = ToyDecoder(case["config"])
    ps, n_prompt = case["page_size"], case["n_prompt"]
    pool = PagePool(8, ps)
    cache = PagedDecoderCache(dec, pool, dtype=torch.bfloat16)
    sess = DecodeSession(dec, cache, 0)
    toks = [int(t) for t in case["tokens"]]
    logits = sess.prefill(toks[:n_prompt])
    assert relative_error(logits, case["logits"][0]) <= 2e-2
    for i in range(10):  # teacher-forced on the reference tokens
        logits = sess.step(toks[n_prompt + i])
        assert relative_error(logits, case["logits"][i + 1]) <= 2e-2
