"""Trace replay on the device engine: reference workload
traces drive real GPU stores (K1 appends, K3/K2 attention, K0 fork copies)
and the per-event audit of the device-backed pool equals the reference's
own `account` (tests/golden/trace_cases.json)."""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import relative_error  # noqa: E402
from paper_2506_07311_b200 import workload as W  # noqa: E402
from replay import as_numpy  # noqa: E402

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "trace_cases.json")))
CFG = W.KvBytesConfig(**GOLDEN["bytes_config"])


def _case(pred):
    return next(c for c in GOLDEN["cases"] if pred(c))


@pytest.mark.parametrize("which", ["fork", "chat", "ladder"])
@pytest.mark.parametrize("ps", [16, 64])
def test_device_replay_account_matches_reference(which, ps):
    case = {
        "fork": lambda: _case(lambda c: c["generator"] is None),
        "chat": lambda: _case(lambda c: c["generator"] and c["generator"][0] == "gen_chat_growth"),
        "ladder": lambda: _case(lambda c: c["generator"] and c["generator"][1] == [3, "ladder"]),
    }[which]()
    trace = W.Trace.from_jsonl(case["jsonl"])
    rep = W.DeviceReplay(trace, page_size=ps, hq=8, hkv=2, head_dim=128, dtype="bf16",
                         attend=which != "ladder")
    acct = rep.run(CFG)
    want = case["reports"][str(ps)]["paged"]
    got = acct.to_dict(include_series="series" in want)
    assert got == want
    assert rep.stats["appended_tokens"] == sum(
        getattr(ev, "prompt_len", 0) + getattr(ev, "n_tokens", 0) for ev in trace.events)
    if which == "ladder":
        assert rep.pool.census().live_pages == 0  # every page back


def test_device_replay_attention_and_fork_contents():
    """After the fork trace: the last attention (c's decode burst over its
    inherited context) matches float64 over the store's own K/V, and forked
    children read their parent's prefix bit-exactly."""
    ev = [W.Arrive("root", 700), W.ForkEvent("root", "a", 700), W.ForkEvent("root", "b", 333),
          W.Decode("a", 50), W.Decode("b", 20)]
    trace = W.Trace("t", None, ev)
    rep = W.DeviceReplay(trace, page_size=16, hq=8, hkv=2, head_dim=128, dtype="bf16")
    rep.run()
    st = rep.store
    kr, vr = st.gather("root", 700)
    ka, va = st.gather("a", 750)
    kb, vb = st.gather("b", 353)
    assert torch.equal(ka[:700], kr) and torch.equal(va[:700], vr)
    assert torch.equal(kb[:333], kr[:333]) and torch.equal(vb[:333], vr[:333])
    seq, q, out = rep.last_output
    assert seq == "b"
    n = q.shape[0]
    k = kb.double().repeat_interleave(4, 1)
    v = vb.double().repeat_interleave(4, 1)
    s = torch.einsum("qhd,khd->hqk", q.to(torch.bfloat16).double(), k) / np.sqrt(128)
    pos = torch.arange(353 - n, 353, device=s.device)
    s = s.masked_fill(torch.arange(353, device=s.device)[None, :] > pos[:, None], float("-inf"))
    ref = torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), v)
    assert relative_error(as_numpy(out), ref.cpu().numpy()) <= 6e-3
