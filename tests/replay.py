"""Replay helpers shared by the oracle tests and the engine parity tests.

Scripts recorded from the real reference (tests/golden/make_golden.py) are
replayed on any implementation with the reference's duck-typed API; errors are
compared by class name, allocator state by `dump()`.
"""

from __future__ import annotations

import numpy as np


def run_pool_op(pool, op):
    kind = op["op"]
    if kind == "reserve":
        return [int(p) for p in pool.reserve(op["seq"], op["len"])]
    if kind == "grow":
        return [int(p) for p in pool.grow(op["seq"], op["len"])]
    if kind == "free":
        return int(pool.free(op["seq"]))
    if kind == "fork":
        return [int(p) for p in pool.fork(op["parent"], op["seq"], op["len"]).entries]
    if kind == "privatize":
        r = pool.privatize(op["seq"], op["block"])
        return None if r is None else int(r)
    if kind == "set_len":
        pool.table(op["seq"]).logical_len = op["len"]
        return None
    if kind == "translate":
        a = pool.translate(op["seq"], op["pos"])
        if isinstance(a, tuple):
            return [int(a[0]), int(a[1])]
        return [int(a.page_id), int(a.offset)]
    raise ValueError(kind)


def replay_pool_script(script, make_pool):
    """Yield (step, outcome, dump) for every recorded step."""
    pool = make_pool(script["capacity"], script["page_size"])
    for step in script["steps"]:
        try:
            out = {"ok": True, "ret": run_pool_op(pool, step["op"])}
        except Exception as exc:  # compared by class name with the reference
            out = {"ok": False, "err": type(exc).__name__}
        yield step, out, pool.dump()


def replay_store_script(meta, arrays, prefix, make_pool, make_store):
    pool = make_pool(meta["capacity"], meta["page_size"])
    store = make_store(pool, meta["heads"], meta["dim"])
    for op in meta["ops"]:
        try:
            kind = op["op"]
            if kind == "reserve":
                pool.reserve(op["seq"], op["len"])
            elif kind == "grow":
                pool.grow(op["seq"], op["len"])
            elif kind == "assign":
                k = prefix + op["key"]
                store.assign(op["seq"], arrays[k + "_pos"], arrays[k + "_k"], arrays[k + "_v"])
            elif kind == "fork":
                pool.fork(op["parent"], op["seq"], op["len"])
            else:
                pool.free(op["seq"])
            ok, err = True, None
        except Exception as exc:
            ok, err = False, type(exc).__name__
        assert ok == op["ok"], (op, err)
        if not ok:
            assert err == op["err"], (op, err)
    return pool, store


def as_numpy(x):
    if hasattr(x, "detach"):
        x = x.detach()
        if x.dtype.is_floating_point and x.element_size() == 2 and str(x.dtype) == "torch.bfloat16":
            x = x.float()
        return x.cpu().numpy()
    return np.asarray(x)
