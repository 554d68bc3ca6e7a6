"""The reference's own test suite, unmodified, against the engine.

tests/golden/reference_suite/ holds verbatim copies of the reference's
pkg/tests/test_{pool,store,attention}.py (sha256-pinned in MANIFEST.json).
Each file runs in a subprocess with `pagedkv` aliased to the numpy-facing
drop-in namespace `paper_2506_07311_b200.pagedkv` — the import swap a
reference user makes.  The pool suite is host-only (the native allocator);
the store and attention suites launch the K1 / K0 / K2 / K3 kernels and need
the GPU.  Where the reference tree is mounted the copies are also checked
byte-for-byte against it.
"""

import hashlib
import json
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "tests", "golden", "reference_suite")
REFERENCE_TESTS = "/root/reference/pkg/tests"

with open(os.path.join(SUITE, "MANIFEST.json")) as _f:
    MANIFEST = json.load(_f)


def test_vendored_suite_is_unmodified():
    for name, digest in MANIFEST["files"].items():
        with open(os.path.join(SUITE, name), "rb") as f:
            data = f.read()
        assert hashlib.sha256(data).hexdigest() == digest, name
        live = os.path.join(REFERENCE_TESTS, name)
        if os.path.exists(live):
            with open(live, "rb") as f:
                assert f.read() == data, f"{name} differs from the reference's copy"


def _run_suite(name: str):
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
    env.pop("PYTEST_ADDOPTS", None)
    cmd = [sys.executable, "-m", "pytest", "-q", "-c", os.path.join(SUITE, "pytest.ini"), "--rootdir", SUITE,
           os.path.join(SUITE, name)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=SUITE)
    tail = r.stdout[-3000:] + r.stderr[-2000:]
    passed = int(m.group(1)) if (m := re.search(r"(\d+) passed", r.stdout)) else 0
    failed = int(m.group(1)) if (m := re.search(r"(\d+) failed", r.stdout)) else 0
    errors = int(m.group(1)) if (m := re.search(r"(\d+) error", r.stdout)) else 0
    return r.returncode, passed, failed + errors, tail


def test_reference_pool_suite_passes_unmodified():
    rc, passed, failed, tail = _run_suite("test_pool.py")
    assert rc == 0 and failed == 0, tail
    assert passed == 20, tail


@pytest.mark.gpu
def test_reference_store_suite_passes_unmodified():
    rc, passed, failed, tail = _run_suite("test_store.py")
    assert rc == 0 and failed == 0, tail
    assert passed == 15, tail


@pytest.mark.gpu
def test_reference_attention_suite_passes_unmodified():
    """34 tests; the reference itself fails test_no_allowed_keys_is_an_error
    with an IndexError — the engine raises NoAllowedKeys."""
    rc, passed, failed, tail = _run_suite("test_attention.py")
    assert rc == 0 and failed == 0, tail
    assert passed == 34, tail  # with pool 20 + store 15: the reference's 69
