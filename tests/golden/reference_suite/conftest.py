"""Runs the reference's own tests (verbatim copies of /root/reference/pkg/
tests/test_{pool,store,attention}.py, see README.md here) against the
engine: `import pagedkv` resolves to the numpy-facing drop-in namespace
paper_2506_07311_b200.pagedkv.  Driven by tests/test_reference_suite.py in a
subprocess so the alias never meets the real reference package."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2506_07311_b200 import pagedkv  # noqa: E402

pagedkv.install_alias("pagedkv")
