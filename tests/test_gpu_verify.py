"""The reference's self-verification suites (verify.py:520-603) run on the
device engine: oracle equivalence over the seeded
instance grid, paged == gathered bitwise, skip soundness, softmax row sums,
the allocator stress script with its mirror and census oracles, fork
isolation — and the fault hook must make it fail."""

import pytest

pytest.importorskip("torch")

from paper_2506_07311_b200 import ConfigError  # noqa: E402
from paper_2506_07311_b200 import verify as V  # noqa: E402

pytestmark = pytest.mark.gpu

NAMES = ["attention-oracle-equivalence", "paged-vs-gathered-agreement", "block-skip-soundness",
         "softmax-row-sums", "allocator-census-and-mirror", "fork-write-isolation"]


@pytest.mark.parametrize("seed", [0, 7])
def test_verification_passes_on_the_device(seed):
    r = V.run_verification(instances=50, seed=seed, script_ops=1500, isolation_rounds=60)
    assert [c.name for c in r.checks] == NAMES
    assert r.passed, r.to_dict()


def test_injected_block_table_fault_is_detected():
    r = V.run_verification(instances=8, seed=0, script_ops=50, isolation_rounds=2, inject_fault="block-table")
    by = {c.name: c for c in r.checks}
    assert not by["attention-oracle-equivalence"].passed
    assert not r.passed


def test_zero_instances_rejected():
    with pytest.raises(ConfigError):
        V.run_verification(instances=0)
