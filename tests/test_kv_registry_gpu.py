"""Device KV registry and paged block tables (asb_kv_*).

The protocol restates KvCacheRegistry (/root/reference/proj/src/executor.cpp:43-82) and
must behave exactly like its own test (/root/reference/proj/tests/test_executor.cpp:53-75):
sealed / unsealed transitions, prefix growth, PROTOCOL on a read of an unsealed session and on
a shrinking commit.  Block tables are integer state and must be bit-exact and deterministic:
LIFO reuse of freed blocks, 64-token blocks, one table per session growing with its KV.
"""
import numpy as np
import pytest

from paper_2603_10342_b200._lib import AsbError
from paper_2603_10342_b200.device import KvPool, Lane, Model

pytestmark = pytest.mark.gpu

PROTOCOL = 3


@pytest.fixture(scope="module")
def model():
    return Model("tiny", seed=3, max_context=4096)


def _status(fn):
    try:
        fn()
    except AsbError as e:
        return e.status
    return 0


def test_registry_sequence_matches_reference(model):
    kv = KvPool(model, num_blocks=128)
    assert _status(lambda: kv.require_sealed(0)) == PROTOCOL       # never committed
    kv.commit(0, 3000)
    assert kv.prefix(0) == 3000
    kv.require_sealed(0)
    kv.append(0, 40)
    assert kv.prefix(0) == 3040
    kv.require_sealed(0)
    kv.begin_write(0)
    assert _status(lambda: kv.require_sealed(0)) == PROTOCOL       # open for a resume write
    kv.commit(0, 3096)                                             # resume of 56 on 3040
    assert kv.prefix(0) == 3096
    kv.require_sealed(0)
    assert _status(lambda: kv.commit(0, 2999)) == PROTOCOL         # shrink is a protocol error


def test_block_tables_bit_exact_and_lifo(model):
    kv = KvPool(model, num_blocks=64)
    lane = Lane(model, max_tokens=512, max_segments=8)
    free0 = kv.free_blocks()
    rng = np.random.default_rng(0)
    # session 0: 130 tokens -> 3 blocks; session 1: 64 tokens -> 1 block; then session 0 grows
    lane.forward(kv, [(0, 130, 0)], rng.integers(0, model.vocab, 130))
    lane.forward(kv, [(1, 64, 0)], rng.integers(0, model.vocab, 64))
    lane.forward(kv, [(0, 70, 0)], rng.integers(0, model.vocab, 70))   # 200 tokens -> 4 blocks
    lane.wait()
    t0, t1 = kv.block_table(0), kv.block_table(1)
    assert len(t0) == 4 and len(t1) == 1 and kv.length(0) == 200 and kv.length(1) == 64
    assert len(set(t0) | set(t1)) == 5 and kv.free_blocks() == free0 - 5
    # a fresh pool replays the same allocation exactly (deterministic integer state)
    kv2 = KvPool(model, num_blocks=64)
    lane.forward(kv2, [(0, 130, 0)], rng.integers(0, model.vocab, 130))
    lane.forward(kv2, [(1, 64, 0)], rng.integers(0, model.vocab, 64))
    lane.forward(kv2, [(0, 70, 0)], rng.integers(0, model.vocab, 70))
    lane.wait()
    assert kv2.block_table(0) == t0 and kv2.block_table(1) == t1
    # release returns the blocks; the next session reuses them last-freed-first (LIFO)
    kv.release(1)
    assert kv.free_blocks() == free0 - 4
    lane.forward(kv, [(2, 10, 0)], rng.integers(0, model.vocab, 10))
    lane.wait()
    assert kv.block_table(2) == t1


def test_pool_exhaustion_is_infeasible_not_a_crash(model):
    kv = KvPool(model, num_blocks=2)
    lane = Lane(model, max_tokens=512, max_segments=8)
    st = _status(lambda: lane.forward(kv, [(0, 200, 0)], np.zeros(200, dtype=np.int32)))
    assert st == 6  # ASB_ERR_INFEASIBLE


def test_failed_forward_leaves_registry_untouched(model):
    """A forward that fails part-way (pool exhaustion on its second segment, max_context on a
    the lane limit) must not half-commit: lengths, block tables and the free list are unchanged,
    and the next forward writes at the right positions (runtime.cu asb_forward)."""
    kv = KvPool(model, num_blocks=4)
    lane = Lane(model, max_tokens=1024, max_segments=8)
    lane.forward(kv, [(0, 64, 0)], np.zeros(64, dtype=np.int32))
    lane.wait()
    before = (kv.length(0), kv.block_table(0), kv.free_blocks())
    # session 0 grows by one block (fits), session 1 needs 4 blocks (does not): whole call fails
    st = _status(lambda: lane.forward(kv, [(0, 10, 0), (1, 200, 0)], np.zeros(210, dtype=np.int32)))
    assert st == 6
    assert (kv.length(0), kv.block_table(0), kv.free_blocks()) == before
    assert kv.length(1) == 0 and kv.block_table(1) == []
    # over the lane's token limit: rejected before any registry change
    st = _status(lambda: lane.forward(kv, [(0, 1, 0), (2, 5000, 0)], np.zeros(5001, dtype=np.int32)))
    assert st != 0
    assert (kv.length(0), kv.block_table(0), kv.free_blocks()) == before
    lane.forward(kv, [(0, 1, 1)], np.zeros(1, dtype=np.int32))
    lane.wait()
    assert kv.length(0) == 65
