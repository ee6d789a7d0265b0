"""Memory-store invariants of the C ABI (load_memory / put surface,
cache_manager.hpp:69-184) that the advisor flagged in round 1.

* An all-reused layer may run in place on an HBM arena only when the layout
  covers the arena's whole payload extent: the query's K/V go into the spare
  rows after it.  A layout that is a strict prefix of an arena's owners must
  not write into the next owner's cached KV.
* plan_keep rejects a schedule whose length is not num_layers
  (recompute.hpp:144, ConfigError).
* A put of another block size never silently drops the owner's other
  still-current layers.
"""
import numpy as np
import pytest

import paper_2602_23592_b200 as kb

pytestmark = pytest.mark.gpu

L, H, d, MLP, V = 4, 2, 256, 256, 256  # head_dim 128: the tcgen05 FAST kernels


@pytest.mark.parametrize("numerics", [kb.PARITY, kb.FAST])
def test_prefix_layout_keeps_next_owner_kv(ko, numerics):
    p = ko.make_instance(17, 3, L, H, d, MLP, V)
    starts = np.concatenate([[0], np.cumsum(p.seg_len)])
    with kb.Context(L, H, d, MLP, V, 17, numerics) as ctx:
        ctx.model_init()
        # owners A, B, C in ONE batch: one arena [A | B | C | spare]
        ctx.memory_compute_batch([(kb.SEGMENT, 0), (kb.SEGMENT, 1), (kb.SEGMENT, 2)], [1, 1, 1],
                                 [[int(p.seg_len[0])], [int(p.seg_len[1])], [int(p.seg_len[2])]], p.tokens)
        nC = int(p.seg_len[2])
        before = [ctx.memory_read(kb.SEGMENT, 2, l, nC) for l in range(L)]
        # layout [A, B]: a strict prefix of the arena's owners
        lay = kb.Layout(p.seg_len[:2], p.tokens[: starts[2]])
        plan = np.zeros((L, 2), np.uint8)
        plan[0] = 1  # layers >= 1 reuse every segment (the aliasing candidates)
        ctx.selective_prefill(lay, p.query, plan)
        ctx.plan_keep(lay, p.query, np.array([1.0, 0.3, 0.2, 0.1]))
        for l in range(L):
            k, v = ctx.memory_read(kb.SEGMENT, 2, l, nC)
            assert np.array_equal(k, before[l][0]) and np.array_equal(v, before[l][1]), l
        # and the full layout still aliases in place with identical results to a fresh context
        lay3 = kb.Layout(p.seg_len, p.tokens)
        got = ctx.selective_prefill(lay3, p.query, np.vstack([np.ones(3), np.zeros((L - 1, 3))]).astype(np.uint8))
    if numerics == kb.PARITY:
        w = ko.model_init(L, H, d, MLP, V, 17)
        ref = ko.selective_prefill(p, w, np.vstack([np.ones(3), np.zeros((L - 1, 3))]).astype(np.uint8))
        scale = float(np.max(np.abs(ref["final_hidden"])))
        assert float(np.max(np.abs(got["final_hidden"] - ref["final_hidden"]))) <= 2e-6 * scale


def test_schedule_length_is_checked():
    with kb.Context(L, H, d, MLP, V, 3, kb.PARITY) as ctx:
        ctx.model_init()
        lay = kb.Layout(np.array([4, 5], np.int32), np.arange(9, dtype=np.int32))
        ctx.memory_compute_layout(lay)
        with pytest.raises(kb.KeepError) as e:
            ctx.plan_keep(lay, np.array([1, 2], np.int32), np.ones(L - 1))
        assert e.value.code == 1
        with pytest.raises(kb.KeepError) as e:
            ctx.plan_keep_batch(lay, np.array([[1, 2]], np.int32), np.ones(L + 1))
        assert e.value.code == 1


def test_put_of_other_size_does_not_drop_current_layers():
    rng = np.random.default_rng(0)
    with kb.Context(L, H, d, MLP, V, 3, kb.PARITY) as ctx:
        k5, v5 = rng.standard_normal((2, 5, d)).astype(np.float32)
        k6, v6 = rng.standard_normal((2, 6, d)).astype(np.float32)
        ctx.memory_put(kb.SEGMENT, 9, 1, 0, k5, v5)
        with pytest.raises(kb.KeepError) as e:  # layer 0 (5 tokens, version 1) is still current
            ctx.memory_put(kb.SEGMENT, 9, 1, 1, k6, v6)
        assert e.value.code == 2
        k, v = ctx.memory_read(kb.SEGMENT, 9, 0, 5)
        assert np.array_equal(k, k5) and np.array_equal(v, v5)
        # a newer version makes layer 0 stale: replacing the block is then the reference's behaviour
        ctx.memory_put(kb.SEGMENT, 9, 2, 1, k6, v6)
        k, v = ctx.memory_read(kb.SEGMENT, 9, 1, 6)
        assert np.array_equal(k, k6) and np.array_equal(v, v6)
        with pytest.raises(kb.KeepError) as e:
            ctx.load_memory(kb.SEGMENT, 9, 0)
        assert e.value.code == 4
