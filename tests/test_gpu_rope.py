"""The opt-in RoPE position re-shift hook (north_star subsystem 3).

The reference is NoPE (model.hpp:3-8), so there is no oracle and
every parity test runs with the hook off (theta = 0, the identity).  What the
hook must satisfy is checked by construction: layer-0 keys depend on the token
alone, so a cached block computed at owner-local positions and re-shifted by
its layout offset must equal the keys recomputed at their layout positions
(rotation composition R(delta) R(p) = R(p + delta)); values are never rotated.
"""
import numpy as np
import pytest

import paper_2602_23592_b200 as kb

pytestmark = pytest.mark.gpu

L, H, d, MLP, V = 2, 2, 256, 256, 512  # head_dim 128


def layer0_kv(numerics, plan0, theta):
    rng = np.random.default_rng(3)
    seg_len = np.array([7, 9, 6], np.int32)
    tokens = rng.integers(0, V, int(seg_len.sum())).astype(np.int32)
    query = rng.integers(0, V, 5).astype(np.int32)
    lay = kb.Layout(seg_len, tokens)
    with kb.Context(L, H, d, MLP, V, 11, numerics) as ctx:
        ctx.set_rope(theta)
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        plan = np.array([plan0, plan0], np.uint8)
        ctx.prefill_begin(lay, query)
        for l in range(L):
            ctx.prefill_layer(plan[l], summary=False)
        _, kv = ctx.prefill_finish(kv=True)
        cached = [ctx.memory_read(kb.SEGMENT, i, 0, int(seg_len[i])) for i in range(3)]
    return kv[0], seg_len, cached


@pytest.mark.parametrize("numerics,tol", [(kb.PARITY, 2e-6), (kb.FAST, 2e-2)])
def test_reshifted_cached_keys_equal_recomputed(numerics, tol):
    theta = 10000.0
    full, seg_len, cached = layer0_kv(numerics, [1, 1, 1], theta)      # every row recomputed at its position
    reuse, _, _ = layer0_kv(numerics, [1, 0, 0], theta)                # segments 1, 2 from the cache, re-shifted
    starts = np.concatenate([[0], np.cumsum(seg_len)])
    for i in (1, 2):
        a, b = starts[i], starts[i + 1]
        kf, kr = full[0, a:b].astype(np.float64), reuse[0, a:b].astype(np.float64)
        assert np.max(np.abs(kf - kr)) <= tol * np.max(np.abs(kf))
        assert np.array_equal(full[1, a:b], reuse[1, a:b]) or numerics == kb.FAST  # values: no rotation
        # the cache itself holds owner-local positions: without the re-shift the keys would differ
        assert np.max(np.abs(cached[i][0].astype(np.float64) - kf)) > 10 * tol * np.max(np.abs(kf))


def test_rope_off_is_the_reference_path():
    full0, _, _ = layer0_kv(kb.PARITY, [1, 0, 0], 0.0)
    with kb.Context(L, H, d, MLP, V, 11, kb.PARITY) as ctx:
        assert ctx.set_rope(0.0) is ctx
    full1, _, _ = layer0_kv(kb.PARITY, [1, 0, 0], 0.0)
    assert np.array_equal(full0, full1)


def test_rope_scope_errors():
    lay = kb.Layout(np.array([4, 5], np.int32), np.arange(9, dtype=np.int32))
    with kb.Context(L, H, d, MLP, V, 11, kb.PARITY) as ctx:
        with pytest.raises(kb.KeepError):
            ctx.set_rope(-1.0)
        ctx.set_rope(500.0).model_init()
        ctx.memory_compute_layout(lay)
        with pytest.raises(kb.KeepError) as e:
            ctx.plan_keep_batch(lay, np.array([[1, 2]], np.int32), np.ones(L))
        assert e.value.code == 1
        ctx.plan_keep(lay, np.array([1, 2], np.int32), np.ones(L))  # the single-query path runs
