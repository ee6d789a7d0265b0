"""PARITY on the tensor-core paths (head_dim >= 32: Ozaki int8 projections,
fp64 DMMA attention with the summary bins fused into the context pass as
E . Z on the DMMA) against the CPU oracle on instances the d=64 goldens do not
reach: many 32-key chunks per split, segments straddling chunk and tile
boundaries, 1-token segments (up to 32 destination segments per chunk), static
groups and several key splits.

Selections bit-exact; summaries within the fp64 summation-order tolerance of
tests/test_gpu_parity.py; hidden states within 2e-6 of the max magnitude.
"""
import numpy as np
import pytest

import paper_2602_23592_b200 as kb

pytestmark = pytest.mark.gpu

CASES = [  # seed, S, L, H, d, mlp, V, seg lo, seg hi, qlen
    (101, 40, 3, 2, 256, 256, 300, 8, 12, 8),
    (102, 120, 3, 2, 256, 512, 400, 8, 12, 8),
    (103, 200, 2, 4, 512, 512, 500, 1, 3, 8),     # 1-3 token segments: up to 32 segments per chunk
    (104, 90, 3, 1, 128, 256, 256, 20, 40, 5),   # segments longer than a chunk
    (105, 300, 2, 2, 128, 256, 512, 1, 1, 4),    # every key its own segment
    (106, 64, 3, 4, 256, 256, 256, 8, 12, 8),    # head_dim 64
    (107, 64, 3, 8, 256, 256, 256, 8, 12, 8),    # head_dim 32
]


def layout_with_groups(p, S):
    # every third block of 4 segments is a static group (joint KV), the rest dynamic
    units, i, u = [], 0, 0
    while i < S:
        e = min(S, i + 4)
        if u % 3 == 0:
            units.append((i, e, kb.GROUP, u))
        else:
            units += [(k, k + 1, kb.SEGMENT, k) for k in range(i, e)]
        i, u = e, u + 1
    return kb.Layout(p.seg_len, p.tokens, units), [(b, e, 1 if k == kb.GROUP else 0) for b, e, k, _ in units]


def rel(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b.astype(np.float64)))) / max(float(np.max(np.abs(b))), 1e-30)


@pytest.mark.parametrize("case", CASES, ids=[str(c[0]) for c in CASES])
def test_parity_tensor_core_paths_match_oracle(ko, case):
    seed, S, L, H, d, mlp, V, lo, hi, qlen = case
    p = ko.make_instance(seed, S, L, H, d, mlp, V, lo, hi, qlen)
    lay, units = layout_with_groups(p, S)
    p.units = units
    r = ko.ratio_schedule(L, 0.5)
    w = ko.model_init(L, H, d, mlp, V, seed)
    ref = ko.plan_keep(p, w, r)
    with kb.Context(L, H, d, mlp, V, seed, kb.PARITY) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        got = ctx.plan_keep(lay, p.query, r, summaries=True)
    assert np.array_equal(got["plan"], ref["plan"])
    assert got["orders"] == ref["orders"] and np.array_equal(got["hops"], ref["hops"])
    for l in range(L):
        assert float(np.max(np.abs(got["qts"][l] - ref["qts"][l]))) <= 1e-12, l
        assert float(np.max(np.abs(got["sts"][l] - ref["sts"][l]))) <= 1e-12, l
    assert rel(got["final_hidden"], ref["final_hidden"]) <= 2e-6
