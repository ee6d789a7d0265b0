"""MLP rows in chunks (abi.cu mlp_chunk_rows: the [rows x f] hidden buffer
bounded for batches with ~10^5 active rows per query).  A prefill with tiny
chunks (KEEP_MLP_CHUNK_ROWS, read once per process, so this runs in a
subprocess) keeps every plan and stays within each numerics mode's
tolerance of the default (chunks under 64 rows take the DFMA / skinny GEMMs
instead of the tensor-core ones, so the bits may differ; at production sizes
every chunk is >= 32K rows and row-local)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, json, numpy as np
sys.path.insert(0, %r)
import paper_2602_23592_b200 as kb
from paper_2602_23592_b200.synth import group_units, make_instance_layout
out = {}
for name, mode, d in (("parity", kb.PARITY, 256), ("fast", kb.FAST, 256)):
    inst = make_instance_layout(5, 30, 300)
    lay = kb.Layout(inst.seg_len, inst.tokens, group_units(30, 4, 0.5))
    with kb.Context(3, 2, d, 2 * d, 300, 5, mode) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        r = ctx.plan_keep(lay, inst.query, kb.ratio_schedule(3, 0.5))
        b = ctx.plan_keep_batch(lay, np.stack([inst.query, inst.query[::-1]]), kb.ratio_schedule(3, 0.5), final_hidden=True)
    out[name] = {"plan": r["plan"].tolist(), "bplan": b[1]["plan"].tolist(),
                 "fh": r["final_hidden"][-8:].astype(float).tolist(), "bfh": b[1]["final_hidden"][-8:].astype(float).tolist()}
print(json.dumps(out))
""" % ROOT


def run(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_mlp_row_chunks_keep_results():
    base = run({})
    chunked = run({"KEEP_MLP_CHUNK_ROWS": "37"})
    for name, tol in (("parity", 2e-6), ("fast", 3e-2)):
        a, b = base[name], chunked[name]
        assert a["plan"] == b["plan"] and a["bplan"] == b["bplan"], name
        for k in ("fh", "bfh"):
            x, y = np.array(a[k]), np.array(b[k])
            assert float(np.max(np.abs(x - y))) <= tol * float(np.max(np.abs(x))), (name, k)
