"""The one-pass fused-bins context pass (attn_dmma.cu: exp against each row's
own-key score instead of the row max, no max pass) and the max-pass path it falls back to.

tests/test_gpu_parity_tc.py holds PARITY to the CPU oracle on the
tensor-core paths (selections bit-exact, summaries within 1e-12).  It runs
here in a fresh process four ways: the default (one pass where the
Cauchy-Schwarz bound admits it); the bound forced to 0 so every summary layer
takes the max pass; the bound lifted so every summary layer takes the one pass
(these instances' scores are small); and the one-pass layer off.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{}, {"KEEP_REF_MAX_LIMIT": "0"}, {"KEEP_REF_MAX_LIMIT": "100000"},
                                 {"KEEP_REF_MAX": "0"}],
                         ids=["default", "forced-max-pass", "forced-one-pass", "one-pass-off"])
def test_parity_tc_under_reference_score_modes(env):
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity_tc.py")],
                       cwd=ROOT, env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
