"""The one-pass fused-bins context pass (attn_dmma.cu: exp against each row's
own-key score instead of the row max, no max pass) and its rerun path.

tests/test_gpu_parity_tc.py holds PARITY to the CPU oracle on the
tensor-core paths (selections bit-exact, summaries within 1e-12).  It runs
here in a fresh process three ways: the default one-pass layer; with the
overflow bound forced to 2^0 so every summary layer takes the rerun (max pass,
then the context pass against the row max); and with the one-pass layer off.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{}, {"KEEP_REF_MAX_LIMIT": "0"}, {"KEEP_REF_MAX": "0"}],
                         ids=["one-pass", "forced-rerun", "max-pass"])
def test_parity_tc_under_reference_score_modes(env):
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity_tc.py")],
                       cwd=ROOT, env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
