"""The reference-side integration (integration/b200_backend.hpp):
the UNMODIFIED reference's plan_keep on the CPU against the same call through
the adapter on the B200 -- the reference's own loop over the B200 cursor and
selector, and the one-call device loop -- on identical weights, memory
(static groups and dynamic segments) and query.  integration/_bin/keep_b200_demo
is compiled against /root/reference/proj/include by integration/Makefile."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "integration", "_bin", "keep_b200_demo")


@pytest.mark.parametrize("args", [
    ["2", "24", "4", "4", "32", "64", "128"],        # the reference's toy shape
    ["7", "40", "3", "2", "256", "256", "256"],      # head_dim 128: Ozaki + DMMA kernels
    ["11", "16", "5", "4", "64", "128", "128"],
])
def test_reference_plan_keep_through_the_adapter(args):
    if not os.path.exists(DEMO):
        pytest.skip("integration demo not built (needs /root/reference at build time)")
    r = subprocess.run([DEMO] + args, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "-> OK" in r.stdout
