"""The PARITY softmax's table-based fp64 exp (csrc/f64_exp.cuh) against the
host libm exp (what the reference's std::exp calls, prefill.hpp:143-146):
within 2 ulp over the softmax's argument range, exact 0 below the underflow
threshold, exact 1 at 0, subnormal results correctly scaled."""
import numpy as np
import pytest

import paper_2602_23592_b200 as kb

pytestmark = pytest.mark.gpu


def gpu_exp(x):
    import torch
    xt = torch.tensor(x, dtype=torch.float64, device="cuda")
    yt = torch.empty_like(xt)
    lib = kb.load_library()
    assert lib.keep_debug_exp_f64(xt.data_ptr(), yt.data_ptr(), len(x)) == 0
    return yt.cpu().numpy()


def ulps(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.abs(a - b) / np.spacing(np.maximum(np.abs(b), np.finfo(np.float64).tiny))


def test_exp_within_two_ulp():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(-745.0, 256.0, 2_000_000), rng.uniform(-1.0, 1.0, 1_000_000),
                        rng.uniform(-40.0, 0.0, 1_000_000), -np.arange(0, 700, 1.0 / 64)])
    y, ref = gpu_exp(x), np.exp(x)
    normal = ref >= np.finfo(np.float64).tiny
    assert float(np.max(ulps(y[normal], ref[normal]))) <= 2.0
    assert gpu_exp(np.array([0.0]))[0] == 1.0


def test_exp_underflow_and_subnormals():
    x = np.array([-745.3, -800.0, -1e18, -np.finfo(np.float64).max, -744.0, -740.0, -709.0, -708.5])
    y, ref = gpu_exp(x), np.exp(x)
    assert np.all(y[:4] == 0.0)
    # subnormal range: the absolute error is at most a couple of subnormal steps
    assert np.all(np.abs(y[4:] - ref[4:]) <= 2 * np.maximum(np.spacing(ref[4:]), 5e-324))
