"""CPU-side checks of the product library (no GPU needed): it builds, loads,
exports every entry point declared in include/keep_b200.h, its host-only
functions match the oracle, and it fails loudly (an error code, not a crash or
a silent CPU path) when no B200 is present."""
import ctypes
import os

import numpy as np
import pytest

import paper_2602_23592_b200 as kb

LIB = kb.LIB_PATH


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    return kb.load_library()


def test_every_declared_symbol_is_exported(lib):
    names = kb.exported_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    # the C ABI is plain C: no C++ mangled product symbols leak out
    nm = os.popen(f"nm -D --defined-only {LIB}").read()
    exported = [l.split()[-1] for l in nm.splitlines() if " T " in l]
    assert all(s.startswith("keep_") for s in exported if not s.startswith("_")), exported[:20]


def test_library_targets_sm100a(lib):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {LIB} 2>&1").read()
    assert "sm_100a" in out, out[:400]


def test_host_schedule_matches_oracle(lib, ko, golden):
    for c in golden["ratio_schedule"]:
        if "error" in c:
            with pytest.raises(kb.KeepError) as ei:
                kb.ratio_schedule(c["L"], c["r_avg"])
            assert ei.value.kind == c["error"]
        else:
            assert [float(x) for x in kb.ratio_schedule(c["L"], c["r_avg"])] == c["r"]
    for c in golden["layer_budget"]:
        assert kb.layer_budget(c["ratio"], c["S"]) == c["budget"]


def test_no_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(kb.KeepError) as ei:
        kb.Context(4, 4, 32, 64, 128, 1)
    assert ei.value.kind in ("ConfigError", "CudaError")


def test_config_validation_codes(lib):
    cfg = kb.keep_config(4, 3, 32, 64, 128, kb.PARITY, 1, 0, 1, 0, 0)  # d % H != 0
    h = ctypes.c_void_p()
    rc = lib.keep_ctx_create(ctypes.byref(cfg), ctypes.byref(h))
    assert rc == kb.CONFIG
    assert b"divisible" in lib.keep_last_error()
