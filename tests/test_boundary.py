"""CPU-side checks of the drop-in boundary (no GPU needed)."""

import os
import re

import numpy as np
import pytest

import paper_1707_05141_b200 as bf
from paper_1707_05141_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "batchfact_b200.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"BF_API\s+[\w\s\*]*?\b(bf_\w+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 15
    assert sorted(_lib.EXPORTS) == syms
    L = _lib.load()
    for s in syms:
        assert getattr(L, s) is not None
    assert b"sm_100a" in L.bf_version()


def test_argument_errors_surface_as_valueerror_without_gpu():
    # validation happens before any launch: m < n must fail with the reference's message
    L = _lib.load()
    rc = L.bf_qr_batched_f64(1, 2, 3, None, None, None, 16, None, 0, None)
    assert rc == _lib.BF_ERR_ARG
    assert "qr requires m >= n" in _lib.last_error()
    opts = bf.JacobiOptions().to_c(np.float64)
    rc = L.bf_svd_batched_f64(1, 3, 4, None, None, None, None, None, None, None, opts, None, 0, None)
    assert rc == _lib.BF_ERR_ARG and "svd requires m >= n" in _lib.last_error()
    rc = L.bf_rsvd_batched_f64(1, 8, 8, 8, 1, 0, 0, 0, None, None, None, None, None, None, 0, None)
    assert rc == _lib.BF_ERR_ARG and "exceeds min(m, n)" in _lib.last_error()
    bopts = bf.BlockJacobiOptions(method="gram").to_c(np.float64)
    rc = L.bf_block_svd_batched_f64(1, 4, 8, None, None, None, None, None, None, None, bopts, None, 0, None)
    assert rc == _lib.BF_ERR_ARG


def test_options_validation_matches_reference():
    with pytest.raises(ValueError):
        bf.JacobiOptions(tolerance=0.0)
    with pytest.raises(ValueError):
        bf.JacobiOptions(max_sweeps=0)
    with pytest.raises(ValueError):
        bf.JacobiOptions(ordering="zigzag")
    with pytest.raises(ValueError):
        bf.BlockJacobiOptions(method="qr")
    with pytest.raises(ValueError):
        bf.BlockJacobiOptions(block_width=0)
    with pytest.raises(ValueError):
        bf.RsvdOptions(k=0)
    with pytest.raises(ValueError):
        bf.RsvdOptions(k=4, q_iterations=1)
    assert bf.JacobiOptions().resolve_tolerance(np.float32) == 1e-6
    assert bf.BlockJacobiOptions().resolve_tolerance(np.float64) == 1e-13


def test_round_robin_schedule_host_logic():
    s = bf.round_robin_schedule(8)
    assert s.steps[0] == [(0, 7), (1, 6), (2, 5), (3, 4)]
    assert s.steps[1] == [(0, 6), (5, 7), (1, 4), (2, 3)]
    from oracle import oracle as orc

    for n in range(2, 130, 2):
        ref = orc.round_robin(n)
        got = np.array(bf.round_robin_schedule(n).steps)
        assert np.array_equal(got, ref)
    with pytest.raises(ValueError):
        bf.round_robin_schedule(7)


def test_as_matrix_and_batch_error_types():
    a = bf.as_matrix([[1, 2], [3, 4]])
    assert a.dtype == np.float64 and a.flags.f_contiguous
    with pytest.raises(ValueError):
        bf.as_matrix(np.zeros(3))
    e = bf.BatchError(3, ValueError("x"))
    assert e.index == 3 and "batch entry 3" in str(e)


def test_gemm_argument_errors_without_gpu():
    L = _lib.load()
    rc = L.bf_gemm_batched_f64(1, 4, 4, 4, None, 2, 16, 0, None, 4, 16, 0, None, 4, 16, None)
    assert rc == _lib.BF_ERR_ARG and "lda" in _lib.last_error()
    rc = L.bf_gemm_batched_f64(1, 4, 4, 4, None, 4, 16, 0, None, 4, 16, 0, None, 3, 16, None)
    assert rc == _lib.BF_ERR_ARG and "ldc" in _lib.last_error()
    assert L.bf_gemm_batched_f64(0, 4, 4, 4, None, 4, 16, 0, None, 4, 16, 0, None, 4, 16, None) == _lib.BF_OK


def test_batch_apply_contract():
    """batch_apply (core.py:97-123): per-entry results independent of threads, lowest failing
    index raised as BatchError after the whole batch ran. Host orchestration, no GPU."""
    import paper_1707_05141_b200 as bf

    ran = []

    def op(x):
        ran.append(x)
        if x in (3, 5):
            raise ValueError(f"bad {x}")
        return x * x

    assert bf.batch_apply(range(4), lambda x: x + 1) == [1, 2, 3, 4]
    assert bf.batch_apply(range(10), lambda x: x * 2, threads=4) == [2 * i for i in range(10)]
    with pytest.raises(bf.BatchError) as ei:
        bf.batch_apply(range(8), op, threads=3)
    assert ei.value.index == 3 and isinstance(ei.value.cause, ValueError)
    assert sorted(ran) == list(range(8))  # every entry still ran
