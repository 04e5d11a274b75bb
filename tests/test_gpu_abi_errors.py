"""Argument checking of the newer C-ABI entry points: bad calls come back as
status codes (mapped to the reference's exception classes), never as
crashes or silent garbage."""

import ctypes as C

import numpy as np
import pytest
import torch

import paper_2109_01173_b200 as pb
from paper_2109_01173_b200 import _native as nat

pytestmark = pytest.mark.gpu


def lib():
    return nat.lib()


def test_reduced_solve_object_guards():
    x, y = pb.build_direction_sets(pb.SQUARE, 1, 9, pb.BCKind.DIRICHLET)
    op, _ = pb.elliptic_operator(x, y, 1.0)
    out = C.c_void_p()
    assert lib().sfb_reduced_create(None, op.native(), C.byref(out)) == nat.ERR_ARG
    # a preconditioner that is not a spectral-sum sandwich
    pre = pb.make_preconditioner("elliptic_square", x, y, mode="inverse")
    h = pre.native(op.shape)
    assert lib().sfb_reduced_create(h, op.native(), C.byref(out)) == nat.ERR_ARG
    assert "spectral-sum" in nat.last_error()
    # shape mismatch between cache and operator
    x2, y2 = pb.build_direction_sets(pb.SQUARE, 1, 11, pb.BCKind.DIRICHLET)
    op2, _ = pb.elliptic_operator(x2, y2, 1.0)
    cache = pb.build_spectral_cache(op)
    assert lib().sfb_reduced_create(cache.native(), op2.native(), C.byref(out)) == nat.ERR_ARG
    with pytest.raises(pb.OperatorError):
        pb.solve_reduced(op, np.zeros(op2.shape), cache)


def test_scatter_gemm_and_copy_guards():
    A = torch.zeros((8, 8), dtype=torch.float64, device="cuda")
    seg_bad = (C.c_int * 3)(0, 5, 7)  # does not cover M = 8
    dst = (C.c_void_p * 2)(A.data_ptr(), A.data_ptr())
    ldd = (C.c_int * 2)(8, 8)
    assert lib().sfb_dgemm_nt_scatter(A.data_ptr(), 8, A.data_ptr(), 8, 8, 8, 8, 2, seg_bad, dst, ldd, 0,
                                      nat.stream()) == nat.ERR_ARG
    assert lib().sfb_dgemm_nt_scatter(A.data_ptr(), 8, A.data_ptr(), 8, 8, 8, 8, 9, seg_bad, dst, ldd, 0,
                                      nat.stream()) == nat.ERR_ARG
    assert lib().sfb_copy2d(A.data_ptr(), 8, A.data_ptr(), 8, 0, 8, nat.stream()) == nat.OK  # empty: no-op


def test_imex_run_and_frame_guards():
    res = nat.ImexResult()
    assert lib().sfb_imex_heat_run(None, None, 0, 0, None, 0, None, 1, 0, 0.0, 1, None, 0, None, None,
                                   C.byref(res), nat.stream()) == nat.ERR_ARG
    assert lib().sfb_imex_rds_run(None, None, None, None, 0.0, 1, 0, 0.0, 1, 0.0, None, None, 0, None, None,
                                  C.byref(res), nat.stream()) == nat.ERR_ARG
    out = torch.empty((4, 4), dtype=torch.int16, device="cuda")
    assert lib().sfb_frame_pgm16(None, 4, 4, 4, out.data_ptr(), None, nat.stream()) == nat.ERR_ARG
    lam = np.zeros(3)
    assert lib().sfb_geigh(0, None, 0, None, 0, nat.dptr(lam), None, 0, nat.stream()) == nat.ERR_ARG


def test_pcg_shape_reports_solver_grid():
    x, y = pb.build_direction_sets(pb.CAP_DOMAIN, 2, (12, 8), pb.BCKind.DIRICHLET)
    op, rhs_of = pb.elliptic_operator(x, y, 1.0)
    pre = pb.make_preconditioner("elliptic_xnormal", x, y)
    pb.mo_pcg(op, np.ones(op.shape), precond=pre, stop=pb.relative_residual(1e-6), max_iter=50)
    s = pb.solvers._cached_solver(op, pre)
    qy, qx = C.c_int(0), C.c_int(0)
    assert lib().sfb_pcg_shape(s.handle.p, C.byref(qy), C.byref(qx)) == nat.OK
    assert (qy.value, qx.value) == op.shape
