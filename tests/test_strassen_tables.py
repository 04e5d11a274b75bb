"""The bilinear algorithm behind the Strassen schedule of the dense preconditioner
products (csrc/vector.cu: StrassenIn / StrassenDown / StrassenUp), restated with
numpy on scalar blocks: L levels = 7^L leaf products, leaf l = (i_1 * 7 + i_2) * 7
+ ..., blocks indexed by quadrant digits q = 2 * (lower half) + (right half), most
significant first; the right operand is given transposed (Bt), as the DMMA GEMM
takes it.  A CPU check of the tables and index conventions the kernels use."""

import itertools

import numpy as np
import pytest

# product i: first quadrant (+1), second quadrant or -1, second sign  (side 0: A, side 1: Bt)
QA = ((0, 2, 0, 3, 0, 2, 1), (0, 0, 2, 1, 3, 0, 1))
QB = ((3, 3, -1, -1, 1, 0, 3), (3, -1, 3, 0, -1, 2, 3))
MINUS = ((False, False, False, False, False, True, True), (False, False, True, True, False, False, False))
# product i adds into C quadrant CA[i] (+) and CB[i] (sign MB[i]; -1: none)
CA = (0, 2, 1, 0, 1, 3, 0)
CB = (3, 3, 3, 2, 0, -1, -1)
MB = (False, True, False, False, True, False, False)


def quad_row(idx, L):
    return sum(((idx >> (2 * l + 1)) & 1) << l for l in range(L))


def quad_col(idx, L):
    return sum(((idx >> (2 * l)) & 1) << l for l in range(L))


def down(x, L, side):
    """All 7^L leaf operands of the 4^L block values x (depth-first, as StrassenDown)."""
    if L == 0:
        return [x[0]]
    ns = 4 ** (L - 1)
    out = []
    for i in range(7):
        qa, qb = QA[side][i], QB[side][i]
        y = [x[qa * ns + m] if qb < 0 else
             (x[qa * ns + m] - x[qb * ns + m] if MINUS[side][i] else x[qa * ns + m] + x[qb * ns + m])
             for m in range(ns)]
        out += down(y, L - 1, side)
    return out


def up(leaves, L):
    """The 4^L blocks of C from the 7^L leaf products (as StrassenUp)."""
    if L == 0:
        return [leaves[0]]
    ns, per = 4 ** (L - 1), 7 ** (L - 1)
    out = [0.0] * (4 ** L)
    for i in range(7):
        y = up(leaves[i * per:(i + 1) * per], L - 1)
        for m in range(ns):
            out[CA[i] * ns + m] += y[m]
            if CB[i] >= 0:
                out[CB[i] * ns + m] += -y[m] if MB[i] else y[m]
    return out


@pytest.mark.parametrize("L", [1, 2, 3])
def test_flattened_strassen_is_the_matrix_product(L):
    n = 2 ** L
    rng = np.random.default_rng(L)
    A, B = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    Bt = B.T.copy()
    blocks = lambda M: [M[quad_row(q, L), quad_col(q, L)] for q in range(4 ** L)]  # noqa: E731
    la, lb = down(blocks(A), L, 0), down(blocks(Bt), L, 1)
    assert len(la) == 7 ** L
    c = up([a * b for a, b in zip(la, lb)], L)
    C = np.empty((n, n))
    for q in range(4 ** L):
        C[quad_row(q, L), quad_col(q, L)] = c[q]
    assert np.allclose(C, A @ B, rtol=0, atol=1e-12)


def test_quadrant_digits_cover_the_block_grid():
    for L in (1, 2, 3):
        cells = {(quad_row(q, L), quad_col(q, L)) for q in range(4 ** L)}
        assert cells == set(itertools.product(range(2 ** L), repeat=2))
    # top-level quadrant = most significant digit: block rows >= 4 of an 8 x 8 grid belong to quadrants 2, 3
    assert all((quad_row(q, 3) >= 4) == (q >> 4 in (2, 3)) for q in range(64))


def test_leaf_dimensions_of_the_baseline_shapes():
    """Odd shapes are padded to a multiple of 2^(L+1) inside the passes (bench.py restates the
    library's rule for its roofline block): cfg5 q = 8192 runs 1024^3 leaves, cfg4 q = 4095 and
    cfg3 q = 2047 run 512^3 leaves."""
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    assert bench.strassen_leaf(8192, 3) == 1024
    assert bench.strassen_leaf(4095, 3) == 512
    assert bench.strassen_leaf(2047, 2) == 512
    assert bench.strassen_leaf(319, 2) == 80 and bench.strassen_leaf(319, 2) % 2 == 0
