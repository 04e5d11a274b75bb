"""Sylvester term lists U -> sum_t G_t U H_t, applied on the B200.

Drop-in for operators.py of the reference: the same constructors, pruning
rule, term ordering, error messages and grid conventions (rows follow y,
columns follow x; operators.py:1-9).  The factors stay banded (``Band``)
and are uploaded once, in band storage, the first time an operator is used
on the device; ``apply`` then runs the fused banded kernel
(csrc/banded.cu) instead of 2T dense GEMMs (operators.py:124-131).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _native as nat
from .banded import Band, as_band, band_arrays
from .exceptions import OperatorError
from .fem1d import BCKind, DirectionSet
from .geometry import DomainSpec

PRUNE_TOL = 1e-15
KRONECKER_GUARD = 200_000
MAX_BAND_WIDTH = 9  # widest band the fused kernel is instantiated for (k <= 4)
MAX_BAND_TERMS = 5


# ---------------------------------------------------------------- grids ----
def vec(U) -> np.ndarray:
    """Column-stacking vectorisation (operators.py:29-31)."""
    return np.asarray(U).reshape(-1, order="F")


def unvec(v, shape) -> np.ndarray:
    return np.asarray(v).reshape(shape, order="F")


def full_node_grid(domain: DomainSpec, x: DirectionSet, y: DirectionSet):
    """Physical coordinates of all nodes, each (Ny+1, Nx+1) (operators.py:39-45)."""
    xr = x.basis.nodes_full + domain.x_offset
    yr = y.basis.nodes_full
    X = np.asarray(domain.profile(yr), dtype=float)[:, None] * xr[None, :]
    return X, np.broadcast_to(yr[:, None], X.shape).copy()


def physical_grid(domain: DomainSpec, x: DirectionSet, y: DirectionSet):
    """Physical coordinates of the retained nodes, each (q_y, q_x) (operators.py:300-307)."""
    xr = x.basis.nodes + domain.x_offset
    yr = y.basis.nodes
    X = np.asarray(domain.profile(yr), dtype=float)[:, None] * xr[None, :]
    return X, np.broadcast_to(yr[:, None], X.shape).copy()


def expand_with_boundary(U, x: DirectionSet, y: DirectionSet):
    """Scatter retained dofs into the full node grid (operators.py:48-56)."""
    full_shape = (y.basis.n_sub + 1, x.basis.n_sub + 1)
    U = np.asarray(U, dtype=float)
    if U.shape == full_shape:
        return np.array(U, copy=True)
    out = np.zeros(full_shape)
    out[np.ix_(y.basis.dof_map >= 0, x.basis.dof_map >= 0)] = U
    return out


def interior_values(F, x: DirectionSet, y: DirectionSet):
    F = np.asarray(F, dtype=float)
    return F[np.ix_(y.basis.dof_map >= 0, x.basis.dof_map >= 0)]


def _check_full_grid(shape, x: DirectionSet, y: DirectionSet):
    want = (y.basis.n_sub + 1, x.basis.n_sub + 1)
    if tuple(shape) != want:
        raise OperatorError(f"nodal source must cover the full node grid {want} "
                            f"(boundary included), got {tuple(shape)}")


@dataclass
class GridFunction:
    """Nodal coefficient matrix plus its discretisation (operators.py:76-94)."""

    values: np.ndarray
    bc: BCKind
    degree: int
    n_sub: tuple

    @property
    def shape(self):
        return self.values.shape

    def vec(self):
        return vec(self.values)

    @classmethod
    def from_vec(cls, v, shape, bc, degree, n_sub):
        return cls(values=unvec(v, shape), bc=bc, degree=degree, n_sub=tuple(n_sub))


# ------------------------------------------------------------ factors -----
def _factor(m):
    if isinstance(m, Band):
        return m
    if sp.issparse(m):
        return Band(m)
    return np.asarray(m, dtype=float)


def _max_abs(m) -> float:
    if isinstance(m, Band):
        return m.max_abs()
    return float(np.max(np.abs(m))) if m.size else 0.0


def _half_bandwidth(m) -> int:
    if isinstance(m, Band):
        return m.half_bandwidth()
    r, c = np.nonzero(m)
    return int(np.max(np.abs(c - r))) if r.size else 0


def _odd_width(w: int) -> int:
    return w if w % 2 == 1 else w + 1


class SylvesterOperator:
    """Linear map U -> sum_i G_i U H_i over q_y x q_x grids (operators.py:97-133)."""

    def __init__(self, terms, symmetric: bool = False, positive_definite: bool = False):
        kept = []
        for G, H in terms:
            G, H = _factor(G), _factor(H)
            if _max_abs(G) <= PRUNE_TOL or _max_abs(H) <= PRUNE_TOL:  # operators.py:106-107
                continue
            kept.append((G, H))
        if not kept:
            raise OperatorError("operator has no nonzero terms")
        qy, qx = kept[0][0].shape[0], kept[0][1].shape[0]
        for G, H in kept:
            if tuple(G.shape) != (qy, qy) or tuple(H.shape) != (qx, qx):
                raise OperatorError("inconsistent term factor shapes")
        self.terms = kept
        self.symmetric = symmetric
        self.positive_definite = positive_definite
        self.shape = (qy, qx)
        self._handle = None
        self._pcg_cache = {}

    def __len__(self):
        return len(self.terms)

    # ---- device form ---------------------------------------------------
    @property
    def half_bandwidth(self) -> int:
        return max(max(_half_bandwidth(G), _half_bandwidth(H)) for G, H in self.terms)

    @property
    def banded(self) -> bool:
        return (2 * self.half_bandwidth + 1 <= MAX_BAND_WIDTH
                and len(self.terms) <= MAX_BAND_TERMS)

    def band_layout(self):
        """(width, offset, gband[T][qy][w], hband[T][qx][w]) as uploaded."""
        b = self.half_bandwidth
        w = 2 * b + 1
        g = band_arrays([G for G, _ in self.terms], True, w, -b)
        h = band_arrays([H for _, H in self.terms], False, w, -b)
        return w, -b, g, h

    def native(self):
        if self._handle is None:
            L = nat.lib()
            qy, qx = self.shape
            out = nat.C.c_void_p()
            if self.banded:
                w, off, g, h = self.band_layout()
                nat.check(L.sfb_op_create(qy, qx, len(self.terms), w, off, nat.host_ptr(g),
                                          w, off, nat.host_ptr(h), nat.C.byref(out)), "operator")
            else:
                G = np.ascontiguousarray(np.stack([np.asarray(G, float) for G, _ in self.terms]))
                H = np.ascontiguousarray(np.stack([np.asarray(H, float) for _, H in self.terms]))
                nat.check(L.sfb_op_create_dense(qy, qx, len(self.terms), nat.host_ptr(G),
                                                nat.host_ptr(H), nat.C.byref(out)), "operator")
            self._handle = nat.Handle(out.value, L.sfb_op_destroy)
        return self._handle.p

    # ---- application ---------------------------------------------------
    def apply(self, U):
        on_dev = nat.is_device(U)
        shape = tuple(U.shape) if on_dev else np.asarray(U).shape
        if shape != self.shape:
            raise OperatorError(f"grid shape {shape} does not match operator {self.shape}")
        h = self.native()
        t = nat.torch()
        Ud = nat.to_device(U)
        W = t.empty_like(Ud)
        qx = self.shape[1]
        nat.check(nat.lib().sfb_op_apply(h, nat.ptr(Ud), qx, nat.ptr(W), qx, nat.stream()), "apply")
        return W if on_dev else nat.to_host(W)

    __call__ = apply


def apply(op: SylvesterOperator, U):
    """Evaluate sum_i G_i U H_i (operators.py:136-138)."""
    return op.apply(U)


def _sparse(m):
    if isinstance(m, Band):
        return m.sparse.tocsr()
    return sp.csr_matrix(np.asarray(m, dtype=float))


def to_kronecker(op: SylvesterOperator) -> sp.csr_matrix:
    """The vec-form sparse matrix with to_kronecker(op) @ vec(U) = vec(op(U))
    (operators.py:141-155): sum_t H_t^T (x) G_t, assembly noise pruned.
    Desk-size cross-check format; the guard is the reference's."""
    qy, qx = op.shape
    if qx * qy > KRONECKER_GUARD:
        raise OperatorError(f"Kronecker assembly guarded at {KRONECKER_GUARD} unknowns, got {qx * qy}")
    out = None
    for G, H in op.terms:
        blk = sp.kron(_sparse(H).T.tocsr(), _sparse(G), format="csr")
        out = blk if out is None else out + blk
    out.data[np.abs(out.data) < PRUNE_TOL] = 0.0
    out.eliminate_zeros()
    return out


# --------------------------------------------------------- rhs builders ---
class RhsBuilder:
    """out = G F H^T over the full node grid F: the weak right-hand side of
    elliptic_operator / parabolic_operator (operators.py:206-207, 228-232,
    266-268, 281-282), evaluated by the banded map kernel.

    Calling it with a numpy array mirrors the reference closure; the IMEX
    drivers use the fused device variants ``heat`` and ``dib``."""

    def __init__(self, G_full: Band, H_full: Band, x: DirectionSet, y: DirectionSet):
        self.G, self.H = as_band(G_full), as_band(H_full)
        self.x, self.y = x, y
        self.out_shape = (y.q, x.q)
        self.in_shape = (y.basis.n_sub + 1, x.basis.n_sub + 1)
        self._handle = None

    def layout(self):
        glo, ghi = self.G.offsets()
        hlo, hhi = self.H.offsets()
        w = _odd_width(max(ghi - glo + 1, hhi - hlo + 1))
        return w, glo, self.G.band_rows(w, glo), hlo, self.H.band_rows(w, hlo)

    def native(self):
        if self._handle is None:
            L = nat.lib()
            w, goff, g, hoff, h = self.layout()
            if w > MAX_BAND_WIDTH:
                raise OperatorError("rhs map wider than the banded kernel supports")
            out = nat.C.c_void_p()
            nat.check(L.sfb_map_create(self.out_shape[0], self.out_shape[1], self.in_shape[0],
                                       self.in_shape[1], w, goff, nat.host_ptr(np.ascontiguousarray(g)),
                                       w, hoff, nat.host_ptr(np.ascontiguousarray(h)),
                                       nat.C.byref(out)), "rhs map")
            self._handle = nat.Handle(out.value, L.sfb_map_destroy)
        return self._handle.p

    def __call__(self, F):
        on_dev = nat.is_device(F)
        _check_full_grid(tuple(F.shape) if on_dev else np.asarray(F).shape, self.x, self.y)
        t = nat.torch()
        Fd = nat.to_device(F)
        out = t.empty(self.out_shape, dtype=t.float64, device="cuda")
        nat.check(nat.lib().sfb_map_apply(self.native(), nat.ptr(Fd), self.in_shape[1], nat.ptr(out),
                                          self.out_shape[1], nat.stream()), "rhs")
        return out if on_dev else nat.to_host(out)

    def heat(self, U, c: float, F=None, out=None, check: bool = True):
        """rhs of W = expand(U) + c F (device tensors); returns (rhs, [max|W|, #nonfinite])."""
        t = nat.torch()
        out = t.empty(self.out_shape, dtype=t.float64, device="cuda") if out is None else out
        rs = 1 if self.y.basis.bc is BCKind.DIRICHLET else 0
        cs = 1 if self.x.basis.bc is BCKind.DIRICHLET else 0
        chk = np.zeros(2)
        nat.check(nat.lib().sfb_map_apply_heat(
            self.native(), nat.ptr(U), U.shape[1], rs, cs, float(c),
            nat.ptr(F) if F is not None else None, self.in_shape[1], nat.ptr(out), self.out_shape[1],
            nat.dptr(chk) if check else None, nat.stream()), "heat rhs")
        return out, chk

    def dib(self, U, V, species: int, tau_rho: float, params, out=None, check: bool = True):
        """rhs of W = U + tau rho f(U,V) (species 0) or V + tau rho g(U,V) (species 1)."""
        t = nat.torch()
        out = t.empty(self.out_shape, dtype=t.float64, device="cuda") if out is None else out
        kp = np.ascontiguousarray(params, dtype=float)
        chk = np.zeros(2)
        nat.check(nat.lib().sfb_map_apply_dib(
            self.native(), nat.ptr(U), nat.ptr(V), U.shape[1], int(species), float(tau_rho),
            nat.dptr(kp), nat.ptr(out), self.out_shape[1], nat.dptr(chk) if check else None,
            nat.stream()), "dib rhs")
        return out, chk


def _interior_selector(d: DirectionSet) -> Band:
    """q x (N+1) 0/1 matrix picking the retained nodes."""
    keep = np.nonzero(d.basis.dof_map >= 0)[0]
    m = sp.csr_matrix((np.ones(keep.size), (np.arange(keep.size), keep)),
                      shape=(keep.size, d.basis.n_sub + 1))
    return Band(m)


# -------------------------------------------------------- constructors ----
def is_unit_degenerate(y: DirectionSet) -> bool:
    """operators.py:158-165."""
    m = y.mats
    scale = max(m.A.max_abs(), 1.0)
    return ((m.M2).max_abs() <= 1e-14 * scale and (m.C2).max_abs() <= 1e-14 * scale
            and (m.B1 - m.A).max_abs() <= 1e-13 * scale
            and (m.M1 - m.M).max_abs() <= 1e-13
            and (m.M3 - m.M).max_abs() <= 1e-13)


def _require_coercive(bc: BCKind, gamma: float) -> None:
    if gamma < 0:
        raise OperatorError("reaction coefficient must be nonnegative")
    if bc is BCKind.NEUMANN and gamma == 0.0:
        raise OperatorError("singular operator: pure Neumann Laplacian needs gamma > 0")


def _lumped_parts(x: DirectionSet, y: DirectionSet):
    if x.lumped is None or y.lumped is None:
        raise OperatorError("direction sets were assembled without lumped matrices")
    lx, ly = x.lumped, y.lumped
    d1 = ly.D1.diagonal()
    return lx, ly, d1, ly.M0 * d1  # diagonal product M0 D1


def elliptic_operator(x: DirectionSet, y: DirectionSet, gamma: float = 0.0, lumped: bool = False):
    """-Laplacian + gamma as a term list, plus its rhs builder (operators.py:177-234)."""
    _require_coercive(x.basis.bc, gamma)
    mx, my = x.mats, y.mats
    if lumped:
        lx, ly, d1, ml = _lumped_parts(x, y)
        terms = [(ly.M0 / d1[:, None], mx.A),
                 (ly.A1 + gamma * ml, lx.M0),
                 (Band.diag(ly.D2.diagonal() ** 2 / d1) @ ly.M0, lx.A2),
                 (-(ly.D2 @ ly.C.T), lx.D3 @ lx.C.T),
                 (-(ly.C @ ly.D2), lx.C @ lx.D3)]
        op = SylvesterOperator(terms, symmetric=True, positive_definite=True)
        rhs = RhsBuilder(ml @ _interior_selector(y), lx.M0 @ _interior_selector(x), x, y)
        return op, rhs
    if is_unit_degenerate(y):
        op = SylvesterOperator([(my.A + 0.5 * gamma * my.M, mx.M),
                                (my.M, mx.A + 0.5 * gamma * mx.M)],
                               symmetric=True, positive_definite=True)
    else:
        op = SylvesterOperator([(my.M1, mx.A), (my.B1 + gamma * my.M3, mx.M), (my.M2, mx.B2),
                                (-my.C2, mx.C1), (-my.C2.T, mx.C1.T)],
                               symmetric=True, positive_definite=True)
    return op, RhsBuilder(my.M3_full, mx.M_full, x, y)


def parabolic_operator(x: DirectionSet, y: DirectionSet, d_u: float, tau: float, lumped: bool = False):
    """Implicit-Euler step operator mass + d tau stiffness and its rhs builder
    (operators.py:237-284)."""
    if d_u <= 0:
        raise OperatorError("diffusion coefficient must be positive")
    if tau < 0:
        raise OperatorError("timestep must be nonnegative")
    mx, my = x.mats, y.mats
    c = d_u * tau
    if lumped:
        lx, ly, d1, ml = _lumped_parts(x, y)
        terms = [(ml + c * ly.A1, lx.M0),
                 (c * (ly.M0 / d1[:, None]), mx.A),
                 (c * (Band.diag(ly.D2.diagonal() ** 2 / d1) @ ly.M0), lx.A2),
                 (-c * (ly.D2 @ ly.C.T), lx.D3 @ lx.C.T),
                 (-c * (ly.C @ ly.D2), lx.C @ lx.D3)]
        op = SylvesterOperator(terms, symmetric=True, positive_definite=True)
        rhs = RhsBuilder(ml @ _interior_selector(y), lx.M0 @ _interior_selector(x), x, y)
        return op, rhs
    terms = [(my.M3 + c * my.B1, mx.M), (c * my.M1, mx.A), (c * my.M2, mx.B2),
             (-c * my.C2, mx.C1), (-c * my.C2.T, mx.C1.T)]
    op = SylvesterOperator(terms, symmetric=True, positive_definite=True)
    return op, RhsBuilder(my.M3_full, mx.M_full, x, y)


def mass_operator(x: DirectionSet, y: DirectionSet, lumped: bool = False) -> SylvesterOperator:
    """U -> M3 U M or its lumped diagonal analogue (operators.py:287-297)."""
    if lumped:
        if x.lumped is None or y.lumped is None:
            raise OperatorError("direction sets were assembled without lumped matrices")
        return SylvesterOperator([(y.lumped.M0 @ y.lumped.D1, x.lumped.M0)],
                                 symmetric=True, positive_definite=True)
    return SylvesterOperator([(y.mats.M3, x.mats.M)], symmetric=True, positive_definite=True)
