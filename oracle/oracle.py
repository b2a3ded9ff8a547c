"""CPU oracle for the ReLCP hot path (arXiv 2506.14097) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this module.  It shares no code with the
CUDA path (paper_2506_14097_b200/), which never imports it.

Plain, slow, obviously correct:
  * geometry (SNSD), broadphase, Delassus apply and the BB projected-gradient
    solve run in `relcp_oracle.c` (plain C loops, fp64, long-double sums);
  * Algorithm 1 and its inertial form Eq. relcp_inertial
     are written out below in numpy, line by line, in the paper's
    own order and notation (Phi-tilde, D_n, b_n = A_n iota(x_{n-1}) - g~_{n-1},
    incremental trial configurations C_{n+1} = C_n + dt G M D_n (g_n - iota g_{n-1})).
  * `enumerate_lcp` solves tiny dense LCPs by trying every support (brute force);
    `pgs` (projected Gauss-Seidel on the assembled A, plain C) cross-checks
    the BB solutions with a different algorithm.

Citations: P:Lnnn = /root/reference/PAPER.md line; R<k> = reading k in DESIGN.md.
Parity pins: tests/test_oracle_*.py.  Whole-step trajectories of the BASELINE
configs have no paper pin: "parity unpinned beyond the oracle".
"""
from __future__ import annotations

import ctypes
import itertools
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "relcp_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

INERTIAL = 0
OVERDAMPED = 1
_lib = None
LIB_OMP = os.path.join(HERE, "liboracle_omp.so")
_lib_omp = None


def build(force: bool = False, openmp: bool = False) -> str:
    """Compile relcp_oracle.c with gcc (no FMA contraction, no fast-math).
    openmp=True builds the timing-only all-core variant liboracle_omp.so
    (bench.py cpu_baseline); every test uses the serial liboracle.so."""
    out = LIB_OMP if openmp else LIB
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu99", "-ffp-contract=off", "-fno-fast-math",
                               *(["-fopenmp"] if openmp else []), "-shared", "-fPIC", "-o", out, SRC, "-lm"])
    return out


def lib(openmp: bool = False):
    global _lib, _lib_omp
    if openmp:
        if _lib_omp is None:
            _lib_omp = _load(build(openmp=True))
        return _lib_omp
    if _lib is None:
        _lib = _load(build())
    return _lib


def _load(path):
    L = ctypes.CDLL(path)
    P = ctypes.c_void_p
    i64 = ctypes.c_int64
    L.orc_snsd_batch.restype = i64
    L.orc_snsd_batch.argtypes = [i64, P, P, P, P, P, P, ctypes.c_int, P, P, P, P, P]
    L.orc_snsd_batch_shapes.restype = i64
    L.orc_snsd_batch_shapes.argtypes = [i64, P, P, P, P, P, P, P, ctypes.c_int, P, P, P, P, P]
    L.orc_broadphase_bruteforce.restype = i64
    L.orc_broadphase_bruteforce.argtypes = [i64, P, P, P, ctypes.c_double, P, P, i64]
    L.orc_broadphase_cells.restype = i64
    L.orc_broadphase_cells.argtypes = [i64, P, P, P, ctypes.c_double, P, P, i64]
    L.orc_delassus_apply.restype = None
    L.orc_delassus_apply.argtypes = [i64, i64, P, P, P, P, P, P, ctypes.c_double, P, P]
    L.orc_wrench.restype = None
    L.orc_wrench.argtypes = [i64, i64, P, P, P, P, P, P, P, P, P]
    L.orc_bbpgd.restype = None
    L.orc_bbpgd.argtypes = [i64, i64, P, P, P, P, P, P, ctypes.c_double, P, P, P,
                            ctypes.c_double, i64, ctypes.c_int, P]
    L.orc_pgs_csr.restype = None
    L.orc_pgs_csr.argtypes = [i64, P, P, P, P, P, P, ctypes.c_double, i64, P]
    return L


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ------------------------------------------------------------------ geometry

def quat_to_rot(q: np.ndarray) -> np.ndarray:
    """Rotation matrices of quaternions (s, w), normalised first."""
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    s, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    R = np.empty(q.shape[:-1] + (3, 3))
    R[..., 0, 0] = 1 - 2 * (y * y + z * z)
    R[..., 0, 1] = 2 * (x * y - s * z)
    R[..., 0, 2] = 2 * (x * z + s * y)
    R[..., 1, 0] = 2 * (x * y + s * z)
    R[..., 1, 1] = 1 - 2 * (x * x + z * z)
    R[..., 1, 2] = 2 * (y * z - s * x)
    R[..., 2, 0] = 2 * (x * z - s * y)
    R[..., 2, 1] = 2 * (y * z + s * x)
    R[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def snsd(pos, quat, axes, box, pi, pj, n_fib: int = 512, shape=None):
    """Shared-normal signed distance for each pair (pi[k], pj[k]) (SURVEY O1,
    P:L225 "points that minimize their shared-normal signed separation
    distance"; P:L678-680 y_b - y_a = Phi n).  shape (N,) int32: 0 ellipsoid
    (axes = semi-axes), 1 spherocylinder (axes[0] = half-length, axes[1] =
    radius; segment distance minus radii); None = all ellipsoids.

    Returns phi (P,), n (P,3) outward normal of a, ra = y_a - x_a (P,3),
    rb = y_b - x_b (P,3), status (P,) 0 = ok, 1 = coincident centres /
    intersecting centrelines, 2 = Newton not certified or mixed shapes."""
    pos, quat, axes = _c(pos, np.float64), _c(quat, np.float64), _c(axes, np.float64)
    box = _c(box if box is not None else np.zeros(3), np.float64)
    pi, pj = _c(pi, np.int32), _c(pj, np.int32)
    P = len(pi)
    phi = np.empty(P)
    n = np.empty((P, 3))
    ra = np.empty((P, 3))
    rb = np.empty((P, 3))
    st = np.empty(P, dtype=np.int32)
    if shape is None:
        lib().orc_snsd_batch(P, _p(pi), _p(pj), _p(pos), _p(quat), _p(axes), _p(box), n_fib,
                             _p(phi), _p(n), _p(ra), _p(rb), _p(st))
    else:
        shape = _c(shape, np.int32)
        lib().orc_snsd_batch_shapes(P, _p(pi), _p(pj), _p(pos), _p(quat), _p(axes), _p(shape), _p(box), n_fib,
                                    _p(phi), _p(n), _p(ra), _p(rb), _p(st))
    return phi, n, ra, rb, st


def bounding_radius(axes, shape=None):
    """Largest distance from the centre to the surface: max semi-axis for an
    ellipsoid, half-length + radius for a spherocylinder, R + r for a torus."""
    axes = np.asarray(axes, dtype=np.float64)
    r = axes.max(axis=1)
    if shape is not None:
        sum_shape = np.isin(np.asarray(shape), (1, 2))
        r = np.where(sum_shape, axes[:, 0] + axes[:, 1], r)
    return r


def broadphase(pos, rad, box, margin, method: str = "auto"):
    """Candidate pairs (i < j) with |x_j - x_i|_min-image < R_i + R_j + margin,
    lexicographic order ("constraints between nearby bodies")."""
    pos, rad = _c(pos, np.float64), _c(rad, np.float64)
    box = _c(box if box is not None else np.zeros(3), np.float64)
    n = len(rad)
    if method == "auto":
        method = "brute" if n <= 4000 else "cells"
    fn = lib().orc_broadphase_bruteforce if method == "brute" else lib().orc_broadphase_cells
    cap = max(16, 64 * n)
    while True:
        oi = np.empty(cap, dtype=np.int32)
        oj = np.empty(cap, dtype=np.int32)
        m = fn(n, _p(pos), _p(rad), _p(box), float(margin), _p(oi), _p(oj), cap)
        if m <= cap:
            return oi[:m].copy(), oj[:m].copy()
        cap = int(m)


# ------------------------------------------------------------------ dynamics

def body_W(sc, quat=None) -> np.ndarray:
    """Per-body 6x6 block W (N,36) frozen at C^k.

    inertial   : M^{-1} = diag(1/m I3, R I_body^{-1} R^T)
    overdamped : local drag (1/xi) diag(1/L I3, 12/L^3 I3), L = major axis
                 length 2 r_3 (Eq. ellipsoid_mobility)
    kinematic bodies (prescribed velocity) get W = 0."""
    n = sc["n"]
    q = sc["quat"] if quat is None else quat
    W = np.zeros((n, 6, 6))
    if sc["dynamics"] == INERTIAL:
        R = quat_to_rot(q)
        Iinv = np.einsum("nij,nj,nkj->nik", R, sc["inv_inertia"], R)
        W[:, 0, 0] = W[:, 1, 1] = W[:, 2, 2] = sc["inv_mass"]
        W[:, 3:, 3:] = Iinv
    else:
        L = 2.0 * bounding_radius(sc["axes"], sc.get("shape"))  # 2 r_3, or l + b for rods (R22)
        xi = sc.get("xi", 1.0)
        for k in range(3):
            W[:, k, k] = 1.0 / (xi * L)
            W[:, 3 + k, 3 + k] = 12.0 / (xi * L ** 3)
    kin = sc.get("kinematic")
    if kin is not None:
        W[kin != 0] = 0.0
    return W.reshape(n, 36)


def rows(nrm, ra, rb):
    """Jacobian row blocks t_a = (y_a - x_a) x n, t_b = (y_b - x_b) x n
    (row of D^T = [-n, -t_a, n, t_b])."""
    return np.cross(ra, nrm), np.cross(rb, nrm)


def delassus_apply(W, ia, ib, nrm, ta, tb, s, x, openmp: bool = False):
    """y = s D^T W D x (plain definition; long-double accumulation in C).
    openmp=True: the timing-only all-core build (bench.py cpu_baseline)."""
    nb = W.shape[0]
    nc = len(ia)
    W, nrm, ta, tb = (_c(a, np.float64) for a in (W, nrm, ta, tb))
    ia, ib = _c(ia, np.int32), _c(ib, np.int32)
    x = _c(x, np.float64)
    y = np.empty(nc)
    lib(openmp).orc_delassus_apply(nb, nc, _p(ia), _p(ib), _p(nrm), _p(ta), _p(tb), _p(W), float(s),
                             _p(x), _p(y))
    return y


def wrench(W, ia, ib, nrm, ta, tb, x):
    """F = D x (N,6) and U = W F (N,6)."""
    nb = W.shape[0]
    W, nrm, ta, tb = (_c(a, np.float64) for a in (W, nrm, ta, tb))
    ia, ib, x = _c(ia, np.int32), _c(ib, np.int32), _c(x, np.float64)
    F = np.empty((nb, 6))
    U = np.empty((nb, 6))
    lib().orc_wrench(nb, len(ia), _p(ia), _p(ib), _p(nrm), _p(ta), _p(tb), _p(W), _p(x), _p(F), _p(U))
    return F, U


def bbpgd(W, ia, ib, nrm, ta, tb, s, q, x0=None, tol=1e-10, max_iter=1_000_000, power_iters=20,
          openmp: bool = False):
    """Solve 0 <= A x + q _|_ x >= 0, A = s D^T W D (Lemma 3) by
    BB projected gradient (reading R1).  Returns x, g, info dict.
    openmp=True: the timing-only all-core build (bench.py cpu_baseline)."""
    nb = W.shape[0]
    nc = len(ia)
    W, nrm, ta, tb, q = (_c(a, np.float64) for a in (W, nrm, ta, tb, q))
    ia, ib = _c(ia, np.int32), _c(ib, np.int32)
    x = np.zeros(nc) if x0 is None else _c(x0, np.float64).copy()
    g = np.empty(nc)
    info = np.zeros(4)
    lib(openmp).orc_bbpgd(nb, nc, _p(ia), _p(ib), _p(nrm), _p(ta), _p(tb), _p(W), float(s), _p(q), _p(x),
                    _p(g), float(tol), int(max_iter), int(power_iters), _p(info))
    return x, g, dict(iterations=int(info[0]), residual=float(info[1]), converged=bool(info[2]),
                      L=float(info[3]))


def assemble_A(W, ia, ib, nrm, ta, tb, s):
    """A = s D^T W D as a scipy CSR matrix, from the plain definition: column
    alpha of D is -[n; t_a] on body ia and +[n; t_b] on body ib (P:L154-157,
    P:L1413), W block diagonal (N 6x6 blocks), A_n = s D^T W D."""
    import scipy.sparse as sp
    nb, nc = W.shape[0], len(ia)
    rows = np.concatenate([6 * np.asarray(ia)[:, None] + np.arange(6), 6 * np.asarray(ib)[:, None] + np.arange(6)])
    vals = np.concatenate([-np.hstack([nrm, ta]), np.hstack([nrm, tb])])
    cols = np.concatenate([np.repeat(np.arange(nc), 6).reshape(nc, 6)] * 2)
    D = sp.csr_matrix((vals.ravel(), (rows.ravel(), cols.ravel())), shape=(6 * nb, nc))
    blk = np.asarray(W, dtype=np.float64).reshape(nb, 6, 6)
    r_ = (6 * np.arange(nb)[:, None, None] + np.arange(6)[None, :, None]) + 0 * np.arange(6)[None, None, :]
    c_ = (6 * np.arange(nb)[:, None, None] + np.arange(6)[None, None, :]) + 0 * np.arange(6)[None, :, None]
    Wb = sp.csr_matrix((blk.ravel(), (r_.ravel(), c_.ravel())), shape=(6 * nb, 6 * nb))  # block diagonal
    return (s * (D.T @ Wb @ D)).tocsr()


def pgs(A, q, x0=None, tol=1e-12, max_sweeps=200_000):
    """Projected Gauss-Seidel on the assembled A (CSR) --
    an LCP algorithm independent of bbpgd.  Returns x, g, info dict."""
    import scipy.sparse as sp
    A = sp.csr_matrix(A)
    A.sort_indices()
    n = A.shape[0]
    indptr = _c(A.indptr, np.int64)
    indices = _c(A.indices, np.int32)
    data = _c(A.data, np.float64)
    q = _c(q, np.float64)
    x = np.zeros(n) if x0 is None else _c(x0, np.float64).copy()
    g = np.empty(n)
    info = np.zeros(3)
    lib().orc_pgs_csr(n, _p(indptr), _p(indices), _p(data), _p(q), _p(x), _p(g), float(tol), int(max_sweeps),
                      _p(info))
    return x, g, dict(sweeps=int(info[0]), residual=float(info[1]), converged=bool(info[2]))


def enumerate_lcp(A, q, tol=1e-12, all_solutions=False):
    """Brute-force LCP 0 <= A x + q _|_ x >= 0: try every support S (2^n),
    solve A_SS x_S = -q_S, accept x_S >= -tol and (A x + q) >= -tol off S."""
    A = np.asarray(A, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    n = len(q)
    sols = []
    for mask in range(1 << n):
        S = [i for i in range(n) if mask >> i & 1]
        x = np.zeros(n)
        if S:
            ASS = A[np.ix_(S, S)]
            xs, *_ = np.linalg.lstsq(ASS, -q[S], rcond=None)
            if np.max(np.abs(ASS @ xs + q[S])) > 1e-9 * (1 + np.max(np.abs(q))):
                continue
            x[S] = xs
        g = A @ x + q
        scale = 1.0 + np.max(np.abs(q))
        if np.all(x >= -tol * scale) and np.all(g >= -1e-9 * scale):
            if not all_solutions:
                return np.maximum(x, 0.0)
            sols.append(np.maximum(x, 0.0))
    if all_solutions:
        return sols
    return None


def network_lcp(sc, tol: float = 1e-10, max_iter: int = 2_000_000):
    """LCP of a given constraint network (BASELINE cfg4): rows t = r x n
    (P:L1413), RHS q = Phi_0 + dt row . U_free with U_free = U^k (inertial,
    F_ext = 0) or 0 (overdamped), A = s D^T W D.
    Returns (x, g, info, W, rows dict)."""
    net = sc["network"]
    W = body_W(sc)
    ta, tb = rows(net["n"], net["ra"], net["rb"])
    ia, ib, nrm = net["ia"], net["ib"], net["n"]
    dt = sc["dt"]
    inertial = sc["dynamics"] == INERTIAL
    U = sc["vel"] if inertial else np.zeros((sc["n"], 6))
    rate = (-(nrm * U[ia, :3]).sum(1) - (ta * U[ia, 3:]).sum(1) + (nrm * U[ib, :3]).sum(1)
            + (tb * U[ib, 3:]).sum(1))
    q = net["phi"] + dt * rate
    s = dt * dt if inertial else dt
    x, g, info = bbpgd(W, ia, ib, nrm, ta, tb, s, q, None, tol, max_iter)
    return x, g, info, W, dict(ia=ia, ib=ib, n=nrm, ta=ta, tb=tb, q=q, s=s)


# ------------------------------------------------------------------- ReLCP

def quat_rate_map(q, omega):
    """G^k on the quaternion block: q_dot = 1/2 (0, omega) (x) q, omega in the
    world frame (reading R6)."""
    s = q[:, 0]
    w = q[:, 1:]
    out = np.empty_like(q)
    out[:, 0] = -0.5 * np.einsum("ij,ij->i", omega, w)
    out[:, 1:] = 0.5 * (s[:, None] * omega + np.cross(omega, w))
    return out


def _margin_for(delta, cutoff, margin):
    """Reading R7: widen the candidate margin (doubling) until it exceeds the
    largest two-body approach 2 delta."""
    while margin <= 2.0 * delta:
        margin *= 2.0
    return margin


def relcp_step(sc, max_recursions: int = 50, lcp_tol: float = 1e-10, f_ext=None,
               n_fib: int = 512, lcp_max_iter: int = 2_000_000, snsd_only: bool = False):
    """One ReLCP time step: Algorithm 1, inertial form Eq.
    relcp_inertial when sc['dynamics'] == INERTIAL.

    Returns dict(pos, quat, vel, constraints=dict(ia, ib, gen, n, ta, tb, phi, q,
    lam), recursions, n_c, iterations, residuals, f, max_overlap, status)."""
    n = sc["n"]
    dt = sc["dt"]
    inertial = sc["dynamics"] == INERTIAL
    s = dt * dt if inertial else dt          # Delta t^2 vs Delta t
    sigma = dt if inertial else 1.0          # U_tot = U_free + sigma W D gamma
    cutoff, eps = sc["cutoff"], sc["eps_ncp"]
    box = sc["box"]
    axes = sc["axes"]
    shape = sc.get("shape")
    rad = bounding_radius(axes, shape)
    pos_k = sc["pos"].copy()
    quat_k = sc["quat"].copy()
    W = body_W(sc)                           # M_k^{-1} or mobility M^k, frozen at C^k
    Wm = W.reshape(n, 6, 6)
    Fext = np.zeros((n, 6)) if f_ext is None else np.asarray(f_ext, dtype=np.float64)

    # --- Algorithm 1 line 1: constraints A_0 between near-contacting pairs at C^k
    margin = cutoff
    pi, pj = broadphase(pos_k, rad, box, margin)
    phi0, n0, ra0, rb0, st0 = snsd(pos_k, quat_k, axes, box, pi, pj, n_fib, shape)
    if np.any(st0 == 1):
        raise ValueError("coincident body centres (degenerate SNSD)")
    keep = phi0 < cutoff                     # reading R5
    ia, ib = pi[keep].copy(), pj[keep].copy()
    nrm = n0[keep].copy()
    ta, tb = rows(nrm, ra0[keep], rb0[keep])
    phi_disc = phi0[keep].copy()
    gen = np.zeros(len(ia), dtype=np.int32)

    # --- line 2: Phi~_0 = Phi_0 + dt D^T (U^k + dt M^{-1} F_ext)   (inertial)
    #              Phi~_0 = Phi_0 + dt D^T M F_ext                   (overdamped)
    if inertial:
        U_free = sc["vel"] + dt * np.einsum("nij,nj->ni", Wm, Fext)
        kin = sc.get("kinematic")
        if kin is not None:
            U_free[kin != 0] = sc["vel"][kin != 0]
    else:
        U_free = np.einsum("nij,nj->ni", Wm, Fext)

    def dT_U(ia_, ib_, nrm_, ta_, tb_, U):
        return (-(nrm_ * U[ia_, :3]).sum(1) - (ta_ * U[ia_, 3:]).sum(1)
                + (nrm_ * U[ib_, :3]).sum(1) + (tb_ * U[ib_, 3:]).sum(1))

    Phi_tilde = phi_disc + dt * dT_U(ia, ib, nrm, ta, tb, U_free)

    # --- line 3: solve 0 <= Phi_1 = Phi~_0 + A_0 gamma_0  _|_ gamma_0 >= 0
    q = Phi_tilde.copy()                     # b_0 = -Phi~_0
    gamma, g, info = bbpgd(W, ia, ib, nrm, ta, tb, s, q, None, lcp_tol, lcp_max_iter)
    iters, resid, conv = [info["iterations"]], [info["residual"]], [info["converged"]]
    q_hist, g_hist = [q.copy()], [g.copy()]
    f_vals = [-0.5 * float(gamma @ delassus_apply(W, ia, ib, nrm, ta, tb, s, gamma))]
    n_c = [len(ia)]
    Phi_lin = g                              # Phi_1 = Phi~_0 + A_0 gamma_0

    # --- line 4: C_1 = C^k + dt G^k (U_free + sigma W D gamma_0)
    _, Uc = wrench(W, ia, ib, nrm, ta, tb, gamma)
    U_tot = U_free + sigma * Uc
    pos_n = pos_k + dt * U_tot[:, :3]
    quat_n = quat_k + dt * quat_rate_map(quat_k, U_tot[:, 3:])
    gamma_prev = gamma

    recursion = 0
    status = 0
    cand = (pi, pj)
    while not snsd_only:
        # --- line 5: exists a body pair with overlap > eps at C_{n+1}?
        delta = float(np.max(np.linalg.norm(pos_n - pos_k, axis=1)))
        new_margin = _margin_for(delta, cutoff, margin)
        if new_margin != margin:
            margin = new_margin
            cand = broadphase(pos_k, rad, box, margin)
        ci, cj = cand
        phin, nn, ran, rbn, stn = snsd(pos_n, quat_n, axes, box, ci, cj, n_fib, shape)
        viol = phin < -eps                   # stopping rule, reading R10
        if not np.any(viol):
            break
        if recursion >= max_recursions:
            status = 1                       # recursion cap (reading R15)
            break
        recursion += 1                       # line 6: n <- n + 1
        # line 7: Delta A_n at C_n (the trial configuration just inspected);
        # frozen normal and lever arms measured from the centres of C_n
        dia, dib = ci[viol], cj[viol]
        dn_ = nn[viol]
        dta, dtb = rows(dn_, ran[viol], rbn[viol])
        dphi = phin[viol]
        # line 8: Phi~_n = append(Phi_n, Phi(C_n)|_{Delta A_n})
        Phi_tilde = np.concatenate([Phi_lin, dphi])
        # line 9: D_n = append(D_{n-1}, new rows)
        ia = np.concatenate([ia, dia]); ib = np.concatenate([ib, dib])
        nrm = np.concatenate([nrm, dn_]); ta = np.concatenate([ta, dta]); tb = np.concatenate([tb, dtb])
        phi_disc = np.concatenate([phi_disc, dphi])
        gen = np.concatenate([gen, np.full(len(dia), recursion, dtype=np.int32)])
        # line 10: solve 0 <= Phi_{n+1} = Phi~_n + A_n (gamma_n - iota(gamma_{n-1})) _|_ gamma_n >= 0
        #          i.e. b_n = A_n iota(x_{n-1}) - g~_{n-1}  (Thm 1)
        x_pad = np.concatenate([gamma_prev, np.zeros(len(dia))])      # iota_{N_C^n}
        A_xpad = delassus_apply(W, ia, ib, nrm, ta, tb, s, x_pad)
        b = A_xpad - Phi_tilde
        q = -b
        gamma, g, info = bbpgd(W, ia, ib, nrm, ta, tb, s, q, x_pad, lcp_tol, lcp_max_iter)
        iters.append(info["iterations"]); resid.append(info["residual"]); conv.append(info["converged"])
        q_hist.append(q.copy()); g_hist.append(g.copy())
        f_vals.append(-0.5 * float(gamma @ delassus_apply(W, ia, ib, nrm, ta, tb, s, gamma)))
        n_c.append(len(ia))
        Phi_lin = g                          # line 11 (= Phi~_n + A_n (gamma_n - iota gamma_{n-1}))
        # line 12: C_{n+1} = C_n + dt G^k (sigma W D_n (gamma_n - iota(gamma_{n-1})))
        _, dU = wrench(W, ia, ib, nrm, ta, tb, gamma - x_pad)
        pos_n = pos_n + dt * sigma * dU[:, :3]
        quat_n = quat_n + dt * quat_rate_map(quat_k, sigma * dU[:, 3:])
        gamma_prev = gamma

    # line 14: accept C^{k+1} = C_{n+1}
    _, Uc = wrench(W, ia, ib, nrm, ta, tb, gamma_prev)
    U_new = U_free + sigma * Uc
    quat_out = quat_n / np.linalg.norm(quat_n, axis=1, keepdims=True)
    pos_out = pos_n.copy()
    per = np.asarray(box) > 0                # wrap each periodic axis (box[k] > 0; min_image is per axis)
    pos_out[:, per] = pos_out[:, per] - box[per] * np.floor(pos_out[:, per] / box[per])
    max_overlap = 0.0
    ci, cj = cand
    phin, *_ = snsd(pos_n, quat_n, axes, box, ci, cj, n_fib, shape)
    if len(phin):
        max_overlap = float(max(0.0, -np.min(phin)))
    return dict(
        pos=pos_out, pos_unwrapped=pos_n, quat=quat_out, vel=U_new if inertial else U_new,
        constraints=dict(ia=ia, ib=ib, gen=gen, n=nrm, ta=ta, tb=tb, phi=phi_disc, q=q, lam=gamma_prev,
                         g=Phi_lin),
        recursions=recursion, n_c=n_c, iterations=iters, residuals=resid, converged=conv,
        f=f_vals, max_overlap=max_overlap, status=status, margin=margin,
        pairs=(pi, pj), U_free=U_free, W=W, s=s, q_hist=q_hist, g_hist=g_hist,
    )
