"""Pins for the oracle's broadphase, Delassus operator and LCP solver.

Broadphase: scipy cKDTree periodic pair search (independent library).
Delassus: single-constraint closed forms, Newton's third law,
angular-momentum balance of SNSD wrenches, symmetry / PSD,
Eq. ellipsoid_mobility values (tests/golden/mobility.txt).
LCP: brute-force support enumeration, SPEC examples, decoupled closed form,
Lemma 5 uniqueness of D x."""
import os

import numpy as np
import pytest
from scipy.spatial import cKDTree

from gen import scenes

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- broadphase

@pytest.mark.parametrize("seed", [1, 2])
def test_broadphase_vs_kdtree(orc, seed):
    sc = scenes.suspension(3000, (1.0, 0.6, 0.4), 0.55, seed)
    rad = sc["axes"].max(1)
    margin = 0.1
    pi, pj = orc.broadphase(sc["pos"], rad, sc["box"], margin, "brute")
    ci, cj = orc.broadphase(sc["pos"], rad, sc["box"], margin, "cells")
    assert np.array_equal(pi, ci) and np.array_equal(pj, cj)
    # kd-tree over the periodic box with the uniform radius (all R equal here)
    tree = cKDTree(np.mod(sc["pos"], sc["box"]), boxsize=sc["box"])
    kd = tree.query_pairs(2 * rad[0] + margin, output_type="ndarray")
    kd = np.sort(kd, axis=1)
    kd = kd[np.lexsort((kd[:, 1], kd[:, 0]))]
    assert np.array_equal(kd[:, 0], pi) and np.array_equal(kd[:, 1], pj)
    # lexicographic order, i < j, no duplicates
    assert np.all(pi < pj)
    key = pi.astype(np.int64) << 32 | pj
    assert np.all(np.diff(key) > 0)


def test_broadphase_cell_size_independent(orc):
    sc = scenes.cfg5(n=8000)
    rad = sc["axes"].max(1)
    a = orc.broadphase(sc["pos"], rad, sc["box"], 0.1, "cells")
    b = orc.broadphase(sc["pos"], rad * 0 + rad.max(), sc["box"], 0.1, "cells")  # same radii
    assert np.array_equal(a[0], b[0])
    c = orc.broadphase(sc["pos"], rad, sc["box"], 0.1, "brute")
    assert np.array_equal(a[0], c[0]) and np.array_equal(a[1], c[1])


# ------------------------------------------------------------------ Delassus

def _net(orc, nb=60, nc=150, seed=0, dynamics=0):
    b, ia, ib, n, ra, rb = scenes.random_constraint_network(nb, nc, seed, dynamics)
    ta, tb = orc.rows(n, ra, rb)
    W = orc.body_W(b)
    return b, ia, ib, n, ta, tb, W


def test_mobility_golden(orc):
    """Eq. ellipsoid_mobility for radii (1,1,2), xi = 1:
    L = 2 r_3 = 4 -> 1/L = 0.25, 12/L^3 = 0.1875 (tests/golden/mobility.txt)."""
    vals = dict(line.split()[:2] for line in open(os.path.join(GOLDEN, "mobility.txt"))
                if line.strip() and not line.startswith("#"))
    sc = dict(n=1, dynamics=1, axes=np.array([[1.0, 1.0, 2.0]]), xi=1.0, quat=np.array([[1.0, 0, 0, 0]]))
    W = orc.body_W(sc).reshape(6, 6)
    assert W[0, 0] == float(vals["translation"]) and W[3, 3] == float(vals["rotation"])
    assert np.count_nonzero(W - np.diag(np.diag(W))) == 0


def test_single_constraint_closed_form(orc):
    """A_11 = s (1/m_a + 1/m_b + t_a^T I_a^-1 t_a + t_b^T I_b^-1 t_b)."""
    b, ia, ib, n, ta, tb, W = _net(orc, 10, 1, 3)
    s = 1e-6
    y = orc.delassus_apply(W, ia, ib, n, ta, tb, s, np.array([1.0]))
    a, c = ia[0], ib[0]
    Ia = W[a].reshape(6, 6)[3:, 3:]
    Ic = W[c].reshape(6, 6)[3:, 3:]
    ref = s * (b["inv_mass"][a] + b["inv_mass"][c] + ta[0] @ Ia @ ta[0] + tb[0] @ Ic @ tb[0])
    assert abs(y[0] - ref) <= 1e-15 * abs(ref)


def test_head_on_spheres(orc):
    """Head-on central contact (zero lever-arm torque): A_11 = s(1/m_a + 1/m_b)."""
    sc = scenes.suspension(2, (0.5, 0.5, 0.5), 0.01, 0)
    pos = np.array([[0, 0, 0], [0.9, 0, 0.0]])
    phi, n, ra, rb, _ = orc.snsd(pos, sc["quat"], sc["axes"], None, [0], [1])
    ta, tb = orc.rows(n, ra, rb)
    assert np.abs(ta).max() < 1e-15 and np.abs(tb).max() < 1e-15
    W = orc.body_W(sc)
    y = orc.delassus_apply(W, [0], [1], n, ta, tb, 2.0, np.array([1.0]))
    ref = 2.0 * (sc["inv_mass"][0] + sc["inv_mass"][1])
    assert abs(y[0] - ref) < 1e-14 * ref


def test_wrench_balance_laws(orc):
    """F = D x on SNSD constraints: total force is zero (Newton's third law,
    P:L151-157) and total torque about the origin is zero (forces act along
    the shared normal line y_b - y_a = Phi n)."""
    sc = scenes.cfg1()
    rad = sc["axes"].max(1)
    box = np.zeros(3)                       # no periodic images for the moment balance
    pi, pj = orc.broadphase(sc["pos"], rad, box, 0.1)
    phi, n, ra, rb, _ = orc.snsd(sc["pos"], sc["quat"], sc["axes"], box, pi, pj)
    ta, tb = orc.rows(n, ra, rb)
    x = np.random.default_rng(0).uniform(0, 1, len(pi))
    F, _ = orc.wrench(orc.body_W(sc), pi, pj, n, ta, tb, x)
    assert np.abs(F[:, :3].sum(0)).max() < 1e-11
    torque = F[:, 3:] + np.cross(sc["pos"], F[:, :3])
    assert np.abs(torque.sum(0)).max() < 1e-10


def test_delassus_symmetric_psd_dense(orc):
    """A = s D^T W D: x^T A y = y^T A x, x^T A x >= 0, and the dense matrix
    from unit columns equals the assembled D^T W D."""
    b, ia, ib, n, ta, tb, W = _net(orc, 30, 80, 5)
    s = 1e-3
    rng = np.random.default_rng(1)
    x, y = rng.standard_normal(80), rng.standard_normal(80)
    Ax, Ay = (orc.delassus_apply(W, ia, ib, n, ta, tb, s, v) for v in (x, y))
    assert abs(x @ Ay - y @ Ax) <= 1e-13 * np.abs(x) @ np.abs(Ay)
    assert x @ Ax >= 0
    cols = np.stack([orc.delassus_apply(W, ia, ib, n, ta, tb, s, e) for e in np.eye(80)], 1)
    D = np.zeros((6 * 30, 80))
    for al in range(80):
        D[6 * ia[al]:6 * ia[al] + 3, al] = -n[al]
        D[6 * ia[al] + 3:6 * ia[al] + 6, al] = -ta[al]
        D[6 * ib[al]:6 * ib[al] + 3, al] = n[al]
        D[6 * ib[al] + 3:6 * ib[al] + 6, al] = tb[al]
    Wd = np.zeros((180, 180))
    for k in range(30):
        Wd[6 * k:6 * k + 6, 6 * k:6 * k + 6] = W[k].reshape(6, 6)
    A = s * D.T @ Wd @ D
    assert np.abs(cols - A).max() <= 1e-13 * np.abs(A).max()
    assert np.linalg.eigvalsh(0.5 * (A + A.T)).min() > -1e-12 * np.abs(A).max()


# ----------------------------------------------------------------------- LCP

def test_lcp_spec_examples(orc):
    """SPEC S:L219-220, S:L229 in the q = -b convention (A=I pinned via a
    unit-diagonal operator is not available matrix-free; use enumeration)."""
    assert np.allclose(orc.enumerate_lcp(np.eye(2), -np.array([-1.0, 2.0])), [0, 2])
    assert np.allclose(orc.enumerate_lcp(np.eye(2), -np.array([-1.0, -3.0])), [0, 0])
    assert np.allclose(orc.enumerate_lcp(np.array([[2.0]]), -np.array([4.0])), [2])


@pytest.mark.parametrize("seed", range(6))
def test_bbpgd_vs_enumeration(orc, seed):
    """Tiny random contact LCPs (N_C <= 10): BBPGD solution equals the
    brute-force support enumeration (Lemma 3/4; SPD so x* unique)."""
    b, ia, ib, n, ta, tb, W = _net(orc, 6, 8 + seed % 3, seed)
    s = 1e-2
    nc = len(ia)
    A = np.stack([orc.delassus_apply(W, ia, ib, n, ta, tb, s, e) for e in np.eye(nc)], 1)
    rng = np.random.default_rng(seed)
    q = rng.uniform(-1, 1, nc)
    x, g, info = orc.bbpgd(W, ia, ib, n, ta, tb, s, q, tol=1e-13)
    ref = orc.enumerate_lcp(A, q)
    assert info["converged"]
    if np.linalg.eigvalsh(A).min() > 1e-8 * np.abs(A).max():
        np.testing.assert_allclose(x, ref, atol=1e-8 * (1 + np.abs(ref).max()))
    assert np.all(x >= 0) and np.all(g >= -1e-12)
    assert np.abs(x * g).max() <= 1e-12 * (1 + np.abs(x).max())


def test_decoupled_constraints_closed_form(orc):
    """Disjoint body pairs: A is diagonal, lambda = max(0, -q / A_aa)."""
    nb = 40
    sc = scenes.suspension(nb, (1.0, 0.6, 0.4), 0.1, 4)
    ia = np.arange(0, nb, 2, dtype=np.int32)
    ib = ia + 1
    rng = np.random.default_rng(4)
    n = rng.standard_normal((len(ia), 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    ta, tb = orc.rows(n, rng.uniform(-1, 1, (len(ia), 3)), rng.uniform(-1, 1, (len(ia), 3)))
    W = orc.body_W(sc)
    s = 1e-6
    q = rng.uniform(-1, 1, len(ia))
    diag = orc.delassus_apply(W, ia, ib, n, ta, tb, s, np.ones(len(ia)))
    x, g, info = orc.bbpgd(W, ia, ib, n, ta, tb, s, q, tol=1e-12)
    np.testing.assert_allclose(x, np.maximum(0, -q / diag), rtol=1e-9, atol=1e-12)


def test_lemma5_unique_D_x(orc):
    """Duplicated constraints make A singular (PSD): lambda is not unique but
    D lambda is (Lemma 5 Case 2).  Two warm starts, same D x."""
    b, ia, ib, n, ta, tb, W = _net(orc, 10, 12, 8)
    ia, ib = np.concatenate([ia, ia]), np.concatenate([ib, ib])
    n, ta, tb = np.concatenate([n, n]), np.concatenate([ta, ta]), np.concatenate([tb, tb])
    s = 1e-2
    q = np.concatenate([np.full(12, -0.3), np.full(12, -0.3)])
    rng = np.random.default_rng(8)
    x1, g1, i1 = orc.bbpgd(W, ia, ib, n, ta, tb, s, q, None, 1e-12)
    x2, g2, i2 = orc.bbpgd(W, ia, ib, n, ta, tb, s, q, rng.uniform(0, 50, 24), 1e-12)
    assert i1["converged"] and i2["converged"]
    F1, _ = orc.wrench(W, ia, ib, n, ta, tb, x1)
    F2, _ = orc.wrench(W, ia, ib, n, ta, tb, x2)
    assert np.abs(F1 - F2).max() <= 1e-6 * np.abs(F1).max()
    assert np.abs(x1 - x2).max() > 1e-3 * np.abs(x1).max()   # multipliers differ


def test_assembled_A_equals_matrix_free(orc):
    """The explicitly assembled s D^T W D (scipy, from the column definition
    of D) equals the matrix-free apply on random vectors."""
    b, ia, ib, n, ta, tb, W = _net(orc, 60, 200, 21)
    s = 3e-3
    A = orc.assemble_A(W, ia, ib, n, ta, tb, s)
    rng = np.random.default_rng(2)
    for _ in range(3):
        x = rng.standard_normal(200)
        y = orc.delassus_apply(W, ia, ib, n, ta, tb, s, x)
        assert np.abs(A @ x - y).max() <= 1e-13 * np.abs(y).max()


@pytest.mark.parametrize("seed", range(4))
def test_pgs_vs_enumeration(orc, seed):
    """PGS (a different algorithm on the assembled matrix) reaches the
    brute-force enumeration's solution on tiny contact LCPs."""
    b, ia, ib, n, ta, tb, W = _net(orc, 6, 8 + seed % 3, 40 + seed)
    s = 1e-2
    A = orc.assemble_A(W, ia, ib, n, ta, tb, s)
    q = np.random.default_rng(seed).uniform(-1, 1, len(ia))
    x, g, info = orc.pgs(A, q, tol=1e-13)
    ref = orc.enumerate_lcp(A.toarray(), q)
    assert info["converged"]
    Ad = A.toarray()
    assert np.abs(Ad @ x - Ad @ ref).max() <= 1e-9 * (1 + np.abs(q).max())
    if np.linalg.eigvalsh(Ad).min() > 1e-8 * np.abs(Ad).max():
        np.testing.assert_allclose(x, ref, atol=1e-8 * (1 + np.abs(ref).max()))


def test_bbpgd_vs_pgs_cfg1(orc):
    """The oracle's BB solution of cfg1's A_0 LCP (435 rows, overlapping
    start) equals projected Gauss-Seidel's on the assembled matrix: D lambda
    and g agree (unique by Lemma 5), and lambda too."""
    sc = scenes.cfg1()
    r = orc.relcp_step(sc, snsd_only=True, lcp_tol=1e-12)
    c, W, s = r["constraints"], r["W"], r["s"]
    q = r["q_hist"][0]
    A = orc.assemble_A(W, c["ia"], c["ib"], c["n"], c["ta"], c["tb"], s)
    x_p, g_p, info = orc.pgs(A, q, tol=1e-12)
    assert info["converged"]
    x_b, g_b = c["lam"], r["g_hist"][0]
    F_p, _ = orc.wrench(W, c["ia"], c["ib"], c["n"], c["ta"], c["tb"], x_p)
    F_b, _ = orc.wrench(W, c["ia"], c["ib"], c["n"], c["ta"], c["tb"], x_b)
    assert np.abs(F_p - F_b).max() <= 1e-6 * np.abs(F_b).max()
    assert np.abs(g_p - g_b).max() <= 1e-6 * np.abs(q).max()
    assert np.abs(x_p - x_b).max() <= 1e-6 * np.abs(x_b).max()


def test_openmp_timing_build_same_apply(orc):
    """bench.py's cpu_baseline times the OpenMP build of the same oracle
    source (liboracle_omp.so): its Delassus apply is bitwise the serial one
    (each thread adds its own bodies' wrench terms in the serial order)."""
    from gen import scenes
    b, ia, ib, n, ra, rb = scenes.local_constraint_network(3000, 9000, 3)
    W = orc.body_W(b)
    ta, tb = orc.rows(n, ra, rb)
    x = np.random.default_rng(0).random(len(ia))
    y1 = orc.delassus_apply(W, ia, ib, n, ta, tb, 1e-6, x)
    y2 = orc.delassus_apply(W, ia, ib, n, ta, tb, 1e-6, x, openmp=True)
    assert np.array_equal(y1, y2)
