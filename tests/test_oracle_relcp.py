"""Pins for the oracle's ReLCP step (Algorithm 1; Eq.
relcp_inertial).

Whole-step trajectories of the BASELINE configs have no paper pin; what the
paper fixes, and what these tests check, are its structural results:
  * spheres: orthogonal motion cannot create overlap -> no augmentation;
  * Cor. 4: small dt -> zero augmentations; large dt augments;
  * Thm 1 / App.: retained entries of q are unchanged across recursions;
  * Thm 1 proof: f_n = -1/2 x^T A_n x is non-increasing;
  * stopping rule: accepted state has Phi >= -eps_NCP;
  * Lemma 8: retained linearised gaps stay >= 0;
  * Newton's third law: contact impulses conserve linear momentum.
"""
import math

import numpy as np
import pytest

from gen import scenes


def _two_body(axes, pos, quat, vel, dt, dynamics=0):
    sc = scenes.suspension(2, (1.0, 1.0, 1.0), 0.01, 0, dt=dt, dynamics=dynamics)
    sc["axes"] = np.asarray(axes, float)
    a, b, c = sc["axes"].T
    m = 4.0 / 3.0 * math.pi * a * b * c
    sc["inv_mass"] = 1.0 / m
    sc["inv_inertia"] = 1.0 / np.stack([m / 5 * (b * b + c * c), m / 5 * (a * a + c * c), m / 5 * (a * a + b * b)], 1)
    sc["pos"] = np.asarray(pos, float)
    sc["quat"] = np.asarray(quat, float)
    sc["vel"] = np.asarray(vel, float)
    sc["box"] = np.zeros(3)
    return sc


@pytest.mark.parametrize("dt", [1e-3, 1e-1, 1.0])
def test_spheres_head_on_never_augment(orc, dt):
    sc = _two_body([[0.5] * 3, [0.7] * 3], [[0, 0, 0], [1.25, 0.1, 0]], [[1, 0, 0, 0]] * 2,
                   [[3, 0, 0, 0, 1, 0], [-2, 0.5, 0, 1, 0, 0]], dt)
    r = orc.relcp_step(sc, lcp_tol=1e-12)
    assert r["recursions"] == 0
    assert r["n_c"] == [1]
    assert r["max_overlap"] <= 1e-9


def _glancing(dt):
    """Two prolate ellipsoids just apart (Phi ~ 0.01), rotated 45 deg, sliding
    into each other (§5.2-like glancing contact)."""
    q = [math.cos(math.pi / 8), 0, 0, math.sin(math.pi / 8)]
    q2 = [math.cos(-math.pi / 8), 0, 0, math.sin(-math.pi / 8)]
    sc = _two_body([[1.0, 0.5, 0.5]] * 2, [[0, 0, 0], [0.8, 1.3, 0.0]], [q, q2],
                   [[0.5, 1.0, 0, 0, 0, 0.3], [-0.5, -1.0, 0, 0, 0, -0.3]], dt)
    phi, *_ = __import__("oracle.oracle", fromlist=["x"]).snsd(sc["pos"], sc["quat"], sc["axes"], None, [0], [1])
    return sc, phi[0]


def test_corollary4_small_dt_no_augmentation(orc):
    sc, phi0 = _glancing(1e-4)
    assert phi0 > 0
    sc["cutoff"] = 0.5
    r = orc.relcp_step(sc, lcp_tol=1e-12)
    assert r["recursions"] == 0 and r["max_overlap"] <= sc["eps_ncp"]


def test_large_dt_augments_and_terminates(orc):
    sc, phi0 = _glancing(0.6)
    sc["cutoff"] = 0.5
    r = orc.relcp_step(sc, lcp_tol=1e-12)
    assert r["recursions"] >= 1
    assert r["status"] == 0 and r["max_overlap"] <= sc["eps_ncp"]


@pytest.fixture(scope="module")
def cfg1_step():
    from oracle import oracle as O
    return O.relcp_step(scenes.cfg1(), lcp_tol=1e-10)


def test_cfg1_terminates_within_tolerance(cfg1_step):
    r = cfg1_step
    assert r["status"] == 0 and r["recursions"] >= 1
    assert r["max_overlap"] <= 1e-5
    assert all(r["converged"])
    assert all(np.diff(r["n_c"]) > 0)


def test_q_retention_identity(cfg1_step):
    """b_n = A_n iota(x_{n-1}) - g~_{n-1} leaves the retained right-hand side
    unchanged: q_{m+1}[A_m] = q_m."""
    qh = cfg1_step["q_hist"]
    for a, b in zip(qh[:-1], qh[1:]):
        scale = np.abs(a).max()
        assert np.abs(b[:len(a)] - a).max() <= 1e-11 * scale


def test_objective_monotone(cfg1_step):
    """f_n(x_n*) = -1/2 x*^T A_n x* is non-increasing in n."""
    f = np.array(cfg1_step["f"])
    assert np.all(np.diff(f) <= 1e-9 * np.abs(f).max())


def test_retained_gaps_nonnegative(cfg1_step):
    """Every constraint of the final LCP has g >= -tol (Lemma 8 at the
    linearised level), lambda >= 0, complementarity."""
    c = cfg1_step["constraints"]
    assert np.all(c["lam"] >= 0)
    assert np.all(c["g"] >= -1e-9)
    assert np.abs(np.minimum(c["lam"], c["g"])).max() <= 1e-9


def test_linear_momentum_conserved(cfg1_step):
    """F_ext = 0, inertial: contact forces are equal and opposite,
    so sum m u is unchanged by the step."""
    sc = scenes.cfg1()
    m = 1.0 / sc["inv_mass"]
    p0 = (m[:, None] * sc["vel"][:, :3]).sum(0)
    p1 = (m[:, None] * cfg1_step["vel"][:, :3]).sum(0)
    scale = (m[:, None] * np.abs(cfg1_step["vel"][:, :3])).sum()
    assert np.abs(p1 - p0).max() <= 1e-12 * scale


def test_gen_blocks_and_pairs(cfg1_step):
    """Append-only blocks: gen is non-decreasing in storage order; within a
    block pairs are strictly increasing (one constraint per pair per recursion)."""
    c = cfg1_step["constraints"]
    assert np.all(np.diff(c["gen"]) >= 0)
    for g in np.unique(c["gen"]):
        sel = c["gen"] == g
        key = c["ia"][sel].astype(np.int64) << 32 | c["ib"][sel]
        assert np.all(np.diff(key) > 0)


def test_overdamped_force_balance(orc):
    """Overdamped, F_ext = 0: U = M D gamma with local drag; sum of forces
    xi L u over bodies vanishes (third law)."""
    sc = scenes.suspension(400, (1.0, 0.5, 0.5), 0.2, 12, dt=1e-2, dynamics=1, velocities=False)
    r = orc.relcp_step(sc, lcp_tol=1e-11, lcp_max_iter=200000)
    assert r["status"] == 0
    L = 2 * sc["axes"].max(1)
    W = orc.body_W(sc).reshape(-1, 6, 6)
    _, U = orc.wrench(orc.body_W(sc), r["constraints"]["ia"], r["constraints"]["ib"], r["constraints"]["n"],
                      r["constraints"]["ta"], r["constraints"]["tb"], r["constraints"]["lam"])
    f = U[:, :3] * L[:, None]
    assert np.abs(f.sum(0)).max() <= 1e-10 * np.abs(f).sum()
    assert r["max_overlap"] <= sc["eps_ncp"]


def _nonspherical_cluster(seed=21, n=64, dt=1e-3):
    """Non-periodic cluster of non-spherical ellipsoids with distinct axes per
    body (a = 1, b ~ U(0.45, 0.8), c ~ U(0.25, 0.42)), uniform orientations,
    u, w ~ N(0, 1), overlapping neighbours; textbook solid-ellipsoid mass
    properties (rho = 1)."""
    sc = scenes.suspension(n, (1.0, 0.6, 0.4), 0.45, seed, dt=dt)
    rng = np.random.default_rng(seed)
    axes = np.stack([np.ones(n), rng.uniform(0.45, 0.8, n), rng.uniform(0.25, 0.42, n)], 1)
    a, b, c = axes.T
    m = 4.0 / 3.0 * math.pi * a * b * c
    sc["axes"] = axes
    sc["inv_mass"] = 1.0 / m
    sc["inv_inertia"] = 1.0 / np.stack([m / 5 * (b * b + c * c), m / 5 * (a * a + c * c), m / 5 * (a * a + b * b)], 1)
    sc["box"] = np.zeros(3)
    return sc


def _world_inertia(quat, inv_inertia):
    """I_world = R diag(I_body) R^T, R the rotation of the unit quaternion
    (s, w): R = I + 2 s [w]x + 2 [w]x^2 (textbook, written here independently)."""
    q = quat / np.linalg.norm(quat, axis=1, keepdims=True)
    s, w = q[:, 0], q[:, 1:]
    K = np.zeros((len(q), 3, 3))
    K[:, 0, 1], K[:, 0, 2], K[:, 1, 2] = -w[:, 2], w[:, 1], -w[:, 0]
    K[:, 1, 0], K[:, 2, 0], K[:, 2, 1] = w[:, 2], -w[:, 1], w[:, 0]
    R = np.eye(3) + 2 * s[:, None, None] * K + 2 * K @ K
    return np.einsum("nij,nj,nkj->nik", R, 1.0 / inv_inertia, R)


def _angular_momentum_defect(O, sc, **kw):
    """|Delta L| / scale over the step, L = sum m x^k x u + I_world(C^k) omega
    about the origin (first-order scheme: momenta at C^k)."""
    r = O.relcp_step(sc, lcp_tol=1e-12, **kw)
    m = 1.0 / sc["inv_mass"]
    Iw = _world_inertia(sc["quat"], sc["inv_inertia"])
    du = r["vel"] - sc["vel"]
    lin = m[:, None] * np.cross(sc["pos"], du[:, :3])
    ang = np.einsum("nij,nj->ni", Iw, du[:, 3:])
    scale = np.abs(lin).sum() + np.abs(ang).sum()
    return np.abs((lin + ang).sum(0)).max() / scale, r, scale


def _relaxed_subcluster():
    """The overlap-free cfg1-relaxed bodies (tests/golden, oracle-made) as a
    NON-periodic cluster (contacts across the periodic faces dropped)."""
    sc = scenes.cfg1_relaxed(dt=1e-3)
    sc["box"] = np.zeros(3)
    return sc


@pytest.mark.parametrize("case", ["cluster-snsd-lcp", "relaxed-relcp"])
def test_angular_momentum_conserved(orc, case, monkeypatch):
    """F_ext = 0, inertial, non-periodic: the contact impulses -gamma n on a at
    y_a and +gamma n on b at y_b act along the common normal line
    (y_b - y_a = Phi n; F_a = -n gamma, T_a = -(y_a - x_a) x n gamma,
    P:L151-157), so its moment about the origin, (y_b - y_a) x n gamma,
    vanishes and sum(m x x u + R I R^T omega) is unchanged for rows discovered
    at C^k: the LCP-SNSD step of a deeply overlapping cluster with distinct
    axes per body, and the ReLCP step of an overlap-free (relaxed) cluster,
    which appends no rows (Cor. 4).  The same check
    on an oracle whose rotational mobility is transposed (R^T I^-1 R instead of
    R I^-1 R^T) must fail: this pins the inertial W block."""
    snsd_only = case == "cluster-snsd-lcp"
    sc = _nonspherical_cluster() if snsd_only else _relaxed_subcluster()
    defect, r, scale = _angular_momentum_defect(orc, sc, snsd_only=snsd_only)
    assert r["recursions"] == 0 and len(r["constraints"]["ia"]) > 20
    assert np.abs(r["constraints"]["lam"]).max() > 0 and scale > 1e-3
    assert defect <= 1e-12, defect

    real = orc.body_W

    def transposed(s, quat=None):
        W = real(s, quat).reshape(-1, 6, 6)
        W[:, 3:, 3:] = np.swapaxes(W[:, 3:, 3:], 1, 2)  # symmetric: no change
        R = orc.quat_to_rot(s["quat"] if quat is None else quat)
        W[:, 3:, 3:] = np.einsum("nji,nj,njk->nik", R, s["inv_inertia"], R)  # R^T I^-1 R
        return W.reshape(-1, 36)

    monkeypatch.setattr(orc, "body_W", transposed)
    bad, _, _ = _angular_momentum_defect(orc, sc, snsd_only=snsd_only)
    assert bad > 1e-6, bad
