"""Pins for the oracle's torus SNSD (minimisation of the
centreline-circle distance minus the minor radii): the chain-link closed
form, separated coplanar rings, the sphere limit (R = 0), the concentric
set-valued case with the deterministic selection rule (DESIGN R23),
brute-force 2-D sampling, collinearity y_b - y_a = Phi n, swap symmetry."""
import math

import numpy as np

S2 = math.sqrt(0.5)
QZ = [1.0, 0.0, 0.0, 0.0]   # ring axis = world z (ring in the x-y plane)
QY = [S2, -S2, 0.0, 0.0]    # body z -> world y (ring in the x-z plane)


def _tori(orc, pos, quat, R, r, pairs=((0, 1),)):
    pos = np.asarray(pos, float)
    n = len(pos)
    axes = np.zeros((n, 3))
    axes[:, 0] = R
    axes[:, 1] = r
    axes[:, 2] = r
    shape = np.full(n, 2, dtype=np.int32)
    pi = np.array([p[0] for p in pairs], dtype=np.int32)
    pj = np.array([p[1] for p in pairs], dtype=np.int32)
    return orc.snsd(pos, np.asarray(quat, float), axes, None, pi, pj, shape=shape)


def test_chain_link_closed_form(orc):
    """Interlocked links at pitch 1.4: the circles are closest at
    (1,0,0) and (0.4,0,0): Phi = 0.6 - 2 r, n = -x."""
    phi, n, ra, rb, st = _tori(orc, [[0, 0, 0], [1.4, 0, 0]], [QZ, QY], [1.0, 1.0], [0.2, 0.2])
    assert st[0] == 0 and abs(phi[0] - 0.2) < 1e-14
    assert np.allclose(n[0], [-1, 0, 0], atol=1e-12)
    assert np.allclose(ra[0], [0.8, 0, 0], atol=1e-12) and np.allclose(rb[0], [-0.8, 0, 0], atol=1e-12)


def test_coplanar_separated(orc):
    phi, n, ra, rb, st = _tori(orc, [[0, 0, 0], [3.0, 0, 0]], [QZ, QZ], [1.0, 1.0], [0.1, 0.2])
    assert abs(phi[0] - 0.7) < 1e-14 and np.allclose(n[0], [1, 0, 0], atol=1e-12)


def test_sphere_limit(orc):
    rng = np.random.default_rng(5)
    for _ in range(10):
        d = rng.normal(size=3) * 2
        q = rng.normal(size=(2, 4))
        phi, n, *_ = _tori(orc, [[0, 0, 0], d], q, [0.0, 0.0], [0.3, 0.4])
        assert abs(phi[0] - (np.linalg.norm(d) - 0.7)) < 1e-14
        assert np.allclose(n[0], d / np.linalg.norm(d), atol=1e-14)


def test_concentric_set_valued_selection(orc):
    """Coaxial coplanar rings R = 1 and 2: every centreline pair at angle
    theta is 1 apart; the rule picks theta_a = 0: y_a on the +x side."""
    phi, n, ra, rb, st = _tori(orc, [[0, 0, 0], [0, 0, 0]], [QZ, QZ], [1.0, 2.0], [0.1, 0.1])
    assert abs(phi[0] - 0.8) < 1e-13
    assert np.allclose(n[0], [1, 0, 0], atol=1e-12)
    assert np.allclose(ra[0], [1.1, 0, 0], atol=1e-12)


def _circle(c, q, R, th):
    q = np.asarray(q) / np.linalg.norm(q)
    s, x, y, z = q
    M = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - s * z), 2 * (x * z + s * y)],
                  [2 * (x * y + s * z), 1 - 2 * (x * x + z * z), 2 * (y * z - s * x)],
                  [2 * (x * z - s * y), 2 * (y * z + s * x), 1 - 2 * (x * x + y * y)]])
    return c + R * (np.outer(np.cos(th), M[:, 0]) + np.outer(np.sin(th), M[:, 1]))


def test_chain_step_augments_and_resolves(orc):
    """Linked chain under pull (gen.scenes.chain_tori): one contact per link
    at C^k, the recursion appends constraints and ends below eps_NCP
    (stopping rule); kinematic end rings keep their velocity."""
    from gen import scenes
    sc = scenes.chain_tori(n=60)
    r = orc.relcp_step(sc, lcp_tol=1e-12, max_recursions=5)
    assert r["n_c"][0] == sc["n"] - 1 and r["recursions"] >= 1
    assert r["status"] == 0 and r["max_overlap"] <= sc["eps_ncp"]
    assert np.allclose(r["vel"][0], sc["vel"][0]) and np.allclose(r["vel"][-1], sc["vel"][-1])


def test_bruteforce_and_invariants(orc):
    rng = np.random.default_rng(9)
    m = 60
    pos = np.zeros((2 * m, 3))
    pos[1::2] = rng.uniform(-2.0, 2.0, size=(m, 3))
    quat = rng.normal(size=(2 * m, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    R = rng.uniform(0.5, 1.2, size=2 * m)
    r = rng.uniform(0.05, 0.2, size=2 * m)
    pairs = [(2 * k, 2 * k + 1) for k in range(m)]
    phi, n, ra, rb, st = _tori(orc, pos, quat, R, r, pairs)
    th = np.linspace(0, 2 * np.pi, 1500, endpoint=False)
    for k, (a, b) in enumerate(pairs):
        assert st[k] == 0
        A = _circle(pos[a], quat[a], R[a], th)
        B = _circle(pos[b], quat[b], R[b], th)
        dmin = np.sqrt(((A[:, None, :] - B[None, :, :]) ** 2).sum(-1)).min()
        exact = phi[k] + r[a] + r[b]
        assert exact <= dmin + 1e-12 and dmin - exact <= 5e-3 * (R[a] + R[b])
        gap = pos[b] + rb[k] - pos[a] - ra[k]
        assert np.allclose(gap, phi[k] * n[k], atol=1e-12)
    sw = [(b, a) for a, b in pairs]
    phi2, n2, *_ = _tori(orc, pos, quat, R, r, sw)
    assert np.allclose(phi2, phi, atol=1e-12)
