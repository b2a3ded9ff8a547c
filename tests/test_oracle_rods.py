"""Pins for the oracle's spherocylinder SNSD (centreline segment
distance minus the cap radii): closed forms (parallel side by side, crossed,
collinear tip to tip, SPEC's parallel example S:L62), the sphere limit, the
parallel-overlap midpoint rule (DESIGN R22), brute-force segment sampling,
swap symmetry and collinearity y_b - y_a = Phi n."""
import math

import numpy as np
import pytest

from gen import scenes

QX = [1.0, 0.0, 0.0, 0.0]                                     # rod along x
QY = [math.cos(math.pi / 4), 0.0, 0.0, math.sin(math.pi / 4)]  # rod along y


def _rods(orc, pos, quat, h, r, pairs=((0, 1),)):
    pos = np.asarray(pos, float)
    n = len(pos)
    axes = np.zeros((n, 3))
    axes[:, 0] = h
    axes[:, 1] = r
    axes[:, 2] = r
    shape = np.ones(n, dtype=np.int32)
    pi = np.array([p[0] for p in pairs], dtype=np.int32)
    pj = np.array([p[1] for p in pairs], dtype=np.int32)
    return orc.snsd(pos, np.asarray(quat, float), axes, None, pi, pj, shape=shape)


def test_spec_parallel_example(orc):
    """l = 2, b = 0.5, parallel along x, centres (0,0,0), (0,1,0) -> Phi = 0.5."""
    phi, n, ra, rb, st = _rods(orc, [[0, 0, 0], [0, 1, 0]], [QX, QX], [1.0, 1.0], [0.25, 0.25])
    assert st[0] == 0 and abs(phi[0] - 0.5) < 1e-15
    assert np.allclose(n[0], [0, 1, 0], atol=1e-15)
    assert np.allclose(ra[0], [0, 0.25, 0], atol=1e-15) and np.allclose(rb[0], [0, -0.25, 0], atol=1e-15)


def test_crossed_and_collinear(orc):
    phi, n, ra, rb, st = _rods(orc, [[0, 0, 0], [0, 0, 1.0]], [QX, QY], [1.0, 1.5], [0.2, 0.3])
    assert abs(phi[0] - 0.5) < 1e-15 and np.allclose(n[0], [0, 0, 1], atol=1e-15)
    phi, n, ra, rb, st = _rods(orc, [[0, 0, 0], [3.0, 0, 0]], [QX, QX], [1.0, 1.0], [0.25, 0.25])
    assert abs(phi[0] - 0.5) < 1e-15 and np.allclose(n[0], [1, 0, 0], atol=1e-15)
    assert np.allclose(ra[0], [1.25, 0, 0], atol=1e-15) and np.allclose(rb[0], [-1.25, 0, 0], atol=1e-15)


def test_parallel_overlap_midpoint_rule(orc):
    """Side by side, projections overlap on [0.5, 1]: the contact sits at 0.75."""
    phi, n, ra, rb, st = _rods(orc, [[0, 0, 0], [1.5, 0.8, 0]], [QX, QX], [1.0, 1.0], [0.25, 0.25])
    assert abs(phi[0] - 0.3) < 1e-15 and np.allclose(n[0], [0, 1, 0], atol=1e-15)
    assert np.allclose(ra[0], [0.75, 0.25, 0], atol=1e-15) and np.allclose(rb[0], [-0.75, -0.25, 0], atol=1e-15)
    # antiparallel (B flipped) gives the same geometry
    qflip = [0.0, 0.0, 0.0, 1.0]  # 180 deg about z: body x -> -x
    phi2, n2, ra2, rb2, _ = _rods(orc, [[0, 0, 0], [1.5, 0.8, 0]], [QX, qflip], [1.0, 1.0], [0.25, 0.25])
    assert abs(phi2[0] - 0.3) < 1e-15 and np.allclose(ra2[0], ra[0], atol=1e-14)


def test_sphere_limit(orc):
    rng = np.random.default_rng(3)
    for _ in range(20):
        d = rng.normal(size=3)
        q = rng.normal(size=(2, 4))
        phi, n, *_ = _rods(orc, [[0, 0, 0], d], q, [0.0, 0.0], [0.3, 0.5])
        assert abs(phi[0] - (np.linalg.norm(d) - 0.8)) < 1e-14
        assert np.allclose(n[0], d / np.linalg.norm(d), atol=1e-14)


def _axis(q):
    q = np.asarray(q) / np.linalg.norm(q)
    s, x, y, z = q
    return np.array([1 - 2 * (y * y + z * z), 2 * (x * y + s * z), 2 * (x * z - s * y)])


def test_bruteforce_sampling_and_invariants(orc):
    rng = np.random.default_rng(11)
    m = 200
    pos = np.zeros((2 * m, 3))
    pos[1::2] = rng.uniform(-2.5, 2.5, size=(m, 3))
    quat = rng.normal(size=(2 * m, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    h = rng.uniform(0.5, 2.0, size=2 * m)
    r = rng.uniform(0.1, 0.3, size=2 * m)
    pairs = [(2 * k, 2 * k + 1) for k in range(m)]
    phi, n, ra, rb, st = _rods(orc, pos, quat, h, r, pairs)
    ts = np.linspace(-1.0, 1.0, 1201)
    for k, (a, b) in enumerate(pairs):
        if st[k] != 0:
            continue
        A = pos[a] + np.outer(ts * h[a], _axis(quat[a]))
        B = pos[b] + np.outer(ts * h[b], _axis(quat[b]))
        dmin = np.sqrt(((A[:, None, :] - B[None, :, :]) ** 2).sum(-1)).min()
        exact = phi[k] + r[a] + r[b]
        assert exact <= dmin + 1e-12 and dmin - exact <= 2e-3 * (h[a] + h[b])
        # collinearity y_b - y_a = Phi n and unit normal
        gap = pos[b] + rb[k] - pos[a] - ra[k]
        assert np.allclose(gap, phi[k] * n[k], atol=1e-13)
        assert abs(np.linalg.norm(n[k]) - 1) < 1e-14
    # swap symmetry
    sw = [(b, a) for a, b in pairs]
    phi2, n2, *_ = _rods(orc, pos, quat, h, r, sw)
    assert np.allclose(phi2, phi, atol=1e-13) and np.allclose(n2, -n, atol=1e-12)


def test_mixed_shapes_undefined(orc):
    pos = np.array([[0, 0, 0], [3, 0, 0.0]])
    axes = np.array([[1, 0.5, 0.5], [1, 0.25, 0.25]])
    phi, n, ra, rb, st = orc.snsd(pos, np.array([QX, QX]), axes, None, [0], [1], shape=np.array([0, 1], np.int32))
    assert st[0] == 2 and math.isnan(phi[0])


def test_rod_colony_recipe(orc):
    sc = scenes.colony_rods(n=1500)
    assert np.all(sc["shape"] == 1)
    ell = 2 * (sc["axes"][:, 0] + sc["axes"][:, 1])  # tip-to-tip length (R22)
    assert ell.min() >= 2.0 and ell.max() <= 4.0 * math.exp(sc["dt"]) + 1e-12
    rad = orc.bounding_radius(sc["axes"], sc["shape"])
    pi, pj = orc.broadphase(sc["pos"], rad, None, 0.1)
    phi, n, *_ = orc.snsd(sc["pos"], sc["quat"], sc["axes"], None, pi, pj, shape=sc["shape"])
    assert np.all(np.isfinite(phi))
    assert phi.min() > -0.06  # growth overlaps only (l e^dt - l <= 0.04 per rod)
    assert np.max(np.abs(n[:, 2])) < 1e-12  # planar


@pytest.mark.parametrize("dt", [1e-3])
def test_rod_step_resolves_growth_overlap(orc, dt):
    """One overdamped ReLCP step of a small rod colony ends with no overlap
    beyond eps_NCP (stopping rule)."""
    sc = scenes.colony_rods(n=300, dt=1e-2)
    r = orc.relcp_step(sc, lcp_tol=1e-10, max_recursions=10)
    assert r["status"] == 0 and r["max_overlap"] <= sc["eps_ncp"]
