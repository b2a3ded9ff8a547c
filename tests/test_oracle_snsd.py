"""Pins for the oracle's shared-normal signed distance (SNSD).

Every check here is fixed by something other than the oracle itself: closed
forms (spheres, aligned axes), the exact signed distance to the Minkowski sum
2E for identical translates (the paper's §5.2 geometry), a dense
surface-sampling brute force, and the geometric identities the paper states
(P:L678-680 y_b - y_a = Phi n; P:L207-211 rate = row . U)."""
import math

import numpy as np
import pytest
from scipy.spatial import cKDTree

from gen import scenes


def _rotz(theta):
    return np.array([math.cos(theta / 2), 0.0, 0.0, math.sin(theta / 2)])


def _ellipsoid_signed_distance(p, e):
    """Signed distance from point p (body frame) to the ellipsoid with
    semi-axes e: the foot x_i = p_i e_i^2/(e_i^2 + t) with
    sum (e_i p_i/(e_i^2+t))^2 = 1; F(t) is decreasing on (-min e^2, inf),
    so bisection finds the unique root there (the nearest foot)."""
    e = np.asarray(e, float)
    p = np.asarray(p, float)

    def F(t):
        return np.sum((e * p / (e * e + t)) ** 2) - 1.0

    lo = -np.min(e * e) * (1 - 1e-15)
    hi = max(1.0, 10 * np.linalg.norm(p) * np.max(e))
    while F(hi) > 0:
        hi *= 2
    for _ in range(300):
        mid = 0.5 * (lo + hi)
        if F(mid) > 0:
            lo = mid
        else:
            hi = mid
    t = 0.5 * (lo + hi)
    x = p * e * e / (e * e + t)
    inside = np.sum((p / e) ** 2) < 1.0
    dist = np.linalg.norm(p - x)
    nrm = x / (e * e)                      # outward normal of the ellipsoid at the foot x
    nrm /= np.linalg.norm(nrm)
    return (-dist if inside else dist), nrm


def test_sphere_limit_closed_form(orc):
    """e1=e2=e3: Phi = |d| - r_a - r_b, n = d/|d|."""
    rng = np.random.default_rng(11)
    P = 200
    pos = rng.uniform(-3, 3, size=(2 * P, 3))
    quat = rng.standard_normal((2 * P, 4))
    r = rng.uniform(0.3, 1.5, size=2 * P)
    axes = np.repeat(r[:, None], 3, axis=1)
    pi = np.arange(0, 2 * P, 2)
    pj = pi + 1
    phi, n, ra, rb, st = orc.snsd(pos, quat, axes, None, pi, pj)
    d = pos[pj] - pos[pi]
    dn = np.linalg.norm(d, axis=1)
    assert np.all(st == 0)
    np.testing.assert_allclose(phi, dn - r[pi] - r[pj], atol=1e-14 * 10, rtol=0)
    np.testing.assert_allclose(n, d / dn[:, None], atol=1e-12)
    # spec example: unit spheres at (0,0,0), (3,0,0) -> phi 1, n (1,0,0), y_a (1,0,0), y_b (2,0,0)
    phi1, n1, ra1, rb1, _ = orc.snsd(np.array([[0, 0, 0], [3, 0, 0.0]]), np.array([[1, 0, 0, 0.0]] * 2),
                                     np.ones((2, 3)), None, [0], [1])
    assert abs(phi1[0] - 1.0) < 1e-15
    np.testing.assert_allclose(ra1[0], [1, 0, 0], atol=1e-15)
    np.testing.assert_allclose(rb1[0] + [3, 0, 0], [2, 0, 0], atol=1e-15)


@pytest.mark.parametrize("dy", [3.0, 2.0, 1.2, 0.8, 0.5, 0.3])
def test_two_ellipsoid_section_5_2_exact(orc, dy):
    """§5.2 geometry: radii (1,1,2), both rotated 45 deg about z,
    centres offset 1 along x.  Identical translates: Phi(d) equals the signed
    distance from d to 2E (Minkowski sum), computed by 1-D bisection."""
    e = np.array([2.0, 1.0, 1.0])          # major axis in the x-y plane (R17)
    q = _rotz(math.pi / 4)
    pos = np.array([[0.0, 0.0, 0.0], [1.0, dy, 0.0]])
    phi, n, ra, rb, st = orc.snsd(pos, np.array([q, q]), np.array([e, e]), None, [0], [1])
    R = orc.quat_to_rot(q)
    p_body = R.T @ (pos[1] - pos[0])
    sd, nb = _ellipsoid_signed_distance(p_body, 2 * e)
    assert st[0] == 0
    assert abs(phi[0] - sd) <= 1e-13
    np.testing.assert_allclose(n[0], R @ nb, atol=1e-9)


def test_identical_translates_random(orc):
    """Random identical translates (any common orientation) vs 2E distance."""
    rng = np.random.default_rng(5)
    for _ in range(40):
        e = np.sort(rng.uniform(0.3, 1.2, 3))[::-1]
        q = rng.standard_normal(4)
        d = rng.standard_normal(3)
        d *= rng.uniform(0.6, 3.5) / np.linalg.norm(d)
        phi, n, *_ , st = orc.snsd(np.array([np.zeros(3), d]), np.array([q, q]), np.array([e, e]), None, [0], [1])
        R = orc.quat_to_rot(q)
        sd, _ = _ellipsoid_signed_distance(R.T @ d, 2 * e)
        assert abs(phi[0] - sd) <= 1e-12, (phi[0], sd)


def test_aligned_axes_closed_form(orc):
    """Identical aligned ellipsoids separated along principal axis k:
    Phi = D - 2 e_k exactly."""
    e = np.array([1.0, 0.6, 0.4])
    for k in range(3):
        for D in [2 * e[k] + 0.5, 2 * e[k] + 1e-3, 2 * e[k] + 3.0]:
            d = np.zeros(3)
            d[k] = D
            phi, n, *_ = orc.snsd(np.array([np.zeros(3), d]), np.array([[1, 0, 0, 0.0]] * 2),
                                  np.array([e, e]), None, [0], [1])
            assert abs(phi[0] - (D - 2 * e[k])) < 1e-14
            assert abs(n[0][k] - 1.0) < 1e-14


def _random_pairs(rng, P, sep_range):
    axes = np.stack([np.ones(2 * P), rng.uniform(0.25, 1.0, 2 * P), rng.uniform(0.25, 1.0, 2 * P)], 1)
    axes = -np.sort(-axes, axis=1)
    quat = rng.standard_normal((2 * P, 4))
    pos = np.zeros((2 * P, 3))
    dirs = rng.standard_normal((P, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    pos[1::2] = dirs * rng.uniform(*sep_range, size=(P, 1))
    return pos, quat, axes, np.arange(0, 2 * P, 2), np.arange(1, 2 * P, 2)


def test_snsd_invariants(orc):
    """Collinearity y_b - y_a = Phi n; y on both surfaces;
    swap symmetry; |n| = 1 -- over separated, touching and overlapping pairs."""
    rng = np.random.default_rng(7)
    pos, quat, axes, pi, pj = _random_pairs(rng, 300, (0.6, 3.5))
    phi, n, ra, rb, st = orc.snsd(pos, quat, axes, None, pi, pj)
    assert np.all(st == 0)
    ya = pos[pi] + ra
    yb = pos[pj] + rb
    resid = np.linalg.norm(yb - ya - phi[:, None] * n, axis=1)
    assert np.all(resid <= 1e-12 * np.maximum(1, np.abs(phi)))
    np.testing.assert_allclose(np.linalg.norm(n, axis=1), 1.0, atol=1e-15)
    for r, idx in ((ra, pi), (rb, pj)):
        R = orc.quat_to_rot(quat[idx])
        body = np.einsum("nji,nj->ni", R, r) / axes[idx]
        np.testing.assert_allclose(np.linalg.norm(body, axis=1), 1.0, atol=1e-13)
    phi2, n2, ra2, rb2, _ = orc.snsd(pos, quat, axes, None, pj, pi)
    np.testing.assert_allclose(phi2, phi, atol=1e-12)
    np.testing.assert_allclose(n2, -n, atol=1e-9)
    assert (phi < 0).sum() > 30 and (phi > 0).sum() > 30


def test_snsd_vs_dense_surface_sampling(orc):
    """Separated random pairs: the minimum distance over dense surface samples
    bounds Phi from above and converges to it (P:L225 definition)."""
    rng = np.random.default_rng(3)
    pos, quat, axes, pi, pj = _random_pairs(rng, 6, (2.3, 3.0))
    phi, *_ = orc.snsd(pos, quat, axes, None, pi, pj)
    m = 120000
    k = np.arange(m) + 0.5
    z = 1 - 2 * k / m
    r = np.sqrt(1 - z * z)
    th = math.pi * (3 - math.sqrt(5)) * k
    unit = np.stack([r * np.cos(th), r * np.sin(th), z], 1)
    for p in range(len(pi)):
        a, b = pi[p], pj[p]
        pts = []
        for idx in (a, b):
            R = orc.quat_to_rot(quat[idx])
            pts.append(pos[idx] + (unit * axes[idx]) @ R.T)
        if phi[p] <= 0:
            continue
        dmin, _ = cKDTree(pts[1]).query(pts[0], k=1)
        bf = dmin.min()
        assert phi[p] <= bf + 1e-12
        assert bf <= phi[p] + 2e-2


def test_rows_match_finite_difference_rate(orc):
    """Linearised rate Phi_dot = row . U: central finite
    difference of Phi under the rigid motion x += eps u, q += eps/2 (0,w) q."""
    rng = np.random.default_rng(9)
    pos, quat, axes, pi, pj = _random_pairs(rng, 40, (0.8, 3.0))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    phi, n, ra, rb, st = orc.snsd(pos, quat, axes, None, pi, pj)
    ta, tb = orc.rows(n, ra, rb)
    U = rng.standard_normal((len(pos), 6))
    rate = (-(n * U[pi, :3]).sum(1) - (ta * U[pi, 3:]).sum(1) + (n * U[pj, :3]).sum(1) + (tb * U[pj, 3:]).sum(1))
    h = 1e-6

    def moved(eps):
        w = U[:, 3:]
        qdot = np.empty_like(quat)
        qdot[:, 0] = -0.5 * (w * quat[:, 1:]).sum(1)
        qdot[:, 1:] = 0.5 * (quat[:, :1] * w + np.cross(w, quat[:, 1:]))
        return pos + eps * U[:, :3], quat + eps * qdot

    pp, qp = moved(h)
    pm, qm = moved(-h)
    fp = orc.snsd(pp, qp, axes, None, pi, pj)[0]
    fm = orc.snsd(pm, qm, axes, None, pi, pj)[0]
    fd = (fp - fm) / (2 * h)
    np.testing.assert_allclose(rate, fd, atol=1e-6 * (1 + np.abs(rate)).max())


def test_cfg1_pair_counts_and_degenerate(orc):
    """cfg1 recipe realises ~2.6k candidates and ~430 near pairs;
    coincident centres report status 1 (reading R4)."""
    sc = scenes.cfg1()
    rad = sc["axes"].max(1)
    pi, pj = orc.broadphase(sc["pos"], rad, sc["box"], 0.1)
    assert 2000 < len(pi) < 3200
    phi, *_, st = orc.snsd(sc["pos"], sc["quat"], sc["axes"], sc["box"], pi, pj)
    assert np.all(st == 0)
    assert 300 < (phi < 0.1).sum() < 600
    _, _, _, _, st = orc.snsd(np.zeros((2, 3)), np.array([[1, 0, 0, 0.0]] * 2), np.ones((2, 3)), None, [0], [1])
    assert st[0] == 1


def _fib(N):
    k = np.arange(N) + 0.5
    z = 1 - 2 * k / N
    r = np.sqrt(1 - z * z)
    th = math.pi * (3 - math.sqrt(5)) * k
    return np.stack([r * np.cos(th), r * np.sin(th), z], 1)


def _overlap_family_pairs(rng, P):
    """Overlapping, NON-identical pairs (independent orientations) of the
    BASELINE shape families: cfg5 (1, 0.6, 0.4), cfg2 (1, 1/r, 1/r) with
    aspect ratio r up to 4, cfg1 (1, 0.5, 0.5), and cfg5 vs cfg2 mixed;
    centre offsets from moderate to deep (|d| ~ U(0.02, 1.6))."""
    fam = rng.integers(0, 4, P)

    def shape(f):
        if f == 0:
            return [1.0, 0.6, 0.4]
        if f == 1:
            r = rng.uniform(1.0, 4.0)
            return [1.0, 1.0 / r, 1.0 / r]
        return [1.0, 0.5, 0.5]

    axes = []
    for f in fam:
        axes += [shape(0), shape(1)] if f == 3 else [shape(f), shape(f)]
    axes = np.array(axes)
    quat = rng.standard_normal((2 * P, 4))
    pos = np.zeros((2 * P, 3))
    d = rng.standard_normal((P, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    pos[1::2] = d * np.where(rng.uniform(size=(P, 1)) < 0.5, rng.uniform(0.02, 0.7, (P, 1)),
                             rng.uniform(0.7, 1.6, (P, 1)))
    return pos, quat, axes, np.arange(0, 2 * P, 2), np.arange(1, 2 * P, 2)


def test_snsd_overlap_global_max_dense_directions(orc):
    """Phi = max_{|n|=1} f(n), f(n) = n.d - h_a(n) - h_b(n) (P:L225,
    P:L678-680) for >= 200 overlapping non-identical pairs, against a brute
    force over 10^6 Fibonacci directions evaluated from the definition
    (Sigma = R diag(e^2) R^T, h = sqrt(n^T Sigma n), written out here):
      * Phi_bf <= Phi + 1e-12: no sampled direction beats the oracle's maximum
        (a missed global maximum shows up here);
      * Phi - Phi_bf <= L_f delta: the sample comes within its covering radius
        delta of the maximiser, |grad f| <= L_f = |d| + max e_a + max e_b.
    The same check on the single-start (d/|d| only) variant of the oracle's
    Newton must FAIL on some deep overlaps: the pin sees a lost multistart."""
    rng = np.random.default_rng(17)
    pos, quat, axes, pi, pj = _overlap_family_pairs(rng, 320)
    phi, n, ra, rb, st = orc.snsd(pos, quat, axes, None, pi, pj)
    phi1, *_ = orc.snsd(pos, quat, axes, None, pi, pj, n_fib=0)  # d/|d| start only
    ov = phi < 0
    assert ov.sum() >= 200 and np.all(st[ov] == 0)
    N = 1_000_000
    U = _fib(N)
    Q = np.stack([U[:, 0] ** 2, U[:, 1] ** 2, U[:, 2] ** 2, 2 * U[:, 0] * U[:, 1], 2 * U[:, 0] * U[:, 2],
                  2 * U[:, 1] * U[:, 2]], 1)
    q = quat / np.linalg.norm(quat, axis=1, keepdims=True)
    s, w = q[:, 0], q[:, 1:]
    K = np.zeros((len(q), 3, 3))
    K[:, 0, 1], K[:, 0, 2], K[:, 1, 2] = -w[:, 2], w[:, 1], -w[:, 0]
    K[:, 1, 0], K[:, 2, 0], K[:, 2, 1] = w[:, 2], -w[:, 1], w[:, 0]
    R = np.eye(3) + 2 * s[:, None, None] * K + 2 * K @ K
    S = np.einsum("nik,nk,njk->nij", R, axes ** 2, R)
    sv = np.stack([S[:, 0, 0], S[:, 1, 1], S[:, 2, 2], S[:, 0, 1], S[:, 0, 2], S[:, 1, 2]], 1)
    d = pos[pj] - pos[pi]
    bf = np.empty(len(pi))
    for c in range(0, len(pi), 16):
        sl = slice(c, c + 16)
        f = U @ d[sl].T - np.sqrt(Q @ sv[pi[sl]].T) - np.sqrt(Q @ sv[pj[sl]].T)
        bf[sl] = f.max(0)
    # covering radius of the direction sample: farthest of 2e5 random probes
    probe = rng.standard_normal((200_000, 3))
    probe /= np.linalg.norm(probe, axis=1, keepdims=True)
    chord, _ = cKDTree(U).query(probe, k=1)
    delta = 2.0 * np.arcsin(chord.max() / 2.0) * 1.25
    Lf = np.linalg.norm(d, axis=1) + axes[pi].max(1) + axes[pj].max(1)
    assert np.all(bf[ov] <= phi[ov] + 1e-12), (bf - phi)[ov].max()
    assert np.all(phi[ov] - bf[ov] <= Lf[ov] * delta)
    assert np.max(phi[ov] - bf[ov]) < 1e-4  # the sample's actual miss is O(delta^2)
    assert np.any(bf[ov] > phi1[ov] + 1e-6), "d/|d|-only Newton passed: the pin is blind to the multistart"
