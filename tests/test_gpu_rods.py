"""Spherocylinder path (P:L1056 segment distance
minus cap radii) on the GPU against the oracle: SNSD of random and parallel
rod pairs, generation on the rod-colony recipe (bit-exact lists), one
ReLCP step, the growth driver (l_dot = l), and the mixed-shape refusal."""
import math

import numpy as np
import pytest

from gen import scenes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    from paper_2506_14097_b200 import relcp
    relcp.load()
    return relcp


def _ctx(R, sc, **kw):
    p = dict(dynamics=sc["dynamics"], dt=sc["dt"], cutoff=sc["cutoff"], eps_ncp=sc["eps_ncp"],
             box=list(sc["box"]), xi=sc.get("xi", 1.0))
    p.update(kw)
    return R.Context(**p)


def test_rod_snsd_parity(orc, R):
    rng = np.random.default_rng(21)
    m = 4000
    pos = np.zeros((2 * m, 3))
    pos[1::2] = rng.uniform(-2.5, 2.5, size=(m, 3))
    quat = rng.normal(size=(2 * m, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    # a block of exactly parallel pairs (shared orientation) for the midpoint rule
    quat[1:400:2] = quat[0:400:2]
    axes = np.zeros((2 * m, 3))
    axes[:, 0] = rng.uniform(0.0, 2.0, size=2 * m)
    axes[:, 1] = axes[:, 2] = rng.uniform(0.1, 0.3, size=2 * m)
    shape = np.ones(2 * m, dtype=np.int32)
    pi = np.arange(0, 2 * m, 2, dtype=np.int32)
    pj = pi + 1
    phi_r, n_r, ra_r, rb_r, st_r = orc.snsd(pos, quat, axes, None, pi, pj, shape=shape)
    ctx = R.Context(dynamics=1, dt=1e-2)
    bodies = R.BodyState(pos, quat, axes, shape=shape)
    phi, n, ra, rb, st = (t.cpu().numpy() for t in ctx.snsd_pairs(bodies, pi, pj))
    assert np.array_equal(st, st_r)
    ok = st_r == 0
    assert ok.sum() > 3900
    assert np.max(np.abs(phi[ok] - phi_r[ok])) <= 1e-12 * 5
    assert np.max(np.abs(n.T[ok] - n_r[ok])) <= 1e-10
    assert np.max(np.abs(ra.T[ok] - ra_r[ok])) <= 1e-9 and np.max(np.abs(rb.T[ok] - rb_r[ok])) <= 1e-9


def test_rod_colony_generate_parity(orc, R):
    sc = scenes.colony_rods(n=1500)
    r = orc.relcp_step(sc, snsd_only=True, lcp_tol=1e-10)
    c = r["constraints"]
    ctx = _ctx(R, sc)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(8 * sc["n"])
    n0, _ = ctx.generate_contacts(bodies, cs)
    pi, pj = (t.cpu().numpy() for t in ctx.get_pairs())
    assert np.array_equal(pi, r["pairs"][0]) and np.array_equal(pj, r["pairs"][1])
    g = cs.to_numpy()
    assert n0 == len(c["ia"]) and np.array_equal(g["ia"], c["ia"]) and np.array_equal(g["ib"], c["ib"])
    assert np.max(np.abs(g["phi"] - c["phi"])) <= 1e-12 * 10
    assert np.max(np.abs(g["n"] - c["n"])) <= 1e-10
    assert np.max(np.abs(g["q"] - r["q_hist"][0])) <= 1e-11


def test_rod_colony_step_parity(orc, R):
    sc = scenes.colony_rods(n=800)
    r = orc.relcp_step(sc, lcp_tol=1e-12, max_recursions=5)
    ctx = _ctx(R, sc, lcp_tol=1e-12, max_recursions=5, lcp_max_iter=2_000_000)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(16 * sc["n"])
    rep = ctx.step(bodies, cs)
    assert rep["n_c"] == r["n_c"] and rep["recursions"] == r["recursions"]
    assert np.max(np.abs(bodies.pos.cpu().numpy() - r["pos"])) <= 1e-9
    assert np.max(np.abs(bodies.quat.cpu().numpy() - r["quat"])) <= 1e-9
    assert rep["max_overlap"] <= sc["eps_ncp"] or rep["status"] != 0


def test_rod_growth_driver(orc, R):
    from paper_2506_14097_b200 import drivers as D
    sc = scenes.colony_rods(n=500)
    ref = dict(sc)
    ref["pos"], ref["quat"], ref["axes"] = sc["pos"].copy(), sc["quat"].copy(), sc["axes"].copy()
    n_c = []
    for k in range(3):
        if k > 0:  # l_dot = l on the tip-to-tip length l = 2 (a0 + r) (R22)
            ref["axes"][:, 0] = (ref["axes"][:, 0] + ref["axes"][:, 1]) * math.exp(sc["dt"]) - ref["axes"][:, 1]
        rr = orc.relcp_step(ref, lcp_tol=1e-12, max_recursions=3)
        ref["pos"], ref["quat"] = rr["pos"], rr["quat"]
        n_c.append(rr["n_c"])
    reps, bodies, cs = D.growth(sc, steps=3, lcp_tol=1e-12, lcp_max_iter=2_000_000, max_recursions=3)
    assert [x["n_c"] for x in reps] == n_c
    assert np.max(np.abs(bodies.axes.cpu().numpy() - ref["axes"])) <= 1e-15
    assert np.max(np.abs(bodies.pos.cpu().numpy() - ref["pos"])) <= 1e-8


def test_mixed_shapes_refused(R):
    pos = np.array([[0, 0, 0], [2.0, 0, 0.0]])  # inside the broadphase range 1 + 1.25 + 0.1
    quat = np.array([[1.0, 0, 0, 0]] * 2)
    axes = np.array([[1, 0.5, 0.5], [1, 0.25, 0.25]])
    ctx = R.Context(dynamics=1, dt=1e-2)
    bodies = R.BodyState(pos, quat, axes, shape=np.array([0, 1], np.int32))
    cs = R.ConstraintStore(8)
    with pytest.raises(R.RelcpError) as e:
        ctx.generate_contacts(bodies, cs)
    assert e.value.code == R.E_DEGENERATE


def _divide_np(sc, l0, rng):
    """Test-side twin of drivers.divide_rods (reading R28, P:L1030-1032,
    P:L1056), written independently in numpy: rods of tip-to-tip length
    l = 2 (a0 + r) >= 2 l0 become two daughters of length l/2 (centreline
    l/2 - 2r) at x -+ (l/4) u, each turned by a random +-0.01 degrees about z;
    daughter B appended in mother order."""
    a = sc["axes"]
    idx = np.flatnonzero(2.0 * (a[:, 0] + a[:, 1]) >= 2.0 * l0)
    m = len(idx)
    if m == 0:
        return sc, 0
    out = dict(sc)
    q = sc["quat"][idx] / np.linalg.norm(sc["quat"][idx], axis=1)[:, None]
    s, x, y, z = q.T
    u = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y + s * z), 2 * (x * z - s * y)], 1)
    r = a[idx, 1]
    ell = 2.0 * (a[idx, 0] + r)
    off = (0.25 * ell)[:, None] * u
    sg = rng.choice(np.array([-1.0, 1.0]), size=(m, 2))
    th = 0.5 * (0.01 * math.pi / 180.0) * sg

    def rot(t):  # q_z(2 t) q: (cos t, 0, 0, sin t) (x) q
        c, sn = np.cos(t), np.sin(t)
        return np.stack([c * s - sn * z, c * x - sn * y, c * y + sn * x, c * z + sn * s], 1)

    pos, quat, axes = sc["pos"].copy(), sc["quat"].copy(), sc["axes"].copy()
    x0 = pos[idx].copy()
    pos[idx] = x0 - off
    quat[idx] = rot(th[:, 0])
    axes[idx, 0] = 0.25 * ell - r
    new_axes = np.stack([0.25 * ell - r, r, a[idx, 2]], 1)
    out["pos"] = np.concatenate([pos, x0 + off])
    out["quat"] = np.concatenate([quat, rot(th[:, 1])])
    out["axes"] = np.concatenate([axes, new_axes])
    for k in ("vel",):
        out[k] = np.concatenate([sc[k], np.zeros((m, 6))])
    for k in ("inv_mass", "inv_inertia", "kinematic", "shape", "growing"):
        if k in sc and sc[k] is not None:
            out[k] = np.concatenate([sc[k], sc[k][idx]])
    out["n"] = len(out["pos"])
    return out, m


def test_rod_division_driver(orc, R):
    """The dividing colony (cells divide into two upon reaching
    2 l_0, daughters turned by +-0.01 degrees): three steps of the GPU
    driver (drivers.colony) against the oracle stepping a numpy twin of the
    same growth and division rule (R22, R28): body counts, rows per LCP and the
    accepted configurations agree, and every step ends below eps_NCP."""
    from paper_2506_14097_b200 import drivers as D
    sc = scenes.colony_rods(n=400)
    l0, seed = 2.0, 1030
    rng = np.random.Generator(np.random.PCG64(seed))
    ref = dict(sc)
    counts, n_c, divs = [], [], []
    for k in range(3):
        m = 0
        if k > 0:
            ref["axes"] = ref["axes"].copy()
            ref["axes"][:, 0] = (ref["axes"][:, 0] + ref["axes"][:, 1]) * math.exp(sc["dt"]) - ref["axes"][:, 1]
            ref, m = _divide_np(ref, l0, rng)
        rr = orc.relcp_step(ref, lcp_tol=1e-12, max_recursions=5)
        ref["pos"], ref["quat"] = rr["pos"], rr["quat"]
        counts.append(ref["n"])
        n_c.append(rr["n_c"])
        divs.append(m)
    reps, bodies, cs = D.colony(sc, steps=3, l0=l0, seed=seed, lcp_tol=1e-12, lcp_max_iter=2_000_000,
                                max_recursions=5)
    assert divs[1] > 0, "the recipe must divide some cells in the first steps"
    assert [x["divisions"] for x in reps] == divs
    assert [x["n_bodies"] for x in reps] == counts
    assert [x["n_c"] for x in reps] == n_c
    assert np.max(np.abs(bodies.axes.cpu().numpy() - ref["axes"])) <= 1e-15
    assert np.max(np.abs(bodies.pos.cpu().numpy() - ref["pos"])) <= 1e-8
    assert all(x["max_overlap"] <= sc["eps_ncp"] for x in reps)
