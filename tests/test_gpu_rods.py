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
        if k > 0:
            ref["axes"][:, 0] *= math.exp(sc["dt"])
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
