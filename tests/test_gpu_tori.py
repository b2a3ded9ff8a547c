"""Torus path (P:L1080 centreline-circle distance
minus the minor radii) on the GPU against the oracle: SNSD of random pairs,
the chain-link closed form, the set-valued selection rule (R23), and
generation + a ReLCP step on a linked chain of rings."""
import math

import numpy as np
import pytest

from gen import scenes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

S2 = math.sqrt(0.5)


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


def test_torus_snsd_parity(orc, R):
    rng = np.random.default_rng(31)
    m = 1500
    pos = np.zeros((2 * m, 3))
    pos[1::2] = rng.uniform(-2.0, 2.0, size=(m, 3))
    quat = rng.normal(size=(2 * m, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    axes = np.zeros((2 * m, 3))
    axes[:, 0] = rng.uniform(0.5, 1.2, size=2 * m)
    axes[:, 1] = axes[:, 2] = rng.uniform(0.05, 0.2, size=2 * m)
    # chain link and concentric (set-valued) pairs appended
    pos = np.vstack([pos, [[0, 0, 0], [1.4, 0, 0], [0, 0, 0], [0, 0, 0]]])
    quat = np.vstack([quat, [[1, 0, 0, 0], [S2, -S2, 0, 0], [1, 0, 0, 0], [1, 0, 0, 0]]])
    axes = np.vstack([axes, [[1, .2, .2], [1, .2, .2], [1, .1, .1], [2, .1, .1]]])
    shape = np.full(len(pos), 2, dtype=np.int32)
    pi = np.concatenate([np.arange(0, 2 * m, 2), [2 * m, 2 * m + 2]]).astype(np.int32)
    pj = pi + 1
    phi_r, n_r, ra_r, rb_r, st_r = orc.snsd(pos, quat, axes, None, pi, pj, shape=shape)
    ctx = R.Context(dynamics=0, dt=1e-3)
    bodies = R.BodyState(pos, quat, axes, shape=shape)
    phi, n, ra, rb, st = (t.cpu().numpy() for t in ctx.snsd_pairs(bodies, pi, pj))
    assert np.array_equal(st, st_r) and np.all(st == 0)
    assert np.max(np.abs(phi - phi_r)) <= 1e-12 * 5
    assert np.max(np.abs(n.T - n_r)) <= 1e-10
    assert np.max(np.abs(ra.T - ra_r)) <= 1e-9 and np.max(np.abs(rb.T - rb_r)) <= 1e-9
    assert abs(phi[-2] - 0.2) < 1e-13 and abs(phi[-1] - 0.8) < 1e-13


def test_torus_chain_generate_and_step_parity(orc, R):
    sc = scenes.chain_tori(n=60)
    r0 = orc.relcp_step(sc, snsd_only=True, lcp_tol=1e-10)
    ctx = _ctx(R, sc, lcp_tol=1e-12, max_recursions=5, lcp_max_iter=2_000_000)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(16 * sc["n"])
    n0, _ = ctx.generate_contacts(bodies, cs)
    c0 = r0["constraints"]
    g = cs.to_numpy()
    assert n0 == len(c0["ia"]) == sc["n"] - 1  # one contact per link
    assert np.array_equal(g["ia"], c0["ia"]) and np.array_equal(g["ib"], c0["ib"])
    assert np.max(np.abs(g["n"] - c0["n"])) <= 1e-10
    r = orc.relcp_step(sc, lcp_tol=1e-12, max_recursions=5)
    bodies = R.BodyState.from_scene(sc)
    rep = ctx.step(bodies, cs)
    assert rep["n_c"] == r["n_c"] and rep["recursions"] == r["recursions"]
    assert np.max(np.abs(bodies.pos.cpu().numpy() - r["pos"])) <= 1e-9
    assert np.max(np.abs(bodies.vel.cpu().numpy() - r["vel"])) <= 1e-6 * np.max(np.abs(r["vel"]))
