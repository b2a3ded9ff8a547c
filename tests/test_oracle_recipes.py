"""CPU pins for the cfg3 / cfg4 input recipes and the oracle on them.

cfg3 (planar colony): the construction is disjoint before growth (every
oracle SNSD of candidate pairs > 0), z-reflection symmetry makes every SNSD
normal in-plane (|n_z| at rounding level), ~3 contacts per body (BASELINE).
cfg4 (chainmail network): link / row counts, n opposes separation, |r| <= 1.2,
kinematic boundary rows; the oracle's LCP satisfies the KKT conditions
 and D lambda is unique across warm starts although lambda is not
(Lemma 5)."""
import numpy as np

from gen import scenes


def test_cfg3_disjoint_before_growth_and_planar(orc):
    sc = scenes.cfg3(n=1200, growth=0.0)
    pi, pj = orc.broadphase(sc["pos"], sc["axes"].max(1), None, 0.1)
    phi, n, ra, rb, st = orc.snsd(sc["pos"], sc["quat"], sc["axes"], None, pi, pj)
    assert np.all(st == 0)
    assert phi.min() > 0.0
    assert np.max(np.abs(n[:, 2])) < 1e-11
    contacts = 2 * np.sum(phi < 0.1) / sc["n"]
    assert 2.0 < contacts < 4.5
    assert np.all(sc["pos"][:, 2] == 0.0)


def test_cfg3_growth_creates_overlaps(orc):
    sc = scenes.cfg3(n=1200)
    assert sc["growing"].sum() == 600
    pi, pj = orc.broadphase(sc["pos"], sc["axes"].max(1), None, 0.1)
    phi, *_ = orc.snsd(sc["pos"], sc["quat"], sc["axes"], None, pi, pj)
    assert phi.min() < 0.0 and phi.min() > -0.03  # at most growth + gap deep


def test_cfg4_network_recipe():
    k = 12
    sc = scenes.cfg4(n_side=k)
    net = sc["network"]
    links = 2 * k * (k - 1)
    pairs = np.unique(np.stack([net["ia"], net["ib"]], 1), axis=0)
    assert len(pairs) == links
    _, cnt = np.unique(net["ia"].astype(np.int64) * k * k + net["ib"], return_counts=True)
    assert cnt.min() >= 1 and cnt.max() <= 3
    e = sc["pos"][net["ib"]] - sc["pos"][net["ia"]]
    e /= np.linalg.norm(e, axis=1, keepdims=True)
    assert np.all(np.einsum("ij,ij->i", net["n"], e) < 0)  # n opposes separation
    assert np.allclose(np.linalg.norm(net["n"], axis=1), 1.0, atol=1e-15)
    assert np.all(np.linalg.norm(net["ra"], axis=1) <= 1.2 + 1e-12)
    assert np.all(np.linalg.norm(net["rb"], axis=1) <= 1.2 + 1e-12)
    key = net["ia"].astype(np.int64) << 32 | net["ib"]
    assert np.all(np.diff(key) >= 0)
    kin = sc["kinematic"].reshape(k, k)
    assert kin[0].all() and kin[-1].all() and not kin[1:-1].any()
    vy = sc["vel"][:, 1].reshape(k, k)
    assert np.allclose(vy[0], -1) and np.allclose(vy[-1], 1)


def test_cfg4_oracle_kkt_and_unique_wrench(orc):
    sc = scenes.cfg4(n_side=10, c_fixed=3)
    x, g, info, W, rw = orc.network_lcp(sc, 1e-11)
    assert info["converged"]
    assert np.all(x >= 0) and np.all(g >= -1e-11)
    assert np.max(np.abs(np.minimum(x, g))) <= 1e-11
    # A = s (W^1/2 D)^T (W^1/2 D): Lemma 5 fixes W D lambda (= U); the wrench D
    # lambda itself is fixed only on bodies with W > 0 (kinematic rows absorb any)
    F1, U1 = orc.wrench(W, rw["ia"], rw["ib"], rw["n"], rw["ta"], rw["tb"], x)
    x0 = np.random.default_rng(0).uniform(0, 2 * x.max(), size=len(x))
    x2, g2, info2 = orc.bbpgd(W, rw["ia"], rw["ib"], rw["n"], rw["ta"], rw["tb"], rw["s"], rw["q"], x0, 1e-11)
    F2, U2 = orc.wrench(W, rw["ia"], rw["ib"], rw["n"], rw["ta"], rw["tb"], x2)
    assert np.max(np.abs(x - x2)) > 1e-3 * np.max(np.abs(x))  # lambda is not unique here
    assert np.max(np.abs(U1 - U2)) <= 1e-6 * np.max(np.abs(U1))
    free = sc["kinematic"] == 0
    assert np.max(np.abs(F1[free] - F2[free])) <= 1e-6 * np.max(np.abs(F1[free]))
    assert np.max(np.abs(g - g2)) <= 1e-9
