"""GPU checks at BASELINE.json's FULL sizes, in the launch configuration
bench.py times (same kernels, same grids).  The oracle cannot run whole
2M-body steps, so these compare (a) outputs the oracle computes completely
from generator inputs (Delassus apply / wrench on a 2M-body, 10M-row
network), (b) sampled outputs the oracle computes one by one (SNSD of sampled
candidate pairs, broadphase inside a sub-box), and (c) properties that hold
at any size: sorted store, q retention, lambda >= 0, KKT residual,
Newton's third law (linear momentum is conserved), planar
symmetry of cfg3, zero velocity change of kinematic bodies in cfg4."""
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


@pytest.mark.parametrize("shuffled,layout", [(False, 0), (True, 0), (False, 1)])
def test_fullsize_delassus_apply(orc, R, shuffled, layout):
    """2M bodies, 10M rows (cfg5 scale): every output against the oracle at
    1e-12; the shuffled store exercises the general (unsorted) CSR path,
    layout 1 the JDS operator."""
    b, ia, ib, n, ra, rb = scenes.random_constraint_network(2_000_000, 10_000_000, 77)
    if shuffled:
        p = np.random.default_rng(5).permutation(len(ia))
        ia, ib, n, ra, rb = ia[p], ib[p], n[p], ra[p], rb[p]
    ta, tb = np.cross(ra, n), np.cross(rb, n)
    W = orc.body_W(b)
    x = np.random.default_rng(1).standard_normal(len(ia))
    s = 1e-6
    y_ref = orc.delassus_apply(W, ia, ib, n, ta, tb, s, x)
    F_ref, U_ref = orc.wrench(W, ia, ib, n, ta, tb, x)
    ctx = _ctx(R, dict(dynamics=0, dt=1e-3, cutoff=0.1, eps_ncp=1e-5, box=[0, 0, 0]), layout=layout)
    bodies = R.BodyState.from_scene(b)
    cs = R.ConstraintStore.from_rows(ia, ib, n, ta, tb)
    ctx.prepare_operator(bodies, cs)
    assert ctx.stats()["op_layout"] == layout
    xd = torch.as_tensor(x, device="cuda")
    yd = torch.empty_like(xd)
    ctx.delassus_apply(bodies, cs, xd, yd, s)
    assert np.max(np.abs(yd.cpu().numpy() - y_ref)) <= 1e-12 * np.max(np.abs(y_ref))
    F = torch.empty(b["n"], 6, dtype=torch.float64, device="cuda")
    U = torch.empty_like(F)
    ctx.wrench(bodies, cs, xd, F, U)
    assert np.max(np.abs(F.cpu().numpy() - F_ref)) <= 1e-12 * np.max(np.abs(F_ref))
    assert np.max(np.abs(U.cpu().numpy() - U_ref)) <= 1e-12 * np.max(np.abs(U_ref))


@pytest.fixture(scope="module")
def cfg5_full():
    return scenes.cfg5()


def test_fullsize_cfg5_generate(orc, R, cfg5_full):
    sc = cfg5_full
    ctx = _ctx(R, sc)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(12 * sc["n"])
    n0, _ = ctx.generate_contacts(bodies, cs)
    pi, pj = (t.cpu().numpy() for t in ctx.get_pairs())
    assert 20e6 < len(pi) < 23e6 and 5.0e6 < n0 < 5.6e6
    key = pi.astype(np.int64) << 32 | pj
    assert np.all(pi < pj) and np.all(np.diff(key) > 0)
    # broadphase inside a 20^3 sub-box: exact against the oracle's O(N^2) scan
    inside = np.all(sc["pos"] < 20.0, axis=1)
    S = np.flatnonzero(inside)
    ri, rj = orc.broadphase(sc["pos"][S], sc["axes"][S].max(1), sc["box"], sc["cutoff"], "brute")
    ref = set(zip(S[ri].tolist(), S[rj].tolist()))
    mask = inside[pi] & inside[pj]
    got = set(zip(pi[mask].tolist(), pj[mask].tolist()))
    assert len(ref) > 1000 and got == ref
    # sampled SNSD: 3000 candidate pairs, oracle one by one from the generator's bodies
    rng = np.random.default_rng(0)
    k = rng.choice(len(pi), 3000, replace=False)
    phi_r, n_r, *_ = orc.snsd(sc["pos"], sc["quat"], sc["axes"], sc["box"], pi[k], pj[k])
    phi, nn, ra, rb, st = ctx.snsd_pairs(bodies, pi[k], pj[k])
    phi = phi.cpu().numpy()
    assert np.max(np.abs(phi - phi_r)) <= 1e-12 * 4
    ok = np.abs(phi_r) > 1e-9
    assert np.max(np.abs(nn.cpu().numpy().T[ok] - n_r[ok])) <= 1e-10
    # the store holds exactly the candidates with Phi < cutoff: check the sample
    c = cs.to_numpy()
    rows = set(zip(c["ia"].tolist(), c["ib"].tolist()))
    for a, b2, f in zip(pi[k], pj[k], phi_r):
        if abs(f - sc["cutoff"]) > 1e-10:
            assert ((int(a), int(b2)) in rows) == (f < sc["cutoff"])


def test_fullsize_cfg5_step_invariants(orc, R, cfg5_full):
    """The bench workload (2 recursions, 3000-iteration LCP cap)."""
    sc = cfg5_full
    ctx = _ctx(R, sc, lcp_tol=1e-8, lcp_max_iter=3000, max_recursions=2)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(12 * sc["n"])
    ctx.generate_contacts(bodies, cs)
    q0 = cs.q[:cs.count].clone()
    key0 = (cs.ia[:cs.count].long() << 32) | cs.ib[:cs.count].long()
    rep = ctx.step(bodies, cs)
    assert rep["n_c"][0] == len(q0) and rep["recursions"] == 2
    m = cs.count
    ia, ib, gen = cs.ia[:m].long(), cs.ib[:m].long(), cs.gen[:m].long()
    key = (ia << 32) | ib
    # sorted by (ia, ib, gen) (R18)
    assert bool(torch.all(key[1:] >= key[:-1]))
    same = key[1:] == key[:-1]
    assert bool(torch.all(gen[1:][same] > gen[:-1][same]))
    # q retention: generation-0 rows keep q_0
    g0 = gen == 0
    assert torch.equal(key[g0], key0) and torch.equal(cs.q[:m][g0], q0)
    lam = cs.lam[:m]
    assert bool(torch.all(lam >= 0))
    # Newton's third law: total linear momentum unchanged (no external force)
    mass = torch.as_tensor(1.0 / sc["inv_mass"], device="cuda")
    v0 = torch.as_tensor(sc["vel"][:, :3], device="cuda")
    dP = ((bodies.vel[:, :3] - v0) * mass[:, None]).sum(0)
    scale = ((bodies.vel[:, :3] - v0).abs() * mass[:, None]).sum()
    assert float(dP.abs().max()) <= 1e-12 * float(scale)
    # the last LCP's g on the final (augmented) store is the oracle's
    # s D^T W D lambda + q with W frozen at C^k (the generator's orientations)
    c = cs.to_numpy()
    Alam = orc.delassus_apply(orc.body_W(sc), c["ia"], c["ib"], c["n"], c["ta"], c["tb"], sc["dt"] ** 2, c["lam"])
    assert len(c["ia"]) == rep["n_c"][-1]
    assert np.max(np.abs(c["g"] - (Alam + c["q"]))) <= 1e-12 * np.max(np.abs(Alam))


@pytest.mark.parametrize("layout", [0, 1])
def test_fullsize_cfg5_solve_against_oracle_operator(orc, R, cfg5_full, layout):
    """cfg5 A_0 (5.3M rows) solved in the bench's launch configuration (BB,
    3000-iteration cap, compact-row K7): the g the GPU returns equals the
    oracle's own s D^T W D lambda + q on EVERY row (1e-12 of the scale of
    A lambda), and the returned pair satisfies lambda >= 0 and the reported
    residual r = max |min(lambda, g)|."""
    sc = cfg5_full
    ctx = _ctx(R, sc, lcp_tol=1e-8, lcp_max_iter=3000, layout=layout)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(12 * sc["n"])
    ctx.generate_contacts(bodies, cs)
    rep = ctx.solve_lcp(bodies, cs)
    assert ctx.stats()["jds_solves"] == layout
    c = cs.to_numpy()
    lam, g, q = c["lam"], c["g"], c["q"]
    assert np.all(lam >= 0)
    # Alg. 1 "solve" to the stopping tolerance (R2, north_star r < 1e-8)
    assert rep["converged"] and rep["residual"] <= 1e-8
    assert abs(np.max(np.abs(np.minimum(lam, g))) - rep["residual"]) <= 1e-15 + 1e-12 * rep["residual"]
    W = orc.body_W(sc)
    Alam = orc.delassus_apply(W, c["ia"], c["ib"], c["n"], c["ta"], c["tb"], sc["dt"] ** 2, lam)
    assert np.max(np.abs(g - (Alam + q))) <= 1e-12 * np.max(np.abs(Alam))


def test_fullsize_cfg4_lcp(R):
    sc = scenes.cfg4()
    net = sc["network"]
    ctx = _ctx(R, sc, lcp_tol=1e-8, lcp_max_iter=20000)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(len(net["ia"]) + 16)
    ctx.load_constraints(bodies, cs, net["ia"], net["ib"], net["n"], net["ra"], net["rb"], net["phi"])
    rep = ctx.solve_lcp(bodies, cs)
    assert rep["converged"] and rep["residual"] <= 1e-8
    m = cs.count
    lam, g = cs.lam[:m], cs.g[:m]
    assert bool(torch.all(lam >= 0)) and float(torch.minimum(lam, g).abs().max()) <= 1e-8
    U = torch.empty(sc["n"], 6, dtype=torch.float64, device="cuda")
    ctx.prepare_operator(bodies, cs)
    ctx.wrench(bodies, cs, lam.contiguous(), None, U)
    kin = torch.as_tensor(sc["kinematic"], device="cuda") != 0
    assert int(kin.sum()) == 2000 and float(U[kin].abs().max()) == 0.0
    assert 0.4 < float((lam > 0).double().mean()) < 0.9


def test_fullsize_cfg4_6M_lcp(orc, R):
    """cfg4-6M (c = 3 rows per link, 5.994M rows, the
    BASELINE "~6M"): N_C > 6 N_free, so lambda is not unique (Lemma 5,
    P:L333-373, R13); solved to r <= 1e-8 with lambda >= 0, and the returned g
    equals the oracle's own s D^T W D lambda + q on every row (1e-12 of the
    scale of A lambda)."""
    sc = scenes.cfg4(c_fixed=3)
    net = sc["network"]
    assert len(net["ia"]) == 5_994_000
    ctx = _ctx(R, sc, lcp_tol=1e-8, lcp_max_iter=50000)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(len(net["ia"]) + 16)
    ctx.load_constraints(bodies, cs, net["ia"], net["ib"], net["n"], net["ra"], net["rb"], net["phi"])
    rep = ctx.solve_lcp(bodies, cs)
    assert rep["converged"] and rep["residual"] <= 1e-8
    c = cs.to_numpy()
    assert np.all(c["lam"] >= 0)
    W = orc.body_W(sc)
    Alam = orc.delassus_apply(W, c["ia"], c["ib"], c["n"], c["ta"], c["tb"], sc["dt"] ** 2, c["lam"])
    assert np.max(np.abs(c["g"] - (Alam + c["q"]))) <= 1e-12 * np.max(np.abs(Alam))
    assert np.max(np.abs(np.minimum(c["lam"], c["g"]))) <= 1e-8


def test_fullsize_cfg3_step_planar(R):
    sc = scenes.cfg3()
    ctx = _ctx(R, sc, lcp_tol=1e-8, lcp_max_iter=3000, max_recursions=3)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(12 * sc["n"])
    rep = ctx.step(bodies, cs)
    assert 2.5 < 2 * rep["n_c"][0] / sc["n"] < 4.5  # ~3 contacts per body (BASELINE cfg3)
    assert rep["residuals"][0] <= 1e-8
    m = cs.count
    # z-reflection symmetry: every A_0 row (discovered at the planar C^k) is in-plane.
    # (Jammed rows reach lambda ~ 1e3, so the overdamped rotation 12/(xi L^3)
    # tau dt of the first-order update can reach tens of radians; the deep
    # in-plane overlaps this creates at C_1 have out-of-plane SNSD maxima, so
    # later generations may leave the plane -- the oracle follows the same
    # equations; DESIGN.md §2 R21.)
    g0 = cs.gen[:m] == 0
    assert float(cs.n[2, :m][g0].abs().max()) < 1e-11
    assert float(cs.ta[0, :m][g0].abs().max()) < 1e-11 and float(cs.ta[1, :m][g0].abs().max()) < 1e-11
    assert bool(torch.all(cs.lam[:m] >= 0))
    # the regime R21 describes, recorded: the first-order overdamped update turns
    # jammed bodies by ~1 rad (measured 0.97 rad; dt |omega| is larger, the
    # normalised first-order quaternion update saturates) in one dt = 1e-2 step:
    # the recipe is stiff at this dt, which is why later generations may leave
    # the plane
    q0 = torch.as_tensor(sc["quat"], device="cuda")
    q1 = bodies.quat / bodies.quat.norm(dim=1, keepdim=True)
    q0 = q0 / q0.norm(dim=1, keepdim=True)
    ang = 2.0 * torch.acos(torch.clamp((q0 * q1).sum(1).abs(), max=1.0))
    print(f"cfg3 step: max rotation {float(ang.max()):.2f} rad, bodies turned > 1 rad: {int((ang > 1.0).sum())}")
    assert float(ang.max()) > 0.5


def test_fullsize_cfg5_A0_subbox_every_pair(orc, R, cfg5_full):
    """cfg5 A_0 at full size (2M bodies, 21M candidates, 5.3M rows): EVERY row
    whose two bodies lie in the sub-box [0, 45)^3 (~50k bodies, ~0.5M
    candidate pairs, ~130k rows) against the oracle, which runs its own
    broadphase (cells) and SNSD on the generator's bodies: the (ia, ib) list
    is bit-exact outside the R14 guard band, Phi within 1e-12 max(1, |d|),
    n within 1e-10, t_a / t_b within 1e-9 (SURVEY §8(c) tolerances; P:L225,
    P:L425-436).  The library's own guard-band count over all 21M
    pairs is reported (n_guard, R14)."""
    sc = cfg5_full
    ctx = _ctx(R, sc)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(12 * sc["n"])
    ctx.reset_stats()
    n0, _ = ctx.generate_contacts(bodies, cs)
    n_guard = ctx.stats()["n_guard"]
    c = cs.to_numpy()
    L = 45.0
    inside = np.all(sc["pos"] < L, axis=1)
    S = np.flatnonzero(inside)
    ri, rj = orc.broadphase(sc["pos"][S], sc["axes"][S].max(1), None, sc["cutoff"], "cells")
    pi, pj = S[ri], S[rj]
    phi_r, n_r, ra_r, rb_r, st_r = orc.snsd(sc["pos"], sc["quat"], sc["axes"], sc["box"], pi, pj)
    assert np.all(st_r == 0)
    cut = sc["cutoff"]
    guard = np.abs(phi_r - cut) < 1e-10
    keep = (phi_r < cut) & ~guard
    ref_key = (pi.astype(np.int64) << 32) | pj
    m = inside[c["ia"]] & inside[c["ib"]]
    got_key = (c["ia"][m].astype(np.int64) << 32) | c["ib"][m]
    assert np.all(np.diff(got_key) > 0)  # one row per pair, (ia, ib) order
    guard_keys = ref_key[guard]
    got_cmp = got_key[~np.isin(got_key, guard_keys)]
    print(f"cfg5 A0 sub-box: {len(S)} bodies, {len(pi)} candidates, {int(keep.sum())} rows, "
          f"guard-band pairs {int(guard.sum())} (sub-box, oracle) / {n_guard} (all pairs, GPU)")
    assert keep.sum() > 100_000
    assert np.array_equal(got_cmp, ref_key[keep])
    # values of the matched rows
    pos = np.searchsorted(ref_key, got_cmp)
    rows = np.flatnonzero(m)[~np.isin(got_key, guard_keys)]
    d = sc["pos"][c["ib"][rows]] - sc["pos"][c["ia"][rows]]
    d -= sc["box"] * np.rint(d / sc["box"])
    scale = np.maximum(1.0, np.linalg.norm(d, axis=1))
    assert np.max(np.abs(c["phi"][rows] - phi_r[pos]) / scale) <= 1e-12
    assert np.max(np.abs(c["n"][rows] - n_r[pos])) <= 1e-10
    ta_r, tb_r = orc.rows(n_r[pos], ra_r[pos], rb_r[pos])
    assert np.max(np.abs(c["ta"][rows] - ta_r)) <= 1e-9 and np.max(np.abs(c["tb"][rows] - tb_r)) <= 1e-9
    assert n_guard <= 10


def _subbox_min_phi(orc, sc, pos, quat, L=40.0):
    """min Phi over every candidate pair with both centres in [0, L)^3, by the
    oracle's own broadphase (cells) and SNSD."""
    p = np.mod(pos, sc["box"])
    S = np.flatnonzero(np.all(p < L, axis=1))
    ri, rj = orc.broadphase(p[S], sc["axes"][S].max(1), None, sc["cutoff"], "cells")
    phi, *_ = orc.snsd(p, quat, sc["axes"], sc["box"], S[ri], S[rj])
    return float(phi.min()), len(ri)


def test_fullsize_cfg5_relaxed_complete_step(orc, R, cfg5_full):
    """The bench headline: the literal cfg5 start
    relaxed by the library's LCP-SNSD steps; the oracle's SNSD scan of a
    sub-box confirms the relaxed state is overlap-free (Phi >= -eps_NCP; the
    theory's hypothesis).  One inertial step from it with
    fresh N(0,1) velocities is a COMPLETE Algorithm-1 step: every LCP solved
    to r <= 1e-8 (R2), the recursion stops by the rule (P:L645-648,
    status 0, max overlap <= eps_NCP) -- the oracle's scan of the accepted
    sub-box agrees -- and g = the oracle's s D^T W D lambda + q on every row
    of the final store."""
    from paper_2506_14097_b200 import drivers
    lit = cfg5_full
    pos, quat, reps = drivers.relax(lit, max_recursions=0, lcp_max_iter=20000, max_steps=60)
    assert reps[-1]["status"] == 0 and reps[-1]["max_overlap"] <= 0.5 * lit["eps_ncp"]
    pos, quat = pos.cpu().numpy(), quat.cpu().numpy()
    m0, npairs = _subbox_min_phi(orc, lit, pos, quat)
    assert npairs > 100_000 and m0 >= -lit["eps_ncp"], m0
    sc = scenes.with_state(lit, pos, quat, 55, "cfg5-relaxed")
    ctx = _ctx(R, sc, lcp_tol=1e-8, lcp_max_iter=200_000, max_recursions=50)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(12 * sc["n"])
    rep = ctx.step(bodies, cs)
    assert rep["rc"] == 0 and rep["status"] == 0, rep
    assert max(rep["residuals"]) <= 1e-8 and rep["max_overlap"] <= sc["eps_ncp"]
    m1, _ = _subbox_min_phi(orc, sc, bodies.pos.cpu().numpy(), bodies.quat.cpu().numpy())
    assert m1 >= -sc["eps_ncp"] - 1e-12, m1
    c = cs.to_numpy()
    assert np.all(c["lam"] >= 0)
    Alam = orc.delassus_apply(orc.body_W(sc), c["ia"], c["ib"], c["n"], c["ta"], c["tb"], sc["dt"] ** 2, c["lam"])
    assert np.max(np.abs(c["g"] - (Alam + c["q"]))) <= 1e-12 * np.max(np.abs(Alam))
    assert float(np.max(np.abs(np.minimum(c["lam"], c["g"])))) <= 1e-8


def test_fullsize_cfg5_relaxed_dd_step(orc, R, cfg5_full):
    """The headline step, domain-decomposed (relcp_dd_step, 4 virtual parts of
    500k bodies): the same complete Algorithm-1 step as the
    single-domain library -- same recursions, N_C per recursion and rows
    (ia, ib, gen bit-exact), every LCP to r <= 1e-8, status 0 -- with
    configurations equal to the solver tolerance's effect, and g = the
    oracle's s D^T W D lambda + q on every row."""
    from paper_2506_14097_b200 import drivers
    lit = cfg5_full
    pos, quat, _ = drivers.relax(lit, max_recursions=0, lcp_max_iter=20000, max_steps=60)
    sc = scenes.with_state(lit, pos.cpu().numpy(), quat.cpu().numpy(), 55, "cfg5-relaxed")
    kw = dict(lcp_tol=1e-8, lcp_max_iter=200_000, max_recursions=50)
    ctx = _ctx(R, sc, **kw)
    b1 = R.BodyState.from_scene(sc)
    c1 = R.ConstraintStore(12 * sc["n"])
    r1 = ctx.step(b1, c1)
    dd = R.DomainDecomposition(np.array([0, 500_000, 1_000_000, 1_500_000, 2_000_000], dtype=np.int64),
                               dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]), cutoff=sc["cutoff"],
                               eps_ncp=sc["eps_ncp"], **kw)
    b2 = R.BodyState.from_scene(sc)
    c2 = R.ConstraintStore(12 * sc["n"])
    r2 = dd.step(b2, c2)
    assert r2["rc"] == 0 and r2["status"] == 0 and max(r2["residuals"]) <= 1e-8, r2
    assert r2["recursions"] == r1["recursions"] and r2["n_c"] == r1["n_c"]
    assert r2["max_overlap"] <= sc["eps_ncp"]
    g1, g2 = c1.to_numpy(), c2.to_numpy()
    for k in ("ia", "ib", "gen"):
        assert np.array_equal(g1[k], g2[k]), k
    dpos = b2.pos.cpu().numpy() - b1.pos.cpu().numpy()
    dpos -= sc["box"] * np.rint(dpos / sc["box"])
    print(f"dd step: recursions {r2['recursions']}, iterations {r2['iterations']} vs {r1['iterations']}, "
          f"max |dpos| {np.max(np.abs(dpos)):.2e}")
    assert np.max(np.abs(dpos)) <= 1e-6
    Alam = orc.delassus_apply(orc.body_W(sc), g2["ia"], g2["ib"], g2["n"], g2["ta"], g2["tb"], sc["dt"] ** 2,
                              g2["lam"])
    assert np.max(np.abs(g2["g"] - (Alam + g2["q"]))) <= 1e-12 * np.max(np.abs(Alam))
    assert np.all(g2["lam"] >= 0) and float(np.max(np.abs(np.minimum(g2["lam"], g2["g"])))) <= 1e-8
    dd.close()


def _cfg4_fixture():
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg4_full_sample.txt")
    head = {}
    rows, bods = [], []
    for ln in open(path):
        if ln.startswith("# max_abs"):
            t = ln.split()
            head.update(lam=float(t[3]), g=float(t[5]), U=float(t[7]))
        elif ln.startswith("# rows_sha256"):
            head["sha"] = ln.split()[2]
        elif ln.startswith("# oracle.network_lcp"):
            head["tol"] = float(ln.split("tol ")[1].split(")")[0])
        elif ln.startswith("R "):
            rows.append(ln.split()[1:])
        elif ln.startswith("B "):
            bods.append(ln.split()[1:])
    r = np.array(rows, dtype=float)
    b = np.array(bods, dtype=float)
    return head, r[:, 0].astype(np.int64), r[:, 1], r[:, 2], b[:, 0].astype(np.int64), b[:, 1:]


def test_fullsize_cfg4_against_oracle_solution(R):
    """BASELINE cfg4 at full size (10^6 rings, ~4.0M rows): the GPU's solution
    against the ORACLE's own (tests/golden/cfg4_full_sample.txt, written by
    tools/make_cfg4_sample.py from oracle.network_lcp only) on 20,000 sampled
    rows (lambda, g) and 5,000 sampled bodies (U = W D lambda, unique by
    Lemma 5), each within 1e-6 of the oracle's max over ALL rows /
    bodies (north_star; R13), with the GPU residual r <= 1e-8 (Lemma 3,
    P:L280-299).  Both sides solve to the fixture's tolerance or tighter."""
    import hashlib
    head, ri, lam_r, g_r, bi, U_r = _cfg4_fixture()
    sc = scenes.cfg4()
    net = sc["network"]
    assert hashlib.sha256(net["ia"].astype(np.int32).tobytes() + net["ib"].astype(np.int32).tobytes()).hexdigest() \
        == head["sha"]
    ctx = _ctx(R, sc, lcp_tol=min(1e-10, head["tol"]), lcp_max_iter=200_000)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(len(net["ia"]) + 16)
    ctx.load_constraints(bodies, cs, net["ia"], net["ib"], net["n"], net["ra"], net["rb"], net["phi"])
    rep = ctx.solve_lcp(bodies, cs)
    assert rep["converged"] and rep["residual"] <= 1e-8
    lam = cs.lam[:cs.count].cpu().numpy()
    g = cs.g[:cs.count].cpu().numpy()
    # g is fixed only to the solvers' tolerance on active rows (|min(lambda, g)| <= tol on both sides, R2)
    assert np.max(np.abs(g[ri] - g_r)) <= 1e-6 * head["g"] + 2 * head["tol"]
    assert np.max(np.abs(lam[ri] - lam_r)) <= 1e-6 * head["lam"]
    U = torch.empty(sc["n"], 6, dtype=torch.float64, device="cuda")
    ctx.prepare_operator(bodies, cs)
    ctx.wrench(bodies, cs, cs.lam[:cs.count].contiguous(), None, U)
    assert np.max(np.abs(U.cpu().numpy()[bi] - U_r)) <= 1e-6 * head["U"]
