"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on
the same seeded inputs (gen/scenes.py).  Tolerances (BASELINE north_star,
SURVEY §8(c)):
  * constraint pair lists / indices: bit-exact (outside the guard band R14);
  * Delassus apply: ||y - y_ref||_inf <= 1e-12 ||y_ref||_inf;
  * SNSD: Phi 1e-12 max(1, |d|) abs, n 1e-10;
  * LCP: lambda 1e-6 relative (where unique, R13), D lambda and g 1e-6
    relative, GPU residual < tol;
  * trial / accepted configurations 1e-9 abs.
"""
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


def _net(orc, nb, nc, seed, dynamics):
    b, ia, ib, n, ra, rb = scenes.random_constraint_network(nb, nc, seed, dynamics)
    ta, tb = np.cross(ra, n), np.cross(rb, n)
    return b, ia, ib, n, ta, tb


# ------------------------------------------------------------ Delassus apply

@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("dynamics", [0, 1])
@pytest.mark.parametrize("nb,nc", [(7, 1), (97, 1000), (2000, 9973), (5000, 40001)])
def test_delassus_apply_parity(orc, R, dynamics, nb, nc, layout):
    """layout 0 (CSR) and 1 (JDS)."""
    b, ia, ib, n, ta, tb = _net(orc, nb, nc, 11 + nb, dynamics)
    b["dynamics"] = dynamics
    W = orc.body_W(b)
    rng = np.random.default_rng(nb)
    x = rng.standard_normal(nc)
    s = 0.37
    y_ref = orc.delassus_apply(W, ia, ib, n, ta, tb, s, x)
    ctx = _ctx(R, dict(dynamics=dynamics, dt=1e-3, cutoff=0.1, eps_ncp=1e-5, box=[0, 0, 0]), layout=layout)
    bodies = R.BodyState.from_scene(b)
    cs = R.ConstraintStore.from_rows(ia, ib, n, ta, tb, capacity=nc + 13)
    ctx.prepare_operator(bodies, cs)
    assert ctx.stats()["op_layout"] == layout
    xd = torch.as_tensor(x, device="cuda")
    yd = torch.empty_like(xd)
    ctx.delassus_apply(bodies, cs, xd, yd, s)
    y = yd.cpu().numpy()
    assert np.max(np.abs(y - y_ref)) <= 1e-12 * np.max(np.abs(y_ref))
    # determinism: bitwise identical on repeat
    yd2 = torch.empty_like(xd)
    ctx.delassus_apply(bodies, cs, xd, yd2, s)
    assert torch.equal(yd, yd2)
    # wrench F = D x and U = W D x
    F_ref, U_ref = orc.wrench(W, ia, ib, n, ta, tb, x)
    F = torch.empty(nb, 6, dtype=torch.float64, device="cuda")
    U = torch.empty_like(F)
    ctx.wrench(bodies, cs, xd, F, U)
    assert np.max(np.abs(F.cpu().numpy() - F_ref)) <= 1e-12 * np.max(np.abs(F_ref))
    assert np.max(np.abs(U.cpu().numpy() - U_ref)) <= 1e-12 * np.max(np.abs(U_ref))


@pytest.mark.parametrize("shuffled", [False, True])
@pytest.mark.parametrize("dynamics", [0, 1])
def test_delassus_apply_hubs_and_empty_bodies(orc, R, shuffled, dynamics):
    """K6 tile logic: a hub body whose segment spans many 64-entry tiles (700
    rows), a body with 130 rows to one partner, runs of bodies without rows,
    a ragged body count; sorted (a-side in place) and unsorted (general CSR)."""
    rng = np.random.default_rng(42)
    nb = 1000 + 37
    ia = [np.zeros(700, int)]
    ib = [rng.integers(1, nb, size=700)]
    ia.append(np.full(130, 500)); ib.append(np.full(130, 900))
    live = rng.choice(np.arange(1, nb), size=300, replace=False)  # other bodies: sparse
    a = rng.choice(live, size=400); b = rng.choice(live, size=400)
    keep = a != b
    ia.append(a[keep]); ib.append(b[keep])
    ia, ib = np.concatenate(ia), np.concatenate(ib)
    lo, hi = np.minimum(ia, ib), np.maximum(ia, ib)
    o = np.lexsort((hi, lo))
    ia, ib = lo[o].astype(np.int32), hi[o].astype(np.int32)
    nc = len(ia)
    n = rng.normal(size=(nc, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    ta, tb = rng.uniform(-1, 1, size=(nc, 3)), rng.uniform(-1, 1, size=(nc, 3))
    if shuffled:
        p = rng.permutation(nc)
        ia, ib, n, ta, tb = ia[p], ib[p], n[p], ta[p], tb[p]
    b_ = scenes.suspension(nb, (1.0, 0.6, 0.4), 0.3, 5, dynamics=dynamics)
    W = orc.body_W(b_)
    x = rng.standard_normal(nc)
    y_ref = orc.delassus_apply(W, ia, ib, n, ta, tb, 1.0, x)
    F_ref, U_ref = orc.wrench(W, ia, ib, n, ta, tb, x)
    ctx = _ctx(R, dict(dynamics=dynamics, dt=1e-3, cutoff=0.1, eps_ncp=1e-5, box=[0, 0, 0]))
    bodies = R.BodyState.from_scene(b_)
    cs = R.ConstraintStore.from_rows(ia, ib, n, ta, tb)
    ctx.prepare_operator(bodies, cs)
    xd = torch.as_tensor(x, device="cuda")
    yd = torch.empty_like(xd)
    ctx.delassus_apply(bodies, cs, xd, yd, 1.0)
    assert np.max(np.abs(yd.cpu().numpy() - y_ref)) <= 1e-12 * np.max(np.abs(y_ref))
    F = torch.empty(nb, 6, dtype=torch.float64, device="cuda")
    U = torch.empty_like(F)
    ctx.wrench(bodies, cs, xd, F, U)
    assert np.max(np.abs(F.cpu().numpy() - F_ref)) <= 1e-12 * np.max(np.abs(F_ref))
    assert np.max(np.abs(U.cpu().numpy() - U_ref)) <= 1e-12 * np.max(np.abs(U_ref))
    assert np.all(U.cpu().numpy()[np.setdiff1d(np.arange(nb), np.concatenate([ia, ib]))] == 0)


@pytest.mark.parametrize("dynamics", [0, 1])
def test_jds_apply_hubs_and_empty_bodies(orc, R, dynamics):
    """JDS layout: a hub with 700 a-side rows, a hub with 300 b-side
    entries, a pair with 130 parallel rows, runs of bodies without rows, a
    ragged last warp; rows t = r x n (the layout needs the compact rows)."""
    rng = np.random.default_rng(43)
    nb = 1000 + 37
    ia = [np.zeros(700, int), rng.integers(0, 900, size=300)]
    ib = [rng.integers(1, nb, size=700), np.full(300, 950)]
    ia.append(np.full(130, 500)); ib.append(np.full(130, 900))
    live = rng.choice(np.arange(1, nb), size=300, replace=False)
    a = rng.choice(live, size=400); b = rng.choice(live, size=400)
    keep = a != b
    ia.append(a[keep]); ib.append(b[keep])
    ia, ib = np.concatenate(ia), np.concatenate(ib)
    keep = ia != ib
    ia, ib = ia[keep], ib[keep]
    lo, hi = np.minimum(ia, ib), np.maximum(ia, ib)
    o = np.lexsort((hi, lo))
    ia, ib = lo[o].astype(np.int32), hi[o].astype(np.int32)
    nc = len(ia)
    n = rng.normal(size=(nc, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    ta = np.cross(rng.uniform(-1, 1, size=(nc, 3)), n)
    tb = np.cross(rng.uniform(-1, 1, size=(nc, 3)), n)
    b_ = scenes.suspension(nb, (1.0, 0.6, 0.4), 0.3, 5, dynamics=dynamics)
    W = orc.body_W(b_)
    x = rng.standard_normal(nc)
    y_ref = orc.delassus_apply(W, ia, ib, n, ta, tb, 1.0, x)
    F_ref, U_ref = orc.wrench(W, ia, ib, n, ta, tb, x)
    ctx = _ctx(R, dict(dynamics=dynamics, dt=1e-3, cutoff=0.1, eps_ncp=1e-5, box=[0, 0, 0]), layout=1)
    bodies = R.BodyState.from_scene(b_)
    cs = R.ConstraintStore.from_rows(ia, ib, n, ta, tb)
    ctx.prepare_operator(bodies, cs)
    assert ctx.stats()["op_layout"] == 1
    xd = torch.as_tensor(x, device="cuda")
    yd = torch.empty_like(xd)
    ctx.delassus_apply(bodies, cs, xd, yd, 1.0)
    assert np.max(np.abs(yd.cpu().numpy() - y_ref)) <= 1e-12 * np.max(np.abs(y_ref))
    F = torch.empty(nb, 6, dtype=torch.float64, device="cuda")
    U = torch.empty_like(F)
    ctx.wrench(bodies, cs, xd, F, U)
    assert np.max(np.abs(F.cpu().numpy() - F_ref)) <= 1e-12 * np.max(np.abs(F_ref))
    assert np.max(np.abs(U.cpu().numpy() - U_ref)) <= 1e-12 * np.max(np.abs(U_ref))
    assert np.all(U.cpu().numpy()[np.setdiff1d(np.arange(nb), np.concatenate([ia, ib]))] == 0)
    # the same solve on both layouts (q > 0 on the 130 parallel rows: they stay
    # inactive, so the LCP keeps a well-conditioned active set)
    qh = rng.standard_normal(nc) * 1e-3
    qh[(ia == 500) & (ib == 900)] = 1e-3
    q = torch.as_tensor(qh, device="cuda")
    out = []
    for lay in (0, 1):
        c2 = _ctx(R, dict(dynamics=dynamics, dt=1e-3, cutoff=0.1, eps_ncp=1e-5, box=[0, 0, 0]), layout=lay,
                  lcp_tol=1e-10, lcp_max_iter=2_000_000)
        s2 = R.ConstraintStore.from_rows(ia, ib, n, ta, tb)
        s2.q[:nc] = q
        rep = c2.solve_lcp(bodies, s2)
        assert rep["converged"] and c2.stats()["jds_solves"] == lay
        out.append((s2.lam[:nc].cpu().numpy(), s2.g[:nc].cpu().numpy()))
    assert np.max(np.abs(out[0][1] - out[1][1])) <= 1e-6 * np.max(np.abs(out[0][1])) + 1e-9


def test_delassus_empty_and_state(orc, R):
    b, ia, ib, n, ta, tb = _net(orc, 10, 5, 3, 0)
    ctx = _ctx(R, dict(dynamics=0, dt=1e-3, cutoff=0.1, eps_ncp=1e-5, box=[0, 0, 0]))
    bodies = R.BodyState.from_scene(b)
    cs = R.ConstraintStore.from_rows(ia, ib, n, ta, tb)
    x = torch.ones(5, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    with pytest.raises(R.RelcpError) as e:  # operator not prepared
        ctx.delassus_apply(bodies, cs, x, y)
    assert e.value.code == R.E_STATE
    empty = R.ConstraintStore(4)
    ctx.prepare_operator(bodies, empty)
    ctx.delassus_apply(bodies, empty, x, y)  # no-op
    bad = R.ConstraintStore.from_rows([3], [3], n[:1], ta[:1], tb[:1])
    with pytest.raises(R.RelcpError):
        ctx.prepare_operator(bodies, bad)


# ------------------------------------------------------------ LCP

@pytest.fixture(scope="module")
def cfg1_a0(orc):
    sc = scenes.cfg1()
    r = orc.relcp_step(sc, snsd_only=True, lcp_tol=1e-10)
    return sc, r


@pytest.mark.parametrize("cluster", [0, 1])
@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("solver", [0, 1, 2])
def test_lcp_solve_parity_cfg1(orc, R, cfg1_a0, solver, layout, cluster):
    """Every solver, both operator layouts, and for BB on the CSR layout the
    single-cluster loop (cluster = 1, the default at this size) and the
    per-pass kernels (cluster = 0)."""
    sc, r = cfg1_a0
    c = r["constraints"]
    ctx = _ctx(R, sc, lcp_tol=1e-10, solver=solver, lcp_max_iter=2_000_000, layout=layout, cluster=cluster)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore.from_rows(c["ia"], c["ib"], c["n"], c["ta"], c["tb"], q=r["q_hist"][0])
    rep = ctx.solve_lcp(bodies, cs)
    assert rep["converged"] and rep["residual"] <= 1e-10
    # JDS unless the fused APGD solver (CSR only); the cluster loop for BB on CSR
    assert ctx.stats()["jds_solves"] == (1 if layout == 1 and solver != 2 else 0)
    assert ctx.stats()["cluster_solves"] == (1 if cluster and solver == 0 and layout == 0 else 0)
    lam = cs.lam[:cs.count].cpu().numpy()
    g = cs.g[:cs.count].cpu().numpy()
    lam_ref, g_ref = c["lam"], r["g_hist"][0]
    assert np.all(lam >= 0)
    assert np.max(np.abs(lam - lam_ref)) <= 1e-6 * np.max(np.abs(lam_ref))
    assert np.max(np.abs(g - g_ref)) <= 1e-6 * max(1e-300, np.max(np.abs(g_ref))) + 1e-9
    # D lambda (unique by Lemma 5)
    W = r["W"]
    F_ref, _ = orc.wrench(W, c["ia"], c["ib"], c["n"], c["ta"], c["tb"], lam_ref)
    F = torch.empty(sc["n"], 6, dtype=torch.float64, device="cuda")
    ctx.prepare_operator(bodies, cs)
    ctx.wrench(bodies, cs, cs.lam[:cs.count].contiguous(), F, None)
    assert np.max(np.abs(F.cpu().numpy() - F_ref)) <= 1e-6 * np.max(np.abs(F_ref))
    # objective f = -1/2 lambda^T A lambda
    assert abs(rep["objective"] - r["f"][0]) <= 1e-6 * abs(r["f"][0])


@pytest.mark.parametrize("solver", [0, 1, 2])
def test_lcp_solve_parity_shuffled_store(orc, R, cfg1_a0, solver):
    """A caller's store in arbitrary row order (general CSR path: both sides
    in the CSR, K6 SORTED = false; the fused solver falls back to APGD): same
    solution as the oracle, row for row."""
    sc, r = cfg1_a0
    c = r["constraints"]
    perm = np.random.default_rng(17).permutation(len(c["ia"]))
    ctx = _ctx(R, sc, lcp_tol=1e-10, solver=solver, lcp_max_iter=2_000_000)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore.from_rows(c["ia"][perm], c["ib"][perm], c["n"][perm], c["ta"][perm], c["tb"][perm],
                                     q=r["q_hist"][0][perm])
    rep = ctx.solve_lcp(bodies, cs)
    assert rep["converged"] and rep["residual"] <= 1e-10
    lam = cs.lam[:cs.count].cpu().numpy()
    lam_ref = c["lam"][perm]
    assert np.max(np.abs(lam - lam_ref)) <= 1e-6 * np.max(np.abs(lam_ref))
    assert abs(rep["objective"] - r["f"][0]) <= 1e-6 * abs(r["f"][0])


@pytest.mark.parametrize("solver", [0, 1, 2])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_lcp_vs_enumeration_tiny(orc, R, seed, solver):
    """Tiny random LCPs: the GPU solution equals the brute-force support
    enumeration."""
    b, ia, ib, n, ta, tb = _net(orc, 6, 9, 100 + seed, 0)
    b["dynamics"] = 0
    W = orc.body_W(b)
    nc = len(ia)
    A = np.stack([orc.delassus_apply(W, ia, ib, n, ta, tb, 1.0, e) for e in np.eye(nc)], 1)
    q = np.random.default_rng(seed).standard_normal(nc)
    x_ref = orc.enumerate_lcp(A, q)
    ctx = _ctx(R, dict(dynamics=0, dt=1.0, cutoff=0.1, eps_ncp=1e-5, box=[0, 0, 0]), lcp_tol=1e-12,
               solver=solver, lcp_max_iter=2_000_000)
    bodies = R.BodyState.from_scene(b)
    cs = R.ConstraintStore.from_rows(ia, ib, n, ta, tb, q=q)
    rep = ctx.solve_lcp(bodies, cs)
    assert rep["converged"]
    x = cs.lam[:nc].cpu().numpy()
    # compare the unique image A x (Lemma 5) and x itself when A is nonsingular
    assert np.max(np.abs(A @ x - A @ x_ref)) <= 1e-9 * (1 + np.max(np.abs(q)))
    if np.linalg.matrix_rank(A) == nc:
        assert np.max(np.abs(x - x_ref)) <= 1e-6 * max(1.0, np.max(np.abs(x_ref)))


def test_lcp_warm_start_and_zero(orc, R):
    """q >= 0 -> lambda = 0; warm start from the solution converges at once."""
    b, ia, ib, n, ta, tb = _net(orc, 50, 120, 5, 0)
    ctx = _ctx(R, dict(dynamics=0, dt=1.0, cutoff=0.1, eps_ncp=1e-5, box=[0, 0, 0]), lcp_tol=1e-12)
    bodies = R.BodyState.from_scene(b)
    cs = R.ConstraintStore.from_rows(ia, ib, n, ta, tb, q=np.abs(np.random.default_rng(1).standard_normal(120)))
    rep = ctx.solve_lcp(bodies, cs)
    assert rep["converged"] and rep["iterations"] == 0
    assert torch.count_nonzero(cs.lam[:120]).item() == 0
    cs.q[:120] = torch.as_tensor(np.random.default_rng(2).standard_normal(120), device="cuda")
    rep = ctx.solve_lcp(bodies, cs)
    assert rep["converged"]
    rep2 = ctx.solve_lcp(bodies, cs)
    assert rep2["converged"] and rep2["iterations"] <= 1


# ------------------------------------------------------------ SNSD + broadphase

def test_snsd_parity_cfg1_pairs(orc, R, cfg1_a0):
    sc, r = cfg1_a0
    pi, pj = r["pairs"]
    phi_r, n_r, ra_r, rb_r, st_r = orc.snsd(sc["pos"], sc["quat"], sc["axes"], sc["box"], pi, pj)
    ctx = _ctx(R, sc)
    bodies = R.BodyState.from_scene(sc)
    phi, n, ra, rb, st = ctx.snsd_pairs(bodies, pi, pj)
    phi, n, ra, rb, st = (t.cpu().numpy() for t in (phi, n, ra, rb, st))
    assert np.all(st == 0) and np.all(st_r == 0)
    d = sc["pos"][pj] - sc["pos"][pi]
    d -= sc["box"] * np.rint(d / sc["box"])
    dn = np.linalg.norm(d, axis=1)
    assert np.all(np.abs(phi - phi_r) <= 1e-12 * np.maximum(1, dn))
    assert np.max(np.abs(n.T - n_r)) <= 1e-10
    assert np.max(np.abs(ra.T - ra_r)) <= 1e-9 and np.max(np.abs(rb.T - rb_r)) <= 1e-9


def test_snsd_random_overlaps(orc, R):
    """Deep overlaps of elongated pairs (cfg2 shapes), the multistart branch."""
    rng = np.random.default_rng(7)
    m = 3000
    pos = np.zeros((2 * m, 3))
    pos[1::2] = rng.uniform(-1.2, 1.2, size=(m, 3))
    quat = rng.standard_normal((2 * m, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    r = rng.uniform(1, 4, size=2 * m)
    axes = np.stack([np.ones(2 * m), 1 / r, 1 / r], 1)
    pi = np.arange(0, 2 * m, 2, dtype=np.int32)
    pj = pi + 1
    phi_r, n_r, *_ = orc.snsd(pos, quat, axes, None, pi, pj)
    ctx = R.Context(dynamics=1, dt=1e-2)
    bodies = R.BodyState(pos, quat, axes)
    phi, n, ra, rb, st = ctx.snsd_pairs(bodies, pi, pj)
    phi = phi.cpu().numpy()
    dn = np.linalg.norm(pos[pj] - pos[pi], axis=1)
    err = np.abs(phi - phi_r) / np.maximum(1, dn)
    assert np.sum(phi_r < 0) > 500
    assert np.max(err) <= 1e-12, (np.argmax(err), phi[np.argmax(err)], phi_r[np.argmax(err)])


def _quat_R(q):
    s, x, y, z = (q / np.linalg.norm(q, axis=1, keepdims=True)).T
    return np.stack([np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - s * z), 2 * (x * z + s * y)], -1),
                     np.stack([2 * (x * y + s * z), 1 - 2 * (x * x + z * z), 2 * (y * z - s * x)], -1),
                     np.stack([2 * (x * z - s * y), 2 * (y * z + s * x), 1 - 2 * (x * x + y * y)], -1)], 1)


def test_snsd_curvature_certificate(orc, R):
    """Shallow and medium overlaps (cfg5 and cfg2 shapes): with the curvature
    certificate (R29) a certified Newton maximum at depth < rho / 2 (rho = the
    sum of the two smallest radii of curvature, min(e)^2 / max(e) each) is
    taken without the multistart.  Both settings equal the oracle's multistart
    global maximum (Phi 1e-12 max(1, |d|), n 1e-10), the certificate removes
    multistart work, and pairs deeper than rho / 2 still take the multistart."""
    rng = np.random.default_rng(29)
    m = 4000
    quat = rng.standard_normal((2 * m, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    r = rng.uniform(1, 4, size=2 * m)
    axes = np.where((np.arange(2 * m) // 2 % 2 == 0)[:, None], np.array([1.0, 0.6, 0.4]),
                    np.stack([np.ones(2 * m), 1 / r, 1 / r], 1))
    u = rng.standard_normal((m, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    Rm = _quat_R(quat)
    Sig = np.einsum("bij,bj,bkj->bik", Rm, axes ** 2, Rm)
    h = lambda S: np.sqrt(np.einsum("bi,bij,bj->b", u, S, u))
    hs = h(Sig[0::2]) + h(Sig[1::2])
    # |d| = (1 - delta)(h_a + h_b) along u: F(u) = -delta (h_a + h_b) <= Phi <= 0
    delta = rng.uniform(0.0, 0.2, size=m)
    pos = np.zeros((2 * m, 3))
    pos[1::2] = u * ((1 - delta) * hs)[:, None]
    pi = np.arange(0, 2 * m, 2, dtype=np.int32)
    pj = pi + 1
    phi_r, n_r, *_ = orc.snsd(pos, quat, axes, None, pi, pj)
    rmin = lambda e: e.min(1) ** 2 / e.max(1)
    rho = rmin(axes[0::2]) + rmin(axes[1::2])
    shallow = (phi_r <= 0) & (-phi_r < 0.45 * rho)
    assert shallow.sum() > 1000 and (-phi_r > 0.55 * rho).sum() > 100
    dn = np.linalg.norm(pos[pj] - pos[pi], axis=1)
    multi = []
    for cert in (0, 1):
        ctx = R.Context(dynamics=1, dt=1e-2, snsd_cert=cert)
        bodies = R.BodyState(pos, quat, axes)
        ctx.reset_stats()
        phi, n, ra, rb, st = ctx.snsd_pairs(bodies, pi, pj)
        multi.append(ctx.stats()["snsd_multistart"])
        phi, n = phi.cpu().numpy(), n.cpu().numpy().T
        err = np.abs(phi - phi_r) / np.maximum(1, dn)
        assert np.max(err) <= 1e-12, (cert, np.argmax(err), phi[np.argmax(err)], phi_r[np.argmax(err)])
        assert np.max(np.abs(n - n_r)) <= 1e-10
    # a shallow pair whose ascent from d/|d| ends at another local maximum (value
    # <= -rho, never the global one) still takes the multistart: allow 10 %
    assert multi[0] >= (phi_r <= 0).sum() and multi[1] <= multi[0] - 0.9 * shallow.sum() and multi[1] > 0


@pytest.mark.parametrize("n,phi_v", [(512, 0.3), (4000, 0.55), (20000, 0.55)])
def test_broadphase_parity(orc, R, n, phi_v):
    sc = scenes.suspension(n, (1.0, 0.6, 0.4), phi_v, 3)
    ctx = _ctx(R, sc)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(20 * n)
    ctx.generate_contacts(bodies, cs)
    pi, pj = ctx.get_pairs()
    ri, rj = orc.broadphase(sc["pos"], sc["axes"].max(1), sc["box"], sc["cutoff"])
    assert np.array_equal(pi.cpu().numpy(), ri) and np.array_equal(pj.cpu().numpy(), rj)


def test_broadphase_open_planar(orc, R):
    """Non-periodic planar layout (cfg3-like disk in z = 0)."""
    rng = np.random.default_rng(3)
    n = 3000
    ang = rng.uniform(0, 2 * np.pi, n)
    rr = 30 * np.sqrt(rng.uniform(0, 1, n))
    pos = np.stack([rr * np.cos(ang), rr * np.sin(ang), np.zeros(n)], 1)
    axes = np.stack([rng.uniform(0.5, 1.0, n), np.full(n, 0.25), np.full(n, 0.25)], 1)
    quat = np.zeros((n, 4))
    th = rng.uniform(0, np.pi, n)
    quat[:, 0], quat[:, 3] = np.cos(th / 2), np.sin(th / 2)
    ctx = R.Context(dynamics=1, dt=1e-2)
    bodies = R.BodyState(pos, quat, axes)
    cs = R.ConstraintStore(20 * n)
    ctx.generate_contacts(bodies, cs)
    pi, pj = ctx.get_pairs()
    ri, rj = orc.broadphase(pos, axes.max(1), None, 0.1, "brute")
    assert np.array_equal(pi.cpu().numpy(), ri) and np.array_equal(pj.cpu().numpy(), rj)


def test_generate_contacts_parity_cfg1(orc, R, cfg1_a0):
    sc, r = cfg1_a0
    c = r["constraints"]
    ctx = _ctx(R, sc)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(4 * len(c["ia"]))
    n0, rc = ctx.generate_contacts(bodies, cs)
    g = cs.to_numpy()
    assert n0 == len(c["ia"])
    assert np.array_equal(g["ia"], c["ia"]) and np.array_equal(g["ib"], c["ib"])
    assert np.all(g["gen"] == 0)
    # Phi within 1e-12 max(1, |d|) per pair, n within 1e-10
    d = sc["pos"][g["ib"]] - sc["pos"][g["ia"]]
    d -= sc["box"] * np.rint(d / sc["box"])
    assert np.all(np.abs(g["phi"] - c["phi"]) <= 1e-12 * np.maximum(1.0, np.linalg.norm(d, axis=1)))
    assert np.max(np.abs(g["n"] - c["n"])) <= 1e-10
    assert np.max(np.abs(g["ta"] - c["ta"])) <= 1e-9 and np.max(np.abs(g["tb"] - c["tb"])) <= 1e-9
    assert np.max(np.abs(g["q"] - r["q_hist"][0])) <= 1e-11
    # capacity error reports the required size and writes nothing
    small = R.ConstraintStore(3)
    with pytest.raises(R.RelcpError) as e:
        ctx.generate_contacts(bodies, small)
    assert e.value.code == R.E_CAPACITY and small.count == n0


# ------------------------------------------------------------ full step

def _sorted_rows(ia, ib, gen):
    return np.lexsort((ib, ia, gen))


def _compare_step(orc, R, sc, tol_cfg=1e-9, max_recursions=50, solver=0, reorder=1, layout=0, cluster=1):
    # Both sides solve every LCP to r <= 1e-12: two independent solvers that
    # each stop at r <= 1e-10 leave rotations differing by ~1e-9 (measured
    # 1.4e-9 on cfg1), at the edge of the 1e-9 configuration tolerance.
    r = orc.relcp_step(sc, lcp_tol=1e-12, max_recursions=max_recursions)
    ctx = _ctx(R, sc, lcp_tol=1e-12, max_recursions=max_recursions, lcp_max_iter=2_000_000, solver=solver,
               reorder=reorder, layout=layout, cluster=cluster)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(8 * max(1, len(r["constraints"]["ia"])) + 64)
    rep = ctx.step(bodies, cs)
    assert rep["recursions"] == r["recursions"]
    assert (rep["status"] != 0) == (r["status"] != 0)
    assert rep["n_c"] == r["n_c"]
    g = cs.to_numpy()
    c = r["constraints"]
    og, oo = _sorted_rows(g["ia"], g["ib"], g["gen"]), _sorted_rows(c["ia"], c["ib"], c["gen"])
    assert np.array_equal(g["ia"][og], c["ia"][oo]) and np.array_equal(g["ib"][og], c["ib"][oo])
    assert np.array_equal(g["gen"][og], c["gen"][oo])
    # rows found at C^k (gen 0) have identical inputs: n within 1e-10 (SURVEY
    # §8(c)); appended rows are evaluated at trial configurations that agree
    # only to the configuration tolerance (R19, ~1e-9), so n to 1e-8 there
    g0 = g["gen"][og] == 0
    assert np.max(np.abs(g["n"][og][g0] - c["n"][oo][g0]), initial=0.0) <= 1e-10
    assert np.max(np.abs(g["n"][og] - c["n"][oo])) <= 1e-8
    pos = bodies.pos.cpu().numpy()
    dpos = pos - r["pos"]
    if np.all(sc["box"] > 0):
        dpos -= sc["box"] * np.rint(dpos / sc["box"])
    assert np.max(np.abs(dpos)) <= tol_cfg
    assert np.max(np.abs(bodies.quat.cpu().numpy() - r["quat"])) <= tol_cfg
    if bodies.vel is not None:
        v_ref = r["vel"]
        assert np.max(np.abs(bodies.vel.cpu().numpy() - v_ref)) <= 1e-6 * max(1.0, np.max(np.abs(v_ref)))
    assert rep["max_overlap"] <= sc["eps_ncp"] or rep["status"] != 0
    # f_n non-increasing (Thm 1 proof)
    f = np.array(rep["f"])
    assert np.all(np.diff(f) <= 1e-6 * np.max(np.abs(f)) + 1e-12)
    return r, rep, g


@pytest.mark.parametrize("layout", [0, 1])
def test_step_parity_cfg1(orc, R, layout):
    _compare_step(orc, R, scenes.cfg1(), layout=layout)


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("solver", [1, 2])
def test_step_parity_cfg1_apgd(orc, R, solver, layout):
    """The whole step with APGD / fused APGD against the oracle's BB step
    (solution parity: every LCP solved to r <= 1e-12 on both sides)."""
    _compare_step(orc, R, scenes.cfg1(), solver=solver, layout=layout)


@pytest.mark.parametrize("reorder", [0, 2])
def test_step_parity_relabelled_cfg5_recipe(orc, R, reorder):
    """Body-order independence: the cfg5 recipe at 1000 bodies
    under a random relabelling, with the internal cell order off and forced
    on.  The oracle steps the relabelled scene as given; the GPU store comes
    back in the caller's labels, sorted, rows oriented ia < ib (R18)."""
    sc = scenes.relabelled(scenes.suspension(1000, (1.0, 0.6, 0.4), 0.55, 5, dt=1e-3), 17)
    r, rep, g = _compare_step(orc, R, sc, max_recursions=2, reorder=reorder)
    assert np.all(g["ia"] < g["ib"])
    key = g["ia"].astype(np.int64) * (1 << 40) + g["ib"].astype(np.int64) * 64 + g["gen"]
    assert np.all(np.diff(key) > 0)


def test_reorder_same_step(R):
    """The internal order relabels, nothing else: the step of a relabelled
    cfg5-recipe scene (3000 bodies) with reorder off and forced on gives the
    same rows (ids, generations bit-exact; Phi, n, q to rounding), lambda to the
    solver tolerance and the same accepted state."""
    sc = scenes.relabelled(scenes.suspension(3000, (1.0, 0.6, 0.4), 0.55, 5, dt=1e-3), 23)
    out = {}
    for ro in (0, 2):
        ctx = _ctx(R, sc, lcp_tol=1e-12, max_recursions=3, lcp_max_iter=2_000_000, reorder=ro)
        bodies = R.BodyState.from_scene(sc)
        cs = R.ConstraintStore(40000)
        rep = ctx.step(bodies, cs)
        pi, pj = ctx.get_pairs()
        pairs = np.sort(pi.cpu().numpy().astype(np.int64) * sc["n"] + pj.cpu().numpy())
        out[ro] = (rep, cs.to_numpy(), bodies.pos.cpu().numpy(), bodies.vel.cpu().numpy(), pairs)
    (r0, c0, p0, v0, q0), (r2, c2, p2, v2, q2) = out[0], out[2]
    assert r0["n_c"] == r2["n_c"] and r0["recursions"] == r2["recursions"]
    assert np.array_equal(q0, q2)
    for k in ("ia", "ib", "gen"):
        assert np.array_equal(c0[k], c2[k])
    assert np.max(np.abs(c0["phi"] - c2["phi"])) <= 1e-12
    assert np.max(np.abs(c0["n"] - c2["n"])) <= 1e-10
    lam = np.max(np.abs(c0["lam"]))
    assert np.max(np.abs(c0["lam"] - c2["lam"])) <= 1e-6 * lam
    d = p0 - p2
    d -= sc["box"] * np.rint(d / sc["box"])
    assert np.max(np.abs(d)) <= 1e-9
    assert np.max(np.abs(v0 - v2)) <= 1e-6 * max(1.0, np.max(np.abs(v0)))


def test_step_parity_overdamped_cfg2_recipe(orc, R):
    """cfg2 recipe (overdamped local drag, R12) at 400 bodies, recursion cap 1."""
    sc = scenes.cfg2(n=400)
    r, rep, _ = _compare_step(orc, R, sc, max_recursions=1)
    assert rep["status"] == R.W_RECURSION_CAP


def test_step_parity_cfg1_relaxed(orc, R):
    """cfg1-relaxed (overlap-free start): both sides stop after
    the recursion-0 solve (reduction corollary)."""
    r, rep, _ = _compare_step(orc, R, scenes.cfg1_relaxed())
    assert rep["recursions"] == 0 and rep["max_overlap"] <= 1e-5


def test_reduction_corollary_gpu(orc, R):
    """P:L895-900 on the GPU: from the overlap-free cfg1 state, dt = 1e-3 and
    1e-4 end after the recursion-0 solve, the overlap left (eta_1) matches the
    oracle's and falls ~dt^2."""
    eta = {}
    for dt in (1e-3, 1e-4):
        sc = scenes.cfg1_relaxed(dt=dt)
        r = orc.relcp_step(sc, lcp_tol=1e-12)
        ctx = _ctx(R, sc, lcp_tol=1e-12, lcp_max_iter=2_000_000)
        bodies = R.BodyState.from_scene(sc)
        cs = R.ConstraintStore(8000)
        rep = ctx.step(bodies, cs)
        assert rep["recursions"] == 0 == r["recursions"]
        assert abs(rep["max_overlap"] - r["max_overlap"]) <= 1e-9
        eta[dt] = rep["max_overlap"]
    assert eta[1e-4] < eta[1e-3] / 30.0


def test_step_parity_cfg1_bigdt(orc, R):
    """cfg1-bigdt: the relaxed start at dt = 0.1 augments several times; the
    appended rows, generations and the accepted state match the oracle."""
    r, rep, _ = _compare_step(orc, R, scenes.cfg1_relaxed(dt=0.1))
    assert rep["recursions"] >= 1 and rep["status"] == 0


@pytest.mark.parametrize("layout", [0, 1])
def test_step_parity_bigdt_augments(orc, R, layout):
    sc = scenes.suspension(300, (1.0, 0.6, 0.4), 0.3, 9, dt=2e-2)
    r, rep, _ = _compare_step(orc, R, sc, max_recursions=2, layout=layout)
    assert rep["recursions"] >= 1


@pytest.mark.parametrize("layout,cluster", [(0, 1), (1, 1), (0, 0)])
def test_step_parity_cfg5_recipe(orc, R, layout, cluster):
    """cfg5 recipe (the bench workload) at 1000 bodies, two augmentations;
    CSR with the single-cluster BB loop (default), JDS, CSR per-pass kernels."""
    sc = scenes.cfg5(n=1000)
    r, rep, _ = _compare_step(orc, R, sc, max_recursions=2, layout=layout, cluster=cluster)
    assert rep["recursions"] == 2


def test_step_deterministic(R):
    sc = scenes.cfg1()
    out = []
    for _ in range(2):
        ctx = _ctx(R, sc)
        bodies = R.BodyState.from_scene(sc)
        cs = R.ConstraintStore(8000)
        ctx.step(bodies, cs)
        out.append((bodies.pos.clone(), bodies.vel.clone(), cs.lam[:cs.count].clone()))
    assert all(torch.equal(a, b) for a, b in zip(out[0], out[1]))


@pytest.mark.parametrize("solver,cluster", [(0, 0), (0, 1), (2, 0)])
def test_timing_mode_same_result(R, solver, cluster):
    """relcp_set_timing only adds CUDA events (per kernel in the first batch,
    around each CUDA-graph replay after it; around each launch of the
    single-cluster BB loop): the step is bitwise the one run without timing,
    and the stats count the timed iterations."""
    sc = scenes.cfg1()
    out = []
    for timing in (False, True):
        ctx = _ctx(R, sc, solver=solver, lcp_tol=1e-12, cluster=cluster)
        bodies = R.BodyState.from_scene(sc)
        cs = R.ConstraintStore(8000)
        ctx.reset_stats()
        ctx.set_timing(timing)
        rep = ctx.step(bodies, cs)
        st = ctx.stats()
        out.append((bodies.pos.clone(), bodies.vel.clone(), cs.lam[:cs.count].clone()))
        iters = sum(rep["iterations"])
        assert st["lcp_iterations"] == iters
        assert (st["cluster_solves"] > 0) == (cluster == 1 and solver == 0)
        if timing and st["cluster_solves"]:
            assert st["split_timed"] == 0 and st["iter_timed"] == iters and st["iter_ms"] > 0
        elif timing:
            assert iters > 64  # several batches: direct first batch + graph replays
            assert 0 < st["split_timed"] < st["iter_timed"] <= iters
            assert st["iter_ms"] >= st["scatter_ms"] + st["gather_ms"] - 1e-9 > 0
        else:
            assert st["iter_timed"] == 0 and st["iter_ms"] == 0.0
    assert all(torch.equal(a, b) for a, b in zip(out[0], out[1]))


# ------------------------------------------------------------ cfg3 / cfg4 recipes

@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("solver", [0, 1, 2])
@pytest.mark.parametrize("c_fixed", [None, 3])
def test_cfg4_network_lcp_parity(orc, R, c_fixed, solver, layout):
    """Given chainmail network (cfg4 recipe, 16 x 16 rings): rows, q, and the
    solved LCP against the oracle.  c = 3 per link makes N_C exceed the free
    DOFs, so lambda is not unique: compare D lambda and g (Lemma 5, R13)."""
    sc = scenes.cfg4(n_side=16, c_fixed=c_fixed)
    # r <= 1e-12 on both sides: with 1-3 rows per link A is ill-conditioned and
    # r <= 1e-10 leaves lambda determined only to ~2e-6 relative (R19)
    x_ref, g_ref, info, W, rw = orc.network_lcp(sc, 1e-12)
    ctx = _ctx(R, sc, lcp_tol=1e-12, lcp_max_iter=2_000_000, solver=solver, layout=layout)
    bodies = R.BodyState.from_scene(sc)
    net = sc["network"]
    cs = R.ConstraintStore(len(net["ia"]) + 7)
    ctx.load_constraints(bodies, cs, net["ia"], net["ib"], net["n"], net["ra"], net["rb"], net["phi"])
    c = cs.to_numpy()
    assert np.max(np.abs(c["ta"] - rw["ta"])) <= 1e-15 and np.max(np.abs(c["tb"] - rw["tb"])) <= 1e-15
    assert np.max(np.abs(c["q"] - rw["q"])) <= 1e-15
    rep = ctx.solve_lcp(bodies, cs)
    assert rep["converged"] and rep["residual"] <= 1e-12
    lam = cs.lam[:cs.count].cpu().numpy()
    g = cs.g[:cs.count].cpu().numpy()
    assert np.all(lam >= 0)
    gs = max(1e-300, np.max(np.abs(g_ref)))
    assert np.max(np.abs(g - g_ref)) <= 1e-6 * gs + 1e-9
    # unique by Lemma 5: U = W D lambda everywhere, D lambda on bodies with W > 0
    F_ref, U_ref = orc.wrench(W, rw["ia"], rw["ib"], rw["n"], rw["ta"], rw["tb"], x_ref)
    F = torch.empty(sc["n"], 6, dtype=torch.float64, device="cuda")
    U = torch.empty_like(F)
    ctx.prepare_operator(bodies, cs)
    ctx.wrench(bodies, cs, cs.lam[:cs.count].contiguous(), F, U)
    free = sc["kinematic"] == 0
    assert np.max(np.abs(U.cpu().numpy() - U_ref)) <= 1e-6 * np.max(np.abs(U_ref))
    assert np.max(np.abs(F.cpu().numpy()[free] - F_ref[free])) <= 1e-6 * np.max(np.abs(F_ref[free]))
    if c_fixed is None:
        assert np.max(np.abs(lam - x_ref)) <= 1e-6 * np.max(np.abs(x_ref))
    assert np.all(U.cpu().numpy()[~free] == 0)  # kinematic rows: W = 0


def test_cfg3_step_parity(orc, R):
    """Planar growing colony (cfg3 recipe, 800 bodies, overdamped)."""
    sc = scenes.cfg3(n=800)
    r, rep, g = _compare_step(orc, R, sc, max_recursions=3)
    # planar symmetry: normals and torque arms stay in / normal to z = 0
    assert np.max(np.abs(g["n"][:, 2])) < 1e-11
    assert np.max(np.abs(r["pos"][:, 2])) < 1e-11


@pytest.mark.parametrize("hubs", [False, True])
@pytest.mark.parametrize("dynamics", [0, 1])
def test_k6_pipe_bitwise(orc, R, hubs, dynamics):
    """The TMA-staged K6 (params.k6_pipe, from 65,536 bodies)
    computes exactly the per-warp kernel's sums: apply, wrench and a fixed
    number of BB iterations are bitwise equal with the pipeline on and off,
    and the apply matches the oracle at 1e-12.  hubs: bodies with 300-700
    rows make some 32-body groups larger than a stage (warp-0 fallback)."""
    nb, nc = 70_000, 200_000
    b, ia, ib, n, ra, rb = scenes.local_constraint_network(nb, nc, 31, dynamics)
    if hubs:
        rng = np.random.default_rng(3)
        hi = np.concatenate([np.full(700, 1000), np.full(300, 40000)])
        hj = np.concatenate([rng.integers(1001, nb, 700), rng.integers(40001, nb, 300)])
        ia, ib = np.concatenate([ia, hi]).astype(np.int32), np.concatenate([ib, hj]).astype(np.int32)
        n = np.concatenate([n, rng.normal(size=(1000, 3))])
        n /= np.linalg.norm(n, axis=1, keepdims=True)
        ra = np.concatenate([ra, rng.uniform(-0.7, 0.7, (1000, 3))])
        rb = np.concatenate([rb, rng.uniform(-0.7, 0.7, (1000, 3))])
        o = np.lexsort((ib, ia))
        ia, ib, n, ra, rb = ia[o], ib[o], n[o], ra[o], rb[o]
    ta, tb = np.cross(ra, n), np.cross(rb, n)
    m = len(ia)
    x = np.random.default_rng(4).standard_normal(m)
    W = orc.body_W(b)
    y_ref = orc.delassus_apply(W, ia, ib, n, ta, tb, 1e-6, x)
    bodies = R.BodyState.from_scene(b)
    xd = torch.as_tensor(x, device="cuda")
    q = torch.as_tensor(np.random.default_rng(5).standard_normal(m) * 1e-6, device="cuda")
    out = []
    for pipe in (0, 1):
        ctx = _ctx(R, dict(dynamics=dynamics, dt=1e-3, cutoff=0.1, eps_ncp=1e-5, box=[0, 0, 0]), k6_pipe=pipe,
                   lcp_tol=1e-30, lcp_max_iter=40, layout=0)
        cs = R.ConstraintStore.from_rows(ia, ib, n, ta, tb)
        ctx.prepare_operator(bodies, cs)
        y = torch.empty_like(xd)
        ctx.delassus_apply(bodies, cs, xd, y, 1e-6)
        assert np.max(np.abs(y.cpu().numpy() - y_ref)) <= 1e-12 * np.max(np.abs(y_ref))
        F = torch.empty(nb, 6, dtype=torch.float64, device="cuda")
        U = torch.empty_like(F)
        ctx.wrench(bodies, cs, xd, F, U)
        cs.q[:m] = q
        rep = ctx.solve_lcp(bodies, cs)
        out.append((y, F, U, cs.lam[:m].clone(), cs.g[:m].clone(), rep["iterations"]))
    for a, c in zip(out[0][:5], out[1][:5]):
        assert torch.equal(a, c)
    assert out[0][5] == out[1][5] == 40


@pytest.mark.parametrize("nb,hubs", [(20_000, False), (20_000, True), (70_000, False)])
def test_k6_bodies_per_warp_bitwise(orc, R, nb, hubs):
    """K6 with 8, 16 or 32 bodies per warp (params.k6_bpw; auto = 8 up to
    RELCP_K6_SMALL_N bodies) forms every body's sum in the same
    order: apply, wrench and a fixed number of BB iterations are bitwise equal
    across the three, and the apply matches the oracle at 1e-12.  hubs: bodies
    with 300-700 rows (many tiles in one warp); ragged last group (nb % 32)."""
    nb += 13
    nc = 3 * nb
    b, ia, ib, n, ra, rb = scenes.local_constraint_network(nb, nc, 37, 0)
    if hubs:
        rng = np.random.default_rng(6)
        hi = np.concatenate([np.full(700, 1000), np.full(300, nb - 20)])
        hj = np.concatenate([rng.integers(1001, nb, 700), rng.integers(nb - 19, nb, 300)])
        ia, ib = np.concatenate([ia, hi]).astype(np.int32), np.concatenate([ib, hj]).astype(np.int32)
        n = np.concatenate([n, rng.normal(size=(1000, 3))])
        n /= np.linalg.norm(n, axis=1, keepdims=True)
        ra = np.concatenate([ra, rng.uniform(-0.7, 0.7, (1000, 3))])
        rb = np.concatenate([rb, rng.uniform(-0.7, 0.7, (1000, 3))])
        o = np.lexsort((ib, ia))
        ia, ib, n, ra, rb = ia[o], ib[o], n[o], ra[o], rb[o]
    ta, tb = np.cross(ra, n), np.cross(rb, n)
    m = len(ia)
    x = np.random.default_rng(7).standard_normal(m)
    y_ref = orc.delassus_apply(orc.body_W(b), ia, ib, n, ta, tb, 1e-6, x)
    bodies = R.BodyState.from_scene(b)
    xd = torch.as_tensor(x, device="cuda")
    q = torch.as_tensor(np.random.default_rng(8).standard_normal(m) * 1e-6, device="cuda")
    out = []
    for bpw in (8, 16, 32, 0):
        ctx = _ctx(R, dict(dynamics=0, dt=1e-3, cutoff=0.1, eps_ncp=1e-5, box=[0, 0, 0]), k6_bpw=bpw,
                   lcp_tol=1e-30, lcp_max_iter=40, layout=0, cluster=0)
        cs = R.ConstraintStore.from_rows(ia, ib, n, ta, tb)
        ctx.prepare_operator(bodies, cs)
        y = torch.empty_like(xd)
        ctx.delassus_apply(bodies, cs, xd, y, 1e-6)
        assert np.max(np.abs(y.cpu().numpy() - y_ref)) <= 1e-12 * np.max(np.abs(y_ref))
        F = torch.empty(nb, 6, dtype=torch.float64, device="cuda")
        U = torch.empty_like(F)
        ctx.wrench(bodies, cs, xd, F, U)
        cs.q[:m] = q
        rep = ctx.solve_lcp(bodies, cs)
        out.append((y, F, U, cs.lam[:m].clone(), cs.g[:m].clone(), rep["iterations"]))
    for o in out[1:]:
        for a, c in zip(out[0][:5], o[:5]):
            assert torch.equal(a, c)
        assert o[5] == 40
