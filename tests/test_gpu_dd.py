"""Domain-decomposed Delassus apply, BB solve and ReLCP step (SURVEY §8(e) / §8(f) rank 4,
DESIGN.md §8) on one GPU as K virtual parts (halo exchange by device copies),
and the NCCL transport at world size 1, against the CPU oracle:

* apply y = s D^T W D x: 1e-12 of ||y||_inf
  for K = 1..6 parts, empty parts, kinematic bodies, random (all-ghost) and
  lattice-local networks; K = 1 is bitwise the single-domain apply; every K is
  bitwise reproducible run to run (fixed-order halo sums, no atomics);
* solve (Lemma 3): lambda, D lambda and g against the oracle's BB
  solution at 1e-6 with r <= tol, on cfg1's A_0 and the cfg4 ring network;
* 2M bodies x 10M rows (cfg5 scale) in 4 parts: every output at 1e-12.
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


def _offsets(n, K, empty=None):
    off = [round(k * n / K) for k in range(K + 1)]
    if empty is not None:
        off[empty + 1] = off[empty]
    return np.array(off, dtype=np.int64)


def _net(kind, nb, nc, seed, dynamics=0, kinematic=False):
    fn = scenes.local_constraint_network if kind == "local" else scenes.random_constraint_network
    b, ia, ib, n, ra, rb = fn(nb, nc, seed, dynamics)
    if kinematic:
        b["kinematic"] = (np.arange(nb) % 17 == 0).astype(np.int32)
    return b, ia, ib, n, np.cross(ra, n), np.cross(rb, n)


@pytest.mark.parametrize("K,kind,empty,kin", [(1, "local", None, False), (2, "local", None, True),
                                              (3, "random", None, False), (4, "local", 1, False),
                                              (6, "random", 0, True)])
def test_dd_apply_virtual(orc, R, K, kind, empty, kin):
    b, ia, ib, n, ta, tb = _net(kind, 20000, 70000, 11 + K, kinematic=kin)
    W = orc.body_W(b)
    x = np.random.default_rng(K).standard_normal(len(ia))
    s = 1e-6
    y_ref = orc.delassus_apply(W, ia, ib, n, ta, tb, s, x)
    _, U_ref = orc.wrench(W, ia, ib, n, ta, tb, x)
    bodies = R.BodyState.from_scene(b)
    cs = R.ConstraintStore.from_rows(ia, ib, n, ta, tb)
    dd = R.DomainDecomposition(_offsets(b["n"], K, empty), dynamics=0, dt=1e-3, box=[0, 0, 0])
    dd.load(bodies, cs)
    assert sum(dd.info(k)["row_hi"] - dd.info(k)["row_lo"] for k in range(K)) == len(ia)
    xd = torch.as_tensor(x, device="cuda")
    y1, y2 = torch.empty_like(xd), torch.empty_like(xd)
    dd.delassus_apply(xd, y1, s)
    U = torch.empty(b["n"], 6, dtype=torch.float64, device="cuda")
    dd.get_u(U)
    dd.delassus_apply(xd, y2, s)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)  # deterministic
    y = y1.cpu().numpy()
    assert np.max(np.abs(y - y_ref)) <= 1e-12 * np.max(np.abs(y_ref))
    assert np.max(np.abs(U.cpu().numpy() - U_ref)) <= 1e-12 * np.max(np.abs(U_ref))
    if K == 1:  # one part: the single-domain operator, bit for bit
        ctx = R.Context(dynamics=0, dt=1e-3, box=[0, 0, 0])
        ctx.prepare_operator(bodies, cs)
        ys = torch.empty_like(xd)
        ctx.delassus_apply(bodies, cs, xd, ys, s)
        torch.cuda.synchronize()
        assert torch.equal(ys, y1)


def test_dd_apply_fullsize_4parts(orc, R):
    """2M bodies, 10M rows in 4 virtual parts (cfg5 scale): y and U at 1e-12."""
    b, ia, ib, n, ta, tb = _net("local", 2_000_000, 10_000_000, 77)
    W = orc.body_W(b)
    x = np.random.default_rng(1).standard_normal(len(ia))
    y_ref = orc.delassus_apply(W, ia, ib, n, ta, tb, 1e-6, x)
    bodies = R.BodyState.from_scene(b)
    cs = R.ConstraintStore.from_rows(ia, ib, n, ta, tb)
    dd = R.DomainDecomposition(_offsets(b["n"], 4), dynamics=0, dt=1e-3, box=[0, 0, 0])
    dd.load(bodies, cs)
    xd = torch.as_tensor(x, device="cuda")
    y = torch.empty_like(xd)
    dd.delassus_apply(xd, y, 1e-6)
    assert np.max(np.abs(y.cpu().numpy() - y_ref)) <= 1e-12 * np.max(np.abs(y_ref))
    info = [dd.info(k) for k in range(4)]
    assert all(i["n_ghost"] > 0 for i in info[:3]) and info[3]["n_recv"] > 0


@pytest.fixture(scope="module")
def cfg1_a0(orc):
    sc = scenes.cfg1()
    ref = orc.relcp_step(sc, lcp_tol=1e-12, max_recursions=0, snsd_only=True)
    return sc, ref


@pytest.mark.parametrize("K", [1, 3, 5])
def test_dd_solve_cfg1_a0(orc, R, cfg1_a0, K):
    """cfg1's A_0 LCP split over K parts: the oracle's BB solution (r <= 1e-12)."""
    sc, ref = cfg1_a0
    c = ref["constraints"]
    ia, ib, n, ta, tb, q = c["ia"], c["ib"], c["n"], c["ta"], c["tb"], ref["q_hist"][0]
    o = np.lexsort((ib, ia))  # the DD needs rows sorted by ia (R18)
    ia, ib, n, ta, tb, q = ia[o], ib[o], n[o], ta[o], tb[o], q[o]
    x_ref = c["lam"][o]
    g_ref = ref["g_hist"][0][o]
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore.from_rows(ia, ib, n, ta, tb, q=q)
    dd = R.DomainDecomposition(_offsets(sc["n"], K), dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]),
                               lcp_tol=1e-12, lcp_max_iter=2_000_000)
    dd.load(bodies, cs)
    rep = dd.solve_lcp(cs)
    assert rep["converged"] and rep["residual"] <= 1e-12
    lam = cs.lam[:cs.count].cpu().numpy()
    g = cs.g[:cs.count].cpu().numpy()
    assert np.all(lam >= 0)
    assert np.max(np.abs(lam - x_ref)) <= 1e-6 * np.max(np.abs(x_ref))
    assert np.max(np.abs(g - g_ref)) <= 1e-6 * np.max(np.abs(g_ref)) + 1e-12
    W = orc.body_W(sc)
    _, U_ref = orc.wrench(W, ia, ib, n, ta, tb, x_ref)
    U = torch.empty(sc["n"], 6, dtype=torch.float64, device="cuda")
    dd.get_u(U)  # U = W D x of the last scatter: the final iterate's
    # single-domain solve of the same LCP on the GPU: same solution
    cs2 = R.ConstraintStore.from_rows(ia, ib, n, ta, tb, q=q)
    ctx = R.Context(dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]), lcp_tol=1e-12,
                    lcp_max_iter=2_000_000)
    ctx.solve_lcp(bodies, cs2)
    assert np.max(np.abs(cs2.lam[:cs2.count].cpu().numpy() - lam)) <= 1e-6 * np.max(np.abs(x_ref))


@pytest.mark.parametrize("K", [2, 4])
def test_dd_solve_cfg4_rings(orc, R, K):
    """cfg4 ring network (16 x 16, kinematic boundary rows): lambda, U, g."""
    sc = scenes.cfg4(n_side=16)
    x_ref, g_ref, info, W, rw = orc.network_lcp(sc, 1e-12)
    net = sc["network"]
    bodies = R.BodyState.from_scene(sc)
    ctx = R.Context(dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]), lcp_tol=1e-12,
                    lcp_max_iter=2_000_000)
    cs = R.ConstraintStore(len(net["ia"]) + 7)
    ctx.load_constraints(bodies, cs, net["ia"], net["ib"], net["n"], net["ra"], net["rb"], net["phi"])
    dd = R.DomainDecomposition(_offsets(sc["n"], K), dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]),
                               lcp_tol=1e-12, lcp_max_iter=2_000_000)
    dd.load(bodies, cs)
    rep = dd.solve_lcp(cs)
    assert rep["converged"] and rep["residual"] <= 1e-12
    lam = cs.lam[:cs.count].cpu().numpy()
    g = cs.g[:cs.count].cpu().numpy()
    assert np.max(np.abs(g - g_ref)) <= 1e-6 * np.max(np.abs(g_ref)) + 1e-9
    assert np.max(np.abs(lam - x_ref)) <= 1e-6 * np.max(np.abs(x_ref))


def test_dd_nccl_world1(orc, R):
    """The NCCL transport (one rank, one GPU): same operator as one virtual part."""
    b, ia, ib, n, ta, tb = _net("local", 5000, 16000, 5)
    uid = R.dd_nccl_unique_id()
    bodies = R.BodyState.from_scene(b)
    cs = R.ConstraintStore.from_rows(ia, ib, n, ta, tb)
    off = _offsets(b["n"], 1)
    dn = R.DomainDecomposition(off, rank=0, nccl_uid=uid, dynamics=0, dt=1e-3, box=[0, 0, 0])
    dv = R.DomainDecomposition(off, dynamics=0, dt=1e-3, box=[0, 0, 0])
    dn.load(bodies, cs)
    dv.load(bodies, cs)
    x = torch.rand(len(ia), dtype=torch.float64, device="cuda")
    y1, y2 = torch.empty_like(x), torch.empty_like(x)
    dn.delassus_apply(x, y1, 1e-6)
    dv.delassus_apply(x, y2, 1e-6)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    q = torch.as_tensor(np.random.default_rng(2).standard_normal(len(ia)) * 1e-3, device="cuda")
    cs.q[:len(ia)] = q
    cs.lam.zero_()
    rep = dn.solve_lcp(cs)
    assert rep["converged"]
    lam1 = cs.lam[:len(ia)].clone()
    cs.lam.zero_()
    rep2 = dv.solve_lcp(cs)
    assert rep2["iterations"] == rep["iterations"]
    assert torch.equal(lam1, cs.lam[:len(ia)])


# ------------------------------------------------------------ domain-decomposed ReLCP step

def _dd_step_vs_oracle(orc, R, sc, K, max_recursions, rank=-1, uid=None):
    """relcp_dd_step (LCP solves split over K parts) against the oracle's
    Algorithm-1 step: same recursions and N_C per recursion, identical
    (ia, ib, gen) rows, configurations to 1e-9 (both sides solve every LCP to
    r <= 1e-12, as tests/test_gpu_parity.py _compare_step)."""
    r = orc.relcp_step(sc, lcp_tol=1e-12, max_recursions=max_recursions)
    dd = R.DomainDecomposition(_offsets(sc["n"], K), rank=rank, nccl_uid=uid, dynamics=sc["dynamics"],
                               dt=sc["dt"], box=list(sc["box"]), cutoff=sc["cutoff"], eps_ncp=sc["eps_ncp"],
                               xi=sc.get("xi", 1.0), lcp_tol=1e-12, lcp_max_iter=2_000_000,
                               max_recursions=max_recursions)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(8 * max(1, len(r["constraints"]["ia"])) + 64)
    rep = dd.step(bodies, cs)
    assert rep["recursions"] == r["recursions"] and rep["n_c"] == r["n_c"]
    assert (rep["status"] != 0) == (r["status"] != 0)
    g, c = cs.to_numpy(), r["constraints"]
    og, oo = np.lexsort((g["ib"], g["ia"], g["gen"])), np.lexsort((c["ib"], c["ia"], c["gen"]))
    for k in ("ia", "ib", "gen"):
        assert np.array_equal(g[k][og], c[k][oo])
    dpos = bodies.pos.cpu().numpy() - r["pos"]
    if np.all(sc["box"] > 0):
        dpos -= sc["box"] * np.rint(dpos / sc["box"])
    assert np.max(np.abs(dpos)) <= 1e-9
    assert np.max(np.abs(bodies.quat.cpu().numpy() - r["quat"])) <= 1e-9
    assert rep["max_overlap"] <= sc["eps_ncp"] or rep["status"] != 0
    dd.close()
    return rep, bodies, cs


@pytest.mark.parametrize("K", [1, 2, 3])
def test_dd_step_cfg5_recipe(orc, R, K):
    """The bench workload's recipe at 1000 bodies, two augmentations.  The
    generation's SNSD runs split by the owner of i (DistSpec): the A_0 rows
    (gen 0, found at C^k before any solve) are bitwise the single-domain
    step's."""
    sc = scenes.cfg5(n=1000)
    rep, _, cs = _dd_step_vs_oracle(orc, R, sc, K, max_recursions=2)
    assert rep["recursions"] == 2
    ctx = R.Context(dynamics=sc["dynamics"], dt=sc["dt"], box=list(sc["box"]), cutoff=sc["cutoff"],
                    eps_ncp=sc["eps_ncp"], lcp_tol=1e-12, lcp_max_iter=2_000_000, max_recursions=2)
    b1 = R.BodyState.from_scene(sc)
    c1 = R.ConstraintStore(cs.capacity)
    ctx.step(b1, c1)
    g1, g2 = c1.to_numpy(), cs.to_numpy()
    m1, m2 = g1["gen"] == 0, g2["gen"] == 0
    for k in ("ia", "ib", "n", "ta", "tb", "phi"):
        assert np.array_equal(g1[k][m1], g2[k][m2]), k


@pytest.mark.parametrize("K", [2, 4])
def test_dd_step_cfg1(orc, R, K):
    _dd_step_vs_oracle(orc, R, scenes.cfg1(), K, max_recursions=50)


def test_dd_step_nccl_world1(orc, R):
    """NCCL transport at world size 1: the same step as one virtual part, bitwise."""
    sc = scenes.cfg5(n=1000)
    rep_n, b_n, cs_n = _dd_step_vs_oracle(orc, R, sc, 1, 2, rank=0, uid=R.dd_nccl_unique_id())
    rep_v, b_v, cs_v = _dd_step_vs_oracle(orc, R, sc, 1, 2)
    assert rep_n["iterations"] == rep_v["iterations"]
    assert torch.equal(b_n.pos, b_v.pos) and torch.equal(b_n.quat, b_v.quat) and torch.equal(b_n.vel, b_v.vel)
    assert torch.equal(cs_n.lam[:cs_n.count], cs_v.lam[:cs_v.count])
