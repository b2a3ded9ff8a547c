"""Multi-step drivers against the oracle stepped
through the same schedule: cfg2 compaction (box rescale), cfg3 growth, and
the LCP-SNSD vs ReLCP overlap contrast."""
import numpy as np
import pytest

from gen import scenes

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def D():
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    from paper_2506_14097_b200 import drivers
    return drivers


def _oracle_steps(orc, sc, n_steps, before_step, max_recursions):
    sc = dict(sc)
    sc["pos"], sc["quat"], sc["axes"], sc["box"] = (sc["pos"].copy(), sc["quat"].copy(), sc["axes"].copy(),
                                                    sc["box"].copy())
    n_c = []
    for k in range(n_steps):
        before_step(k, sc)
        r = orc.relcp_step(sc, lcp_tol=1e-12, max_recursions=max_recursions)
        sc["pos"], sc["quat"] = r["pos"], r["quat"]
        n_c.append(r["n_c"])
    return sc, n_c


def test_compaction_driver_parity(orc, D):
    sc = scenes.cfg2(n=300)
    steps, phi_end = 200, 0.55
    L0, phi0 = float(sc["box"][0]), sc["phi"]

    def before(k, s):
        L_old = float(s["box"][0])
        L_new = D.box_length(phi0, L0, phi0 + (phi_end - phi0) * (k + 1) / steps)
        s["pos"] = s["pos"] * (L_new / L_old)
        s["box"] = np.full(3, L_new)

    ref, n_c_ref = _oracle_steps(orc, sc, 3, before, 2)
    reps, bodies, cs = D.compaction(sc, steps=steps, phi_end=phi_end, stop_after=3, lcp_tol=1e-12,
                                    lcp_max_iter=2_000_000, max_recursions=2)
    assert [r["n_c"] for r in reps] == n_c_ref
    assert abs(reps[-1]["box"] - ref["box"][0]) <= 1e-12 * ref["box"][0]
    d = bodies.pos.cpu().numpy() - ref["pos"]
    d -= ref["box"] * np.rint(d / ref["box"])
    assert np.max(np.abs(d)) <= 1e-8
    assert np.max(np.abs(bodies.quat.cpu().numpy() - ref["quat"])) <= 1e-8


def test_growth_driver_parity(orc, D):
    sc = scenes.cfg3(n=500)
    grow = sc["growing"]

    def before(k, s):
        if k > 0:
            s["axes"][grow, 0] += 0.01

    ref, n_c_ref = _oracle_steps(orc, sc, 3, before, 2)
    reps, bodies, cs = D.growth(sc, steps=3, lcp_tol=1e-12, lcp_max_iter=2_000_000, max_recursions=2)
    assert [r["n_c"] for r in reps] == n_c_ref
    assert np.max(np.abs(bodies.axes.cpu().numpy() - ref["axes"])) == 0.0
    assert np.max(np.abs(bodies.pos.cpu().numpy() - ref["pos"])) <= 1e-8


def test_snsd_vs_relcp_overlap(D):
    """The paper's point: the plain SNSD LCP leaves true
    overlaps that the ReLCP recursion removes (down to eps_NCP)."""
    sc = scenes.suspension(300, (1.0, 0.6, 0.4), 0.3, 9, dt=2e-2)
    out = D.snsd_vs_relcp(sc, lcp_tol=1e-10, lcp_max_iter=2_000_000)
    assert out["relcp"]["status"] == 0 and out["relcp"]["max_overlap"] <= sc["eps_ncp"]
    assert out["snsd"]["max_overlap"] > 10 * sc["eps_ncp"]
    assert out["snsd"]["recursions"] == 0
