"""Edge cases of the C ABI on the GPU: degenerate pairs, empty contact sets,
a single body, capacity errors, invalid parameters (include/relcp.h)."""
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


def _two(axes, pos, quat, vel):
    sc = scenes.suspension(2, (1.0, 1.0, 1.0), 0.01, 0)
    sc["axes"] = np.asarray(axes, float)
    a, b, c = sc["axes"].T
    m = 4.0 / 3.0 * math.pi * a * b * c
    sc["inv_mass"] = 1.0 / m
    sc["inv_inertia"] = 1.0 / np.stack([m / 5 * (b * b + c * c), m / 5 * (a * a + c * c), m / 5 * (a * a + b * b)], 1)
    sc["pos"], sc["quat"], sc["vel"] = np.asarray(pos, float), np.asarray(quat, float), np.asarray(vel, float)
    sc["box"] = np.zeros(3)
    return sc


def test_coincident_centres_are_degenerate(R):
    sc = _two([[1, .5, .5]] * 2, [[0, 0, 0], [0, 0, 0]], [[1, 0, 0, 0]] * 2, np.zeros((2, 6)))
    ctx = R.Context(dt=1e-3)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(16)
    with pytest.raises(R.RelcpError) as e:
        ctx.generate_contacts(bodies, cs)
    assert e.value.code == R.E_DEGENERATE
    phi, n, ra, rb, st = ctx.snsd_pairs(bodies, [0], [1])
    assert int(st[0]) == 1 and math.isnan(float(phi[0]))


def test_no_contacts_free_flight(R):
    """Bodies far apart: A_0 is empty, the step is the free motion x += dt u."""
    sc = _two([[1, .5, .5]] * 2, [[0, 0, 0], [10, 0, 0]], [[1, 0, 0, 0]] * 2,
              [[1, 2, 3, 0, 0, 0.5], [-1, 0, 0, 0.3, 0, 0]])
    ctx = R.Context(dt=1e-2)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(16)
    rep = ctx.step(bodies, cs)
    assert rep["n_c"] == [0] and rep["recursions"] == 0 and cs.count == 0
    assert np.allclose(bodies.pos.cpu().numpy(), sc["pos"] + 1e-2 * sc["vel"][:, :3], atol=1e-15)
    assert np.allclose(bodies.vel.cpu().numpy(), sc["vel"], atol=0)
    q = bodies.quat.cpu().numpy()
    assert np.allclose(np.linalg.norm(q, axis=1), 1.0, atol=1e-15)


def test_single_body(R):
    sc = _two([[1, .5, .5]], [[1, 2, 3]], [[1, 0, 0, 0]], [[0.1, 0, 0, 0, 0, 0]])
    sc["inv_mass"], sc["inv_inertia"] = sc["inv_mass"][:1], sc["inv_inertia"][:1]
    ctx = R.Context(dt=1e-2)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(4)
    n0, _ = ctx.generate_contacts(bodies, cs)
    assert n0 == 0
    rep = ctx.solve_lcp(bodies, cs)
    assert rep["converged"] and rep["iterations"] == 0


def test_augment_capacity_error_reports_size(R):
    sc = scenes.suspension(300, (1.0, 0.6, 0.4), 0.3, 9, dt=2e-2)
    ctx = R.Context(dt=sc["dt"], box=list(sc["box"]), lcp_tol=1e-8)
    bodies = R.BodyState.from_scene(sc)
    probe = R.ConstraintStore(4000)
    n0, _ = ctx.generate_contacts(bodies, probe)
    cs = R.ConstraintStore(n0)  # room for A_0 only
    ctx.generate_contacts(bodies, cs)
    ctx.solve_lcp(bodies, cs)
    with pytest.raises(R.RelcpError) as e:
        ctx.check_and_augment(bodies, cs, 1)
    assert e.value.code == R.E_CAPACITY and cs.count > n0


def test_check_requires_generate(R):
    sc = scenes.cfg1()
    ctx = R.Context(dt=sc["dt"], box=list(sc["box"]))
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(4000)
    with pytest.raises(R.RelcpError) as e:
        ctx.check_and_augment(bodies, cs, 1)
    assert e.value.code == R.E_STATE


def test_invalid_params_refused(R):
    with pytest.raises(R.RelcpError):
        R.Context(dt=-1.0)
    with pytest.raises(R.RelcpError):
        R.Context(solver=7)
    ctx = R.Context()
    with pytest.raises(R.RelcpError):
        ctx.set_params(max_recursions=1000)


def test_generate_capacity_error_reports_size(R):
    """A_0 larger than the store: E_CAPACITY with the required row count in
    `count` (include/relcp.h), nothing written past capacity."""
    sc = scenes.cfg1()
    ctx = R.Context(dt=sc["dt"], box=list(sc["box"]))
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(16)
    guard = cs.ia.clone()
    with pytest.raises(R.RelcpError) as e:
        ctx.generate_contacts(bodies, cs)
    assert e.value.code == R.E_CAPACITY and cs.count > 16
    assert torch.equal(cs.ia, guard)


def test_nan_input_is_refused(R):
    """A NaN in q: the solve stops with E_NAN instead of iterating on NaNs."""
    sc = scenes.cfg1()
    ctx = R.Context(dt=sc["dt"], box=list(sc["box"]))
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(4000)
    ctx.generate_contacts(bodies, cs)
    cs.q[3] = float("nan")
    with pytest.raises(R.RelcpError) as e:
        ctx.solve_lcp(bodies, cs)
    assert e.value.code == R.E_NAN


@pytest.mark.parametrize("solver", [0, 1, 2])
def test_iteration_cap_returns_warning(R, solver):
    """lcp_max_iter reached: W_MAX_ITER (> 0, not an error), exactly the cap
    executed, the last iterate returned projected (lambda >= 0)."""
    sc = scenes.cfg5(n=1000)  # its A_0 needs ~150 BB iterations at 1e-8
    ctx = R.Context(dt=sc["dt"], box=list(sc["box"]), lcp_tol=1e-14, lcp_max_iter=37, solver=solver)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(4000)
    ctx.generate_contacts(bodies, cs)
    rep = ctx.solve_lcp(bodies, cs)
    assert rep["status"] == R.W_MAX_ITER and not rep["converged"]
    assert rep["iterations"] == 37 and rep["residual"] > 1e-14
    assert bool((cs.lam[:cs.count] >= 0).all())
