"""Multi-step drivers over the C-ABI hot path.

Scenario mechanics only (box rescale, axial growth); every time step is one
`relcp_step` (Algorithm 1) in the CUDA library.

* compaction(...)  cfg2: periodic cube shrunk from phi_0 to phi_end linearly
  in phi over `steps` steps; the centres are rescaled affinely with the box at
  the start of each step (BASELINE cfg2).
* growth(...)      cfg3: a fixed half of the bodies grows its major semi-axis
  by `rate` at the start of every step after the first (the scene already
  holds the first step's growth; BASELINE cfg3).
* colony(...)      the paper's colony: rods grow
  l <- l e^dt (R22) and divide at 2 l_0 (R28, divide_rods).
* snsd_vs_relcp(...) the paper's LCP-SNSD baseline (max_recursions = 0: the
  A_0 solution is accepted as is) against ReLCP on the same state:
  the overlap that remains at the accepted configuration.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import relcp as R


def _ctx_for(sc, **kw):
    p = dict(dynamics=sc["dynamics"], dt=sc["dt"], cutoff=sc["cutoff"], eps_ncp=sc["eps_ncp"],
             box=list(sc["box"]), xi=sc.get("xi", 1.0))
    p.update(kw)
    return R.Context(**p)


def compaction(sc, steps: int = 200, phi_end: float = 0.55, capacity_per_body: int = 16, callback=None,
               stop_after: int | None = None, **kw):
    """Run the compaction (optionally only its first `stop_after` steps);
    returns the per-step reports (+ box length, phi), bodies, store."""
    ctx = _ctx_for(sc, **kw)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(capacity_per_body * sc["n"] + 1024)
    phi0 = sc["phi"]
    L0 = float(sc["box"][0])
    L = L0
    reps = []
    for k in range(steps if stop_after is None else min(steps, stop_after)):
        phi_k = phi0 + (phi_end - phi0) * (k + 1) / steps
        L_new = L0 * (phi0 / phi_k) ** (1.0 / 3.0)
        bodies.pos.mul_(L_new / L)  # affine rescale of the centres with the box
        L = L_new
        ctx.set_params(box=[L, L, L])
        rep = ctx.step(bodies, cs)
        rep.update(step=k, box=L, phi=phi_k)
        reps.append(rep)
        if callback:
            callback(k, bodies, cs, rep)
    return reps, bodies, cs


def growth(sc, steps: int = 10, rate: float = 0.01, capacity_per_body: int = 16, callback=None, **kw):
    """Run the growing colony; returns the per-step reports."""
    ctx = _ctx_for(sc, **kw)
    bodies = R.BodyState.from_scene(sc)
    cs = R.ConstraintStore(capacity_per_body * sc["n"] + 1024)
    grow = torch.as_tensor(sc["growing"], device=bodies.axes.device)
    shape = sc.get("shape")
    rods = shape is not None and bool((shape == 1).all())  # colony rods: l_dot = l
    reps = []
    for k in range(steps):
        if k > 0:
            if rods:
                grow_rods(bodies, sc["dt"], grow)
            else:
                bodies.axes[grow, 0] += rate
        rep = ctx.step(bodies, cs)
        rep.update(step=k)
        reps.append(rep)
        if callback:
            callback(k, bodies, cs, rep)
    return reps, bodies, cs


DIV_ANGLE = 0.01 * math.pi / 180.0  # +-0.01 degrees


def grow_rods(bodies, dt: float, mask=None):
    """l_dot = l on the tip-to-tip length l = 2 (axes[:, 0] + r) (P:L1030,
    R22): l <- l e^dt, i.e. the centreline half-length a0 <- (a0 + r) e^dt - r."""
    a = bodies.axes
    if mask is None:
        a[:, 0] = (a[:, 0] + a[:, 1]) * math.exp(dt) - a[:, 1]
    else:
        a[mask, 0] = (a[mask, 0] + a[mask, 1]) * math.exp(dt) - a[mask, 1]


def _qmul(a, b):
    """Hamilton product of (..., 4) quaternions (s, x, y, z)."""
    s1, x1, y1, z1 = a.unbind(-1)
    s2, x2, y2, z2 = b.unbind(-1)
    return torch.stack([s1 * s2 - x1 * x2 - y1 * y2 - z1 * z2, s1 * x2 + x1 * s2 + y1 * z2 - z1 * y2,
                        s1 * y2 - x1 * z2 + y1 * s2 + z1 * x2, s1 * z2 + x1 * y2 - y1 * x2 + z1 * s2], -1)


def divide_rods(bodies, l0: float, rng):
    """Cell division of the colony (reading R28).
    Every rod whose tip-to-tip length l = 2 (axes[:, 0] + r) has reached 2 l0
    is split at its mid cross-section into two daughters of length l / 2 (= l0
    at l = 2 l0, so the population doubles every ln 2 under l_dot = l): centres
    x -+ (l/4) u along the mother's axis u, centreline l/2 - 2 r, touching tip
    to tip at x and filling the mother's extent (no new overlap).  Each daughter is
    turned by a random +-0.01 degrees about the plane normal z (world frame,
    q <- q_z(delta) q); the signs are drawn from `rng` (numpy Generator),
    two per division in ascending mother order.  Daughter A keeps the
    mother's index, daughter B is appended (mother order).  Scenario
    mechanics between steps, on the device arrays; returns the new BodyState
    and the number of divisions."""
    a = bodies.axes
    idx = torch.nonzero(2.0 * (a[:, 0] + a[:, 1]) >= 2.0 * l0).flatten()
    m = int(idx.numel())
    if m == 0:
        return bodies, 0
    q = bodies.quat[idx]
    q = q / q.norm(dim=1, keepdim=True)
    s, x, y, z = q.unbind(-1)
    u = torch.stack([1 - 2 * (y * y + z * z), 2 * (x * y + s * z), 2 * (x * z - s * y)], -1)  # R(q) e_x
    r = a[idx, 1]
    ell = 2.0 * (a[idx, 0] + r)  # tip-to-tip length
    off = (0.25 * ell)[:, None] * u
    sg = torch.as_tensor(rng.choice(np.array([-1.0, 1.0]), size=(m, 2)), dtype=torch.float64, device=a.device)
    half = 0.5 * DIV_ANGLE * sg
    qz = torch.stack([torch.cos(half), torch.zeros_like(half), torch.zeros_like(half), torch.sin(half)], -1)
    qa, qb = _qmul(qz[:, 0], q), _qmul(qz[:, 1], q)
    pos = bodies.pos.clone()
    quat = bodies.quat.clone()
    axes = bodies.axes.clone()
    x0 = pos[idx]
    pos[idx] = x0 - off
    quat[idx] = qa
    axes[idx, 0] = 0.25 * ell - r
    new_axes = torch.stack([0.25 * ell - r, r, a[idx, 2]], -1)

    def cat(t, extra):
        return None if t is None else torch.cat([t, extra]).contiguous()

    nb = R.BodyState.__new__(R.BodyState)
    nb.pos = cat(pos, x0 + off)
    nb.quat = cat(quat, qb)
    nb.axes = cat(axes, new_axes)
    nb.vel = cat(bodies.vel, torch.zeros(m, 6, dtype=torch.float64, device=a.device))
    nb.inv_mass = cat(bodies.inv_mass, bodies.inv_mass[idx] if bodies.inv_mass is not None else None)
    nb.inv_inertia = cat(bodies.inv_inertia, bodies.inv_inertia[idx] if bodies.inv_inertia is not None else None)
    nb.kinematic = cat(bodies.kinematic, bodies.kinematic[idx] if bodies.kinematic is not None else None)
    nb.shape = cat(bodies.shape, bodies.shape[idx] if bodies.shape is not None else None)
    nb.n = nb.pos.shape[0]
    return nb, m


def colony(sc, steps: int = 10, l0: float = 2.0, seed: int = 1030, capacity_per_body: int = 16, callback=None,
           **kw):
    """The growing and dividing colony: at the start
    of every step after the first, every rod grows l <- l e^dt (grow_rods, R22) and the
    rods at 2 l0 divide (divide_rods, R28); then one relcp_step.  Returns the
    per-step reports (with the body count and divisions), the bodies, the
    store."""
    ctx = _ctx_for(sc, **kw)
    bodies = R.BodyState.from_scene(sc)
    rng = np.random.Generator(np.random.PCG64(seed))
    reps = []
    cs = None
    for k in range(steps):
        ndiv = 0
        if k > 0:
            grow_rods(bodies, sc["dt"])
            bodies, ndiv = divide_rods(bodies, l0, rng)
        if cs is None or cs.capacity < capacity_per_body * bodies.n:
            cs = R.ConstraintStore(2 * capacity_per_body * bodies.n + 1024)
        rep = ctx.step(bodies, cs)
        rep.update(step=k, n_bodies=bodies.n, divisions=ndiv)
        reps.append(rep)
        if callback:
            callback(k, bodies, cs, rep)
    return reps, bodies, cs


def snsd_vs_relcp(sc, capacity_per_body: int = 16, **kw):
    """Max overlap left by one LCP-SNSD step (no recursion) and one ReLCP step."""
    out = {}
    for name, rec in (("snsd", 0), ("relcp", kw.pop("max_recursions", 50))):
        ctx = _ctx_for(sc, max_recursions=rec, **kw)
        bodies = R.BodyState.from_scene(sc)
        cs = R.ConstraintStore(capacity_per_body * sc["n"] + 1024)
        rep = ctx.step(bodies, cs)
        out[name] = dict(max_overlap=rep["max_overlap"], recursions=rep["recursions"], n_c=rep["n_c"],
                         status=rep["status"])
    return out


def relax(sc, dt: float = 1e-2, max_steps: int = 40, target: float | None = None, capacity_per_body: int = 16,
          callback=None, **kw):
    """Overdamped relaxation of a (possibly overlapping) scene to an
    overlap-free state: ReLCP steps (Algorithm 1, overdamped form
    P:L512-522, local drag P:L928-944) with zero velocity and no external
    force until the accepted state's candidate scan has max overlap <= target
    (default eps_NCP / 2, inside the stopping rule P:L645-648).  This is the
    SURVEY §8(d) "-relaxed" companion construction (the theory assumes an
    overlap-free start).  Returns (pos, quat, reports)."""
    s = dict(sc)
    s.update(dynamics=R.OVERDAMPED, dt=dt)
    kw.setdefault("max_recursions", 50)
    kw.setdefault("lcp_tol", 1e-8)
    ctx = _ctx_for(s, **kw)
    bodies = R.BodyState.from_scene(s)
    bodies.vel.zero_()
    cs = R.ConstraintStore(capacity_per_body * sc["n"] + 1024)
    tgt = 0.5 * sc["eps_ncp"] if target is None else target
    reps = []
    for k in range(max_steps):
        rep = ctx.step(bodies, cs)
        rep.update(step=k)
        reps.append(rep)
        if callback:
            callback(k, bodies, cs, rep)
        if rep["status"] == 0 and rep["max_overlap"] <= tgt:
            break
    else:
        raise RuntimeError(f"relax: max overlap {reps[-1]['max_overlap']:.3e} > {tgt:.1e} after {max_steps} steps")
    return bodies.pos.clone(), bodies.quat.clone(), reps


def box_length(phi0: float, L0: float, phi: float) -> float:
    """Cube edge at volume fraction phi for the same bodies (phi L^3 = const)."""
    return L0 * (phi0 / phi) ** (1.0 / 3.0)


__all__ = ["compaction", "growth", "colony", "divide_rods", "grow_rods", "snsd_vs_relcp", "box_length", "math"]
