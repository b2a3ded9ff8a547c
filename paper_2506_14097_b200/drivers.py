"""Multi-step drivers over the C-ABI hot path.

Scenario mechanics only (box rescale, axial growth); every time step is one
`relcp_step` (Algorithm 1) in the CUDA library.

* compaction(...)  cfg2: periodic cube shrunk from phi_0 to phi_end linearly
  in phi over `steps` steps; the centres are rescaled affinely with the box at
  the start of each step (BASELINE cfg2).
* growth(...)      cfg3: a fixed half of the bodies grows its major semi-axis
  by `rate` at the start of every step after the first (the scene already
  holds the first step's growth; BASELINE cfg3).
* snsd_vs_relcp(...) the paper's LCP-SNSD baseline (max_recursions = 0: the
  A_0 solution is accepted as is) against ReLCP on the same state:
  the overlap that remains at the accepted configuration.
"""
from __future__ import annotations

import math

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
                bodies.axes[grow, 0] *= math.exp(sc["dt"])
            else:
                bodies.axes[grow, 0] += rate
        rep = ctx.step(bodies, cs)
        rep.update(step=k)
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


__all__ = ["compaction", "growth", "snsd_vs_relcp", "box_length", "math"]
