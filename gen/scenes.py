"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module only DRAWS inputs (body centres, orientations, shapes, velocities,
masses, box sizes, step parameters).  It holds none of the ReLCP method's
arithmetic: no signed distances, no Jacobian rows, no mobility, no LCP.  Both
the CPU oracle (`oracle/`) and the CUDA path (`paper_2506_14097_b200/`) read
the same dicts produced here; neither imports the other.

Recipes follow BASELINE.json `configs` as read in SURVEY.md §8(d):

* cfg1  512 prolate ellipsoids (1.0, 0.5, 0.5), rho = 1, periodic cube at
  volume fraction 0.30, jittered 8^3 lattice, uniform random quaternions,
  u, w ~ N(0, 1), dt = 1e-3, inertial.
* cfg2  20,000 prolate ellipsoids a = 1, b = c = 1/r, r ~ U(1, 4), periodic
  cube at phi = 0.40 (start of the 0.40 -> 0.55 compaction), jittered 28^3
  lattice, zero velocity, dt = 1e-2, overdamped local drag (xi = 1).
* cfg5  2,000,000 ellipsoids (1.0, 0.6, 0.4), phi = 0.55, jittered 126^3
  lattice, u, w ~ N(0, 1), dt = 1e-3, inertial.  `suspension()` builds the
  same recipe at any body count (parity tests use small counts).

Draws are consumed in a fixed order: site choice, jitter, orientations, shape
parameters, velocities.  RNG = numpy PCG64(seed).  The chosen lattice sites
are kept in lattice (x fastest) order, so body index order is spatially
coherent.
"""
from __future__ import annotations

import math

import numpy as np

INERTIAL = 0
OVERDAMPED = 1


def _uniform_quaternions(rng: np.random.Generator, n: int) -> np.ndarray:
    """Uniform random unit quaternions (s, wx, wy, wz): normalised 4-D Gaussian."""
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q


def _ellipsoid_mass_props(axes: np.ndarray, rho: float = 1.0):
    """Uniform-density solid ellipsoid: m = rho 4/3 pi abc,
    I = m/5 diag(b^2+c^2, a^2+c^2, a^2+b^2) (body property input)."""
    a, b, c = axes[:, 0], axes[:, 1], axes[:, 2]
    m = rho * 4.0 / 3.0 * math.pi * a * b * c
    inertia = np.stack([m / 5.0 * (b * b + c * c),
                        m / 5.0 * (a * a + c * c),
                        m / 5.0 * (a * a + b * b)], axis=1)
    return 1.0 / m, 1.0 / inertia


def _jittered_lattice(rng, n, n_side, box, jitter=0.1):
    """Choose n of n_side^3 sites (seeded permutation), keep them in lattice
    order, jitter each by U(-jitter, jitter) * spacing per axis."""
    n_sites = n_side ** 3
    if n > n_sites:
        raise ValueError("not enough lattice sites")
    chosen = np.sort(rng.permutation(n_sites)[:n])
    ix = chosen % n_side
    iy = (chosen // n_side) % n_side
    iz = chosen // (n_side * n_side)
    spacing = box / n_side
    site = np.stack([ix, iy, iz], axis=1).astype(np.float64) + 0.5
    site += rng.uniform(-jitter, jitter, size=(n, 3))
    return site * spacing


def suspension(n: int, axes, phi: float, seed: int, dt: float = 1e-3,
               dynamics: int = INERTIAL, velocities: bool = True,
               shape_fn=None, name: str = "suspension") -> dict:
    """Periodic cube of `n` ellipsoids at volume fraction `phi` on a jittered lattice."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n_side = int(math.ceil(round(n ** (1.0 / 3.0), 9)))
    while n_side ** 3 < n:
        n_side += 1
    # shape parameters are drawn after positions and orientations, but the box
    # size depends on the mean body volume; for shape laws we use the law's
    # expected volume (documented in DESIGN.md).
    if shape_fn is None:
        ax = np.asarray(axes, dtype=np.float64)
        vol_mean = 4.0 / 3.0 * math.pi * float(np.prod(ax))
    else:
        vol_mean = shape_fn(None)  # expected body volume of the shape law
    box_len = (n * vol_mean / phi) ** (1.0 / 3.0)
    pos = _jittered_lattice(rng, n, n_side, box_len)
    quat = _uniform_quaternions(rng, n)
    if shape_fn is None:
        axes_arr = np.tile(np.asarray(axes, dtype=np.float64), (n, 1))
    else:
        axes_arr = shape_fn(rng, n)
    if velocities:
        vel = rng.standard_normal((n, 6))
    else:
        vel = np.zeros((n, 6))
    inv_mass, inv_inertia = _ellipsoid_mass_props(axes_arr)
    return dict(
        name=name, n=n, pos=pos, quat=quat, axes=axes_arr, vel=vel,
        inv_mass=inv_mass, inv_inertia=inv_inertia,
        kinematic=np.zeros(n, dtype=np.int32),
        box=np.array([box_len] * 3), dt=float(dt), dynamics=int(dynamics),
        xi=1.0, cutoff=0.1, eps_ncp=1e-5, lcp_tol=1e-8, seed=seed, phi=phi,
    )


def _cfg2_shape(rng, n=None):
    """a = 1, b = c = 1/r, r ~ U(1, 4).  Called with rng=None it returns the
    expected volume E[4/3 pi / r^2] = 4/3 pi * (1/(4-1)) * (1 - 1/4) = pi/3."""
    if rng is None:
        return 4.0 / 3.0 * math.pi * (1.0 / 3.0) * (1.0 - 0.25)
    r = rng.uniform(1.0, 4.0, size=n)
    return np.stack([np.ones(n), 1.0 / r, 1.0 / r], axis=1)


def cfg1(seed: int = 1) -> dict:
    return suspension(512, (1.0, 0.5, 0.5), 0.30, seed, dt=1e-3,
                      dynamics=INERTIAL, name="cfg1")


def cfg2(seed: int = 2, n: int = 20000) -> dict:
    return suspension(n, None, 0.40, seed, dt=1e-2, dynamics=OVERDAMPED,
                      velocities=False, shape_fn=_cfg2_shape, name="cfg2")


def cfg5(seed: int = 5, n: int = 2_000_000) -> dict:
    return suspension(n, (1.0, 0.6, 0.4), 0.55, seed, dt=1e-3,
                      dynamics=INERTIAL, name="cfg5" if n == 2_000_000 else f"cfg5-n{n}")


def random_constraint_network(n_bodies: int, n_con: int, seed: int,
                              dynamics: int = INERTIAL):
    """Random Jacobian data for operator-level tests: body pairs (a<b),
    unit normals, lever arms |r| <= 1.2.  Returns bodies dict + (ia, ib, n,
    ra, rb).  Lever arms are raw inputs; each implementation forms its own
    rows t = r x n."""
    rng = np.random.Generator(np.random.PCG64(seed))
    b = suspension(n_bodies, (1.0, 0.6, 0.4), 0.3, seed + 1000,
                   dynamics=dynamics)
    ia = rng.integers(0, n_bodies, size=n_con)
    ib = rng.integers(0, n_bodies, size=n_con)
    same = ia == ib
    ib[same] = (ib[same] + 1) % n_bodies
    lo, hi = np.minimum(ia, ib), np.maximum(ia, ib)
    order = np.lexsort((hi, lo))
    ia, ib = lo[order].astype(np.int32), hi[order].astype(np.int32)
    nrm = rng.standard_normal((n_con, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    ra = rng.uniform(-0.7, 0.7, size=(n_con, 3))
    rb = rng.uniform(-0.7, 0.7, size=(n_con, 3))
    return b, ia, ib, nrm, ra, rb
