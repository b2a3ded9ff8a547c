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


def cfg1_relaxed(dt: float = 1e-3, vel_seed: int = 11) -> dict:
    """the cfg1 bodies at the overlap-free state in
    tests/golden/cfg1_relaxed.txt (written by tools/make_relaxed.py, which runs
    the ORACLE's overdamped relaxation), with fresh u, w ~ N(0, 1) drawn from
    PCG64(vel_seed); inertial, time step `dt` (1e-3 = cfg1; 0.1 = cfg1-bigdt).
    This function only reads the stored state and draws velocities."""
    import os
    sc = cfg1()
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                        "cfg1_relaxed.txt")
    st = np.loadtxt(path, comments="#")
    sc.update(pos=st[:, :3].copy(), quat=st[:, 3:7].copy(), dt=float(dt), name=f"cfg1-relaxed-dt{dt:g}",
              vel=np.random.Generator(np.random.PCG64(vel_seed)).standard_normal((sc["n"], 6)))
    return sc


def cfg2(seed: int = 2, n: int = 20000) -> dict:
    return suspension(n, None, 0.40, seed, dt=1e-2, dynamics=OVERDAMPED,
                      velocities=False, shape_fn=_cfg2_shape, name="cfg2")


def cfg5(seed: int = 5, n: int = 2_000_000) -> dict:
    return suspension(n, (1.0, 0.6, 0.4), 0.55, seed, dt=1e-3,
                      dynamics=INERTIAL, name="cfg5" if n == 2_000_000 else f"cfg5-n{n}")


def with_state(sc: dict, pos, quat, vel_seed: int, name: str) -> dict:
    """A "-relaxed" companion: the scene's bodies at a given
    (relaxed) configuration with fresh u, w ~ N(0, 1) from PCG64(vel_seed).
    Draws only; the configuration comes from the caller (the cfg5-relaxed
    state is relaxed by the library itself, bench.py / drivers.relax)."""
    out = dict(sc)
    out.update(pos=np.ascontiguousarray(pos, dtype=np.float64), quat=np.ascontiguousarray(quat, dtype=np.float64),
               vel=np.random.Generator(np.random.PCG64(vel_seed)).standard_normal((sc["n"], 6)), name=name)
    return out


def colony_rods(seed: int = 7, n: int = 131_072, dt: float = 1e-2, patch: int = 6) -> dict:
    """The paper's colony shape class: spherocylinders
    of diameter b = 0.5 and (tip-to-tip) length l ~ U(2, 4) (between l_0 and
    the division length 2 l_0), planar, packed with the cfg3 row-patch
    construction, every cell grown by l <- l e^dt (l_dot = l) at the start of
    the step; 2^17 cells by default.  Overdamped local drag with L = l (R22).
    Division: drivers.colony / divide_rods (R28)."""
    return cfg3(seed=seed, n=n, patch=patch, rods=True, dt=dt)


def cfg3(seed: int = 3, n: int = 200_000, patch: int = 6, gap: float = 0.005, minor: float = 0.25,
         growth: float = 0.01, dt: float = 1e-2, rods: bool = False) -> dict:
    """Growing-colony-like monolayer (BASELINE cfg3, SURVEY §8(d) row-patch
    construction): ellipsoids (a, 0.25, 0.25), a ~ U(0.5, 1.0), centres in
    z = 0, symmetry axis in-plane.  P x P square patches, each with a director
    theta_p ~ U(0, pi); inside a patch the bodies sit in rows along theta_p at
    row spacing 2*minor + gap, tip to tip with gap `gap` (aligned bodies in
    such rows are disjoint).  A body whose bounding circle (radius a) meets
    the bounding circle of an already accepted body of another patch is
    dropped (greedy, lattice order), so patches never overlap either.  The
    construction runs in a disk sized for `n` bodies; the n bodies nearest
    the centre are kept (ties by index).  Growth: a seeded half of the bodies
    gets a += `growth` (the start-of-step axial growth), which creates the
    small tip overlaps the step resolves.  Overdamped local drag (xi = 1),
    dt = 1e-2, no external force, non-periodic.  Draw order: a per site, patch
    directors, row offsets, growth set."""
    rng = np.random.Generator(np.random.PCG64(seed))
    # tip half-length law: ellipsoid a ~ U(0.5, 1); rod (l + b)/2 with l ~ U(2, 4)
    a_lo, a_hi = (0.5, 1.0) if not rods else (1.0, 2.0)  # rods: half the tip-to-tip length l ~ U(2, 4)
    # disk radius from the realised packing (~0.55 area fraction)
    area_body = math.pi * 0.5 * (a_lo + a_hi) * minor
    fill, rim = (0.55, 4.0) if not rods else (0.40, 3.0 * a_hi)  # long rods lose more at patch borders
    radius = math.sqrt(n * area_body / fill / math.pi) + rim
    side = 2.0 * radius
    psz = side / patch
    theta = rng.uniform(0.0, math.pi, size=(patch, patch))
    pts, angs, majors, owner = [], [], [], []
    for py in range(patch):
        for px in range(patch):
            th = theta[py, px]
            u = np.array([math.cos(th), math.sin(th)])
            v = np.array([-math.sin(th), math.cos(th)])
            cx, cy = -radius + (px + 0.5) * psz, -radius + (py + 0.5) * psz
            half = 0.75 * psz  # rows cover the rotated square patch
            rows = np.arange(-half, half, 2 * minor + gap)
            for rv in rows:
                t = -half + rng.uniform(0.0, 1.0)
                while t < half:
                    a = rng.uniform(a_lo, a_hi)
                    c = np.array([cx, cy]) + (t + a) * u + rv * v
                    t += 2 * a + gap
                    if abs(c[0] - cx) > psz / 2 or abs(c[1] - cy) > psz / 2:
                        continue
                    if c[0] ** 2 + c[1] ** 2 > radius ** 2:
                        continue
                    pts.append(c)
                    angs.append(th)
                    majors.append(a)
                    owner.append(py * patch + px)
    pts = np.array(pts)
    angs = np.array(angs)
    majors = np.array(majors)
    owner = np.array(owner)
    # greedy cross-patch rejection with bounding circles (grid hashing)
    keep = np.ones(len(pts), dtype=bool)
    cell = 2.0 * a_hi  # +-1 cells must reach the largest a_i + a_j
    grid = {}
    for i in range(len(pts)):
        gx, gy = int(math.floor(pts[i, 0] / cell)), int(math.floor(pts[i, 1] / cell))
        ok = True
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for j in grid.get((gx + dx, gy + dy), ()):
                    if owner[j] != owner[i]:
                        d = pts[i] - pts[j]
                        if d @ d < (majors[i] + majors[j]) ** 2:
                            ok = False
                            break
                if not ok:
                    break
            if not ok:
                break
        if ok:
            grid.setdefault((gx, gy), []).append(i)
        else:
            keep[i] = False
    pts, angs, majors = pts[keep], angs[keep], majors[keep]
    r2 = (pts ** 2).sum(1)
    order = np.lexsort((np.arange(len(r2)), r2))[:n]
    order = np.sort(order)  # keep construction (spatially coherent) order
    if len(order) < n:
        raise ValueError(f"cfg3 construction produced {len(order)} < {n} bodies")
    pts, angs, majors = pts[order], angs[order], majors[order]
    grow = np.zeros(n, dtype=bool)
    grow[rng.permutation(n)[: n // 2]] = True
    pos = np.zeros((n, 3))
    pos[:, :2] = pts
    quat = np.zeros((n, 4))
    quat[:, 0] = np.cos(angs / 2)
    quat[:, 3] = np.sin(angs / 2)
    if rods:
        # spherocylinder: tip-to-tip length l = 2 a, grown l <- l e^dt (R22);
        # axes = (centreline / 2, r, r) with centreline = l - 2 r
        ell = 2.0 * majors * math.exp(dt) - 2.0 * minor
        axes = np.stack([0.5 * ell, np.full(n, minor), np.full(n, minor)], axis=1)
        shape = np.ones(n, dtype=np.int32)
        grow[:] = True
        area = (ell * 2 * minor + math.pi * minor ** 2).sum()
    else:
        majors = majors + growth * grow
        axes = np.stack([majors, np.full(n, minor), np.full(n, minor)], axis=1)
        shape = np.zeros(n, dtype=np.int32)
        area = math.pi * (axes[:, 0] * axes[:, 1]).sum()
    inv_mass, inv_inertia = _ellipsoid_mass_props(axes)  # unused: overdamped dynamics
    name = ("rods" if rods else "cfg3") + ("" if n == (131_072 if rods else 200_000) else f"-n{n}")
    return dict(name=name, n=n, pos=pos, quat=quat, axes=axes, shape=shape,
                vel=np.zeros((n, 6)), inv_mass=inv_mass, inv_inertia=inv_inertia,
                kinematic=np.zeros(n, dtype=np.int32), box=np.zeros(3), dt=float(dt), dynamics=OVERDAMPED,
                xi=1.0, cutoff=0.1, eps_ncp=1e-5, lcp_tol=1e-8, seed=seed, growing=grow,
                area_fraction=float(area / (math.pi * (pts ** 2).sum(1).max())))


def cfg4(seed: int = 4, n_side: int = 1000, R: float = 1.0, r: float = 0.2, pitch: float = 1.4,
         c_max: int = 3, c_fixed: int | None = None, dt: float = 1e-3) -> dict:
    """Taut chainmail-like constraint network (BASELINE cfg4):
    n_side x n_side rings (torus R = 1, r = 0.2, rho = 1) on a square lattice
    of pitch 1.4 R in the x-y plane, ring axes alternating x / y in a
    checkerboard.  Every lattice link (a < b) gets c ~ U{1..c_max} (or
    c_fixed) unilateral constraints with raw geometry drawn here:
    normal n = normalize(-e_link + 0.25 g), g ~ N(0, I3) (n opposes
    separation), lever arms r_a = R e_link + rho_a, r_b = -R e_link + rho_b,
    rho uniform in a ball of radius 0.2, gap Phi_0 = 0 (taut).  Rows 0 and
    n_side-1 (y index) are kinematic with velocity -1 / +1 along y; interior
    bodies start with the affine field u_y = -1 + 2 i / (n_side - 1).
    Inertial, dt = 1e-3.  Torus inertia: m = rho 2 pi^2 R r^2,
    I_axis = m (R^2 + 3/4 r^2), I_diam = m (R^2 / 2 + 5/8 r^2), body z =
    ring axis.  Rows are returned sorted by (ia, ib).  Draw order: counts,
    then per row g, rho_a, rho_b."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n = n_side * n_side
    ii, jj = np.divmod(np.arange(n), n_side)  # body = i * n_side + j ; y index i, x index j
    pos = np.stack([jj * pitch * R, ii * pitch * R, np.zeros(n)], axis=1)
    quat = np.zeros((n, 4))
    ax_x = (ii + jj) % 2 == 0
    s = math.sqrt(0.5)
    quat[ax_x] = [s, 0.0, s, 0.0]    # body z -> world x (rotation +90 deg about y)
    quat[~ax_x] = [s, -s, 0.0, 0.0]  # body z -> world y (rotation -90 deg about x)
    m = 2.0 * math.pi ** 2 * R * r * r
    I_axis = m * (R * R + 0.75 * r * r)
    I_diam = m * (0.5 * R * R + 0.625 * r * r)
    inv_mass = np.full(n, 1.0 / m)
    inv_inertia = np.tile([1.0 / I_diam, 1.0 / I_diam, 1.0 / I_axis], (n, 1))
    kin = ((ii == 0) | (ii == n_side - 1)).astype(np.int32)
    vel = np.zeros((n, 6))
    vel[:, 1] = -1.0 + 2.0 * ii / (n_side - 1)
    # links: horizontal (i, j)-(i, j+1), vertical (i, j)-(i+1, j)
    b = np.arange(n).reshape(n_side, n_side)
    la = np.concatenate([b[:, :-1].ravel(), b[:-1, :].ravel()])
    lb = np.concatenate([b[:, 1:].ravel(), b[1:, :].ravel()])
    e = np.concatenate([np.tile([1.0, 0.0, 0.0], (n_side * (n_side - 1), 1)),
                        np.tile([0.0, 1.0, 0.0], (n_side * (n_side - 1), 1))])
    cnt = (np.full(len(la), c_fixed) if c_fixed else rng.integers(1, c_max + 1, size=len(la)))
    ia = np.repeat(la, cnt)
    ib = np.repeat(lb, cnt)
    el = np.repeat(e, cnt, axis=0)
    m_rows = len(ia)
    g = rng.standard_normal((m_rows, 3))
    nrm = -el + 0.25 * g
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)

    def ball(k):
        v = rng.standard_normal((k, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        return v * (0.2 * rng.uniform(0.0, 1.0, size=(k, 1)) ** (1.0 / 3.0))

    ra = R * el + ball(m_rows)
    rb = -R * el + ball(m_rows)
    order = np.lexsort((ib, ia))  # stable: rows of one link keep draw order
    net = dict(ia=ia[order].astype(np.int32), ib=ib[order].astype(np.int32), n=nrm[order], ra=ra[order],
               rb=rb[order], phi=np.zeros(m_rows))
    return dict(name="cfg4" if n_side == 1000 else f"cfg4-{n_side}", n=n, pos=pos, quat=quat,
                axes=np.tile([R + r, R + r, r], (n, 1)), vel=vel, inv_mass=inv_mass, inv_inertia=inv_inertia,
                kinematic=kin, box=np.zeros(3), dt=float(dt), dynamics=INERTIAL, xi=1.0, cutoff=0.1,
                eps_ncp=1e-5, lcp_tol=1e-8, seed=seed, network=net)


def chain_tori(n: int = 200, seed: int = 8, R: float = 1.0, r: float = 0.2, pitch: float = 1.58,
               jitter: float = 0.02, dt: float = 1e-2, pull: float = 3.0) -> dict:
    """Linked chain of tori (the paper's chainmail rings, as a
    1-D chain): ring k at x = k * pitch with ring axis z (even k) or y (odd
    k), so every ring passes through its neighbours' disks.  At pitch 1.58 the
    centreline circles of neighbours are 0.42 apart (Phi = 0.42 - 2 r = 0.02:
    near contact).  Seeded jitter (positions U(+-jitter), small rotations),
    end rings kinematic with velocity -pull / +pull along x, interior velocity
    the affine pull field plus N(0, 1) (u and omega), torus inertia (SURVEY
    G9), inertial, dt = 1e-2."""
    rng = np.random.Generator(np.random.PCG64(seed))
    pos = np.zeros((n, 3))
    pos[:, 0] = np.arange(n) * pitch
    pos += rng.uniform(-jitter, jitter, size=(n, 3))
    s2 = math.sqrt(0.5)
    quat = np.zeros((n, 4))
    quat[0::2] = [1.0, 0.0, 0.0, 0.0]
    quat[1::2] = [s2, -s2, 0.0, 0.0]  # body z -> world y
    tilt = rng.normal(scale=jitter, size=(n, 3))  # small rotation vectors
    ang = np.linalg.norm(tilt, axis=1, keepdims=True)
    dq = np.concatenate([np.cos(ang / 2), np.sin(ang / 2) * tilt / np.maximum(ang, 1e-300)], axis=1)
    # quaternion product dq (x) quat
    w1, v1 = dq[:, :1], dq[:, 1:]
    w2, v2 = quat[:, :1], quat[:, 1:]
    quat = np.concatenate([w1 * w2 - (v1 * v2).sum(1, keepdims=True), w1 * v2 + w2 * v1 + np.cross(v1, v2)], axis=1)
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    m = 2.0 * math.pi ** 2 * R * r * r
    I_axis = m * (R * R + 0.75 * r * r)
    I_diam = m * (0.5 * R * R + 0.625 * r * r)
    kin = np.zeros(n, dtype=np.int32)
    kin[0] = kin[-1] = 1
    vel = rng.standard_normal((n, 6))
    vel[:, 0] += pull * (-1.0 + 2.0 * np.arange(n) / (n - 1))
    vel[0] = [-pull, 0, 0, 0, 0, 0]
    vel[-1] = [pull, 0, 0, 0, 0, 0]
    return dict(name=f"chain{n}", n=n, pos=pos, quat=quat, axes=np.tile([R, r, r], (n, 1)),
                shape=np.full(n, 2, dtype=np.int32), vel=vel, inv_mass=np.full(n, 1.0 / m),
                inv_inertia=np.tile([1.0 / I_diam, 1.0 / I_diam, 1.0 / I_axis], (n, 1)), kinematic=kin,
                box=np.zeros(3), dt=float(dt), dynamics=INERTIAL, xi=1.0, cutoff=0.1, eps_ncp=1e-5,
                lcp_tol=1e-8, seed=seed)


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


def local_constraint_network(n_bodies: int, n_con: int, seed: int, dynamics: int = INERTIAL):
    """Spatially local random Jacobian data at a given size (timing inputs for
    the CPU oracle at cfg5's N and N_C, bench.py cpu_baseline): the cfg5
    suspension's bodies (jittered lattice, phi = 0.55, kept in lattice order)
    and rows between a body and a lattice neighbour (index offset 1, n_side or
    n_side^2, as contacts of the lattice-ordered cfg5 bodies are), unit
    normals, lever arms |r_i| <= 0.7.  Returns bodies dict + (ia, ib, n, ra, rb)
    sorted by (ia, ib)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    b = suspension(n_bodies, (1.0, 0.6, 0.4), 0.55, seed + 1000, dynamics=dynamics)
    n_side = int(math.ceil(round(n_bodies ** (1.0 / 3.0), 9)))
    a = rng.integers(0, n_bodies, size=n_con)
    off = np.array([1, n_side, n_side * n_side])[rng.integers(0, 3, size=n_con)]
    c = (a + off) % n_bodies
    lo, hi = np.minimum(a, c), np.maximum(a, c)
    order = np.lexsort((hi, lo))
    ia, ib = lo[order].astype(np.int32), hi[order].astype(np.int32)
    nrm = rng.standard_normal((n_con, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    ra = rng.uniform(-0.7, 0.7, size=(n_con, 3))
    rb = rng.uniform(-0.7, 0.7, size=(n_con, 3))
    return b, ia, ib, nrm, ra, rb


def relabelled(sc: dict, seed: int) -> dict:
    """The same scene with its bodies relabelled by a seeded random permutation
    (every per-body array permuted alike): the same physical problem, but body
    indices no longer follow space (DESIGN.md §5 "Body order").  Relabelling
    only; no per-body value changes."""
    n = sc["n"]
    perm = np.random.Generator(np.random.PCG64(seed)).permutation(n)
    out = dict(sc)
    for k, v in sc.items():
        if isinstance(v, np.ndarray) and v.ndim >= 1 and v.shape[0] == n and k != "box":
            out[k] = np.ascontiguousarray(v[perm])
    out["name"] = f"{sc['name']}-relabelled{seed}"
    out["relabel"] = perm
    return out
