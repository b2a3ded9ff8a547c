// Geometry kernels: ellipsoid shape matrices, cell-list broadphase (K1/K2)
// and the batched shared-normal signed distance (K3/K10).
//
// SNSD ("the points that minimize their shared-normal signed
// separation distance"; W-W formulation cited at P:L944, not given; reading
// R4): for ellipsoids with Sigma = R diag(e^2) R^T and support function
// h(n) = sqrt(n^T Sigma n),
//     Phi = max_{|n|=1} F(n),  F(n) = n.d - h_a(n) - h_b(n),  d = x_b - x_a,
//     y_a = x_a + Sigma_a n / h_a,  y_b = x_b - Sigma_b n / h_b.
// At a stationary point y_b - y_a = Phi n.
//
// GPU strategy (differs from the oracle's fixed multistart), three kernels
// over compacted work lists so that every stage runs with full warps:
//   stage 0  every pair: F is concave and positively homogeneous on R^3, so
//            Phi >= F(d/|d|); a pair whose bound already clears the threshold
//            is final (status BOUND, phi = the bound); rods and tori are
//            solved here in full; the rest is listed (one atomic per warp).
//   stage 1  listed pairs: damped Riemannian Newton from d/|d|; a maximum with
//            F > 0 is the global one (concavity); F <= 0 (overlap or touching)
//            goes to the stage-2 list with the Newton result as incumbent.
//   stage 2  listed pairs: sample the `n_dirs` Fibonacci directions (table
//            built once per context, k_dirs), Newton from the best four, keep
//            the largest maximum (ties: larger n.d/|d|, then lexicographically
//            smaller n; R4).
#include "common.cuh"
#include "reduce.cuh"

// ------------------------------------------------------------ shape matrices
// Per-body geometry slot Sig (nb, 6), q normalised:
//   ellipsoid      (xx, xy, xz, yy, yz, zz) of R diag(e^2) R^T
//   spherocylinder (u_x, u_y, u_z, h, r, 0): centreline direction u = R e_x,
//                  half-length h = axes[0], cap radius r = axes[1]
__global__ void k_shape(int64_t nb, const double *__restrict__ quat, const double *__restrict__ axes,
                        const int32_t *__restrict__ shape, double *__restrict__ Sig) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        double s = quat[4 * b], x = quat[4 * b + 1], y = quat[4 * b + 2], z = quat[4 * b + 3];
        double inv = 1.0 / sqrt(s * s + x * x + y * y + z * z);
        s *= inv; x *= inv; y *= inv; z *= inv;
        const double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - s * z), 2 * (x * z + s * y)},
                                {2 * (x * y + s * z), 1 - 2 * (x * x + z * z), 2 * (y * z - s * x)},
                                {2 * (x * z - s * y), 2 * (y * z + s * x), 1 - 2 * (x * x + y * y)}};
        double *o = Sig + 6 * b;
        if (shape && shape[b] == RELCP_SHAPE_SPHEROCYLINDER) {
            o[0] = R[0][0]; o[1] = R[1][0]; o[2] = R[2][0];
            o[3] = axes[3 * b]; o[4] = axes[3 * b + 1]; o[5] = 0.0;
            continue;
        }
        if (shape && shape[b] == RELCP_SHAPE_TORUS) {
            // ring frame: e1 = R e_x (slots 0-2) and the ring axis e3 = R e_z
            // (slots 3-5); e2 = e3 x e1; radii (R, r) are read from axes
            o[0] = R[0][0]; o[1] = R[1][0]; o[2] = R[2][0];
            o[3] = R[0][2]; o[4] = R[1][2]; o[5] = R[2][2];
            continue;
        }
        const double e0 = axes[3 * b] * axes[3 * b], e1 = axes[3 * b + 1] * axes[3 * b + 1],
                     e2 = axes[3 * b + 2] * axes[3 * b + 2];
        auto S = [&](int i, int j) { return R[i][0] * e0 * R[j][0] + R[i][1] * e1 * R[j][1] + R[i][2] * e2 * R[j][2]; };
        o[0] = S(0, 0); o[1] = S(0, 1); o[2] = S(0, 2);
        o[3] = S(1, 1); o[4] = S(1, 2); o[5] = S(2, 2);
    }
}

int geo_shape_matrices(relcp_ctx *ctx, int64_t nb, const double *quat, const double *axes, const int32_t *shape,
                       double *Sig) {
    k_shape<<<grid_for(nb), RELCP_NT, 0, ctx->stream>>>(nb, quat, axes, shape, Sig);
    CKL();
    return RELCP_OK;
}

// Spherocylinder pair: closest points of the two centreline segments
// (clamp-and-recompute solution of the convex quadratic
// |d + t u_b - s u_a|^2 on [-h_a, h_a] x [-h_b, h_b]), minus the cap radii.
// Parallel axes: midpoint of the overlap of the projections on u_a (R22).
__device__ int rod_pair(const double *d, const double *ga, const double *gb, double &phi, double *nout, double *ra,
                        double *rb) {
    const double ua[3] = {ga[0], ga[1], ga[2]}, ub[3] = {gb[0], gb[1], gb[2]};
    const double ha = ga[3], rra = ga[4], hb = gb[3], rrb = gb[4];
    const double c = ua[0] * ub[0] + ua[1] * ub[1] + ua[2] * ub[2];
    const double da = ua[0] * d[0] + ua[1] * d[1] + ua[2] * d[2];
    const double db = ub[0] * d[0] + ub[1] * d[1] + ub[2] * d[2];
    const double cx = ua[1] * ub[2] - ua[2] * ub[1], cy = ua[2] * ub[0] - ua[0] * ub[2],
                 cz = ua[0] * ub[1] - ua[1] * ub[0];
    const double cr2 = cx * cx + cy * cy + cz * cz;
    double s, t;
    if (sqrt(cr2) < 1e-12) {
        const double sg = c > 0.0 ? 1.0 : -1.0;
        const double lo = fmax(-ha, da - hb), hi = fmin(ha, da + hb);
        s = lo <= hi ? 0.5 * (lo + hi) : (da > 0.0 ? ha : -ha);
        t = sg * (fmin(fmax(s, da - hb), da + hb) - da);
    } else {
        s = fmin(fmax((da - c * db) / cr2, -ha), ha);
        t = c * s - db;
        if (t < -hb || t > hb) {
            t = fmin(fmax(t, -hb), hb);
            s = fmin(fmax(da + c * t, -ha), ha);
        }
    }
    double v[3];
    for (int k = 0; k < 3; ++k) v[k] = d[k] + t * ub[k] - s * ua[k];
    const double dist = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    if (!(dist >= 1e-12)) {
        phi = nan("");
        for (int k = 0; k < 3; ++k) nout[k] = ra[k] = rb[k] = nan("");
        return 1;  // intersecting centrelines: no normal
    }
    phi = dist - rra - rrb;
    for (int k = 0; k < 3; ++k) {
        const double nk = v[k] / dist;
        nout[k] = nk;
        ra[k] = s * ua[k] + rra * nk;
        rb[k] = t * ub[k] - rrb * nk;
    }
    return 0;
}

// ------------------------------------------------------------ SNSD device code
struct Sym {
    double xx, xy, xz, yy, yz, zz;
};
__device__ __forceinline__ Sym load_sym(const double *__restrict__ p) {
    Sym s;
    s.xx = p[0]; s.xy = p[1]; s.xz = p[2]; s.yy = p[3]; s.yz = p[4]; s.zz = p[5];
    return s;
}
__device__ __forceinline__ void smv(const Sym &S, const double *v, double *o) {
    o[0] = S.xx * v[0] + S.xy * v[1] + S.xz * v[2];
    o[1] = S.xy * v[0] + S.yy * v[1] + S.yz * v[2];
    o[2] = S.xz * v[0] + S.yz * v[1] + S.zz * v[2];
}
__device__ __forceinline__ double d3(const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

struct Eval {
    double f, ha, hb;
    double Sa_n[3], Sb_n[3], v[3];  // v = d - Sa n/ha - Sb n/hb (= y_b - y_a)
};

__device__ __forceinline__ void feval(const double *n, const double *d, const Sym &Sa, const Sym &Sb, Eval &E) {
    smv(Sa, n, E.Sa_n);
    smv(Sb, n, E.Sb_n);
    E.ha = sqrt(d3(n, E.Sa_n));
    E.hb = sqrt(d3(n, E.Sb_n));
    E.f = d3(n, d) - E.ha - E.hb;
    const double ia = 1.0 / E.ha, ib = 1.0 / E.hb;
#pragma unroll
    for (int k = 0; k < 3; ++k) E.v[k] = d[k] - E.Sa_n[k] * ia - E.Sb_n[k] * ib;
}

__device__ __forceinline__ double fval(const double *n, const double *d, const Sym &Sa, const Sym &Sb) {
    double t[3];
    smv(Sa, n, t);
    double ha = sqrt(d3(n, t));
    smv(Sb, n, t);
    double hb = sqrt(d3(n, t));
    return d3(n, d) - ha - hb;
}

// t^T (S/h - (S n)(S n)^T / h^3) u  for the support-function Hessian
__device__ __forceinline__ double hess_form(const Sym &S, const double *Sn, double h, const double *t, const double *u) {
    double Su[3];
    smv(S, u, Su);
    return d3(t, Su) / h - d3(t, Sn) * d3(u, Sn) / (h * h * h);
}

// Damped Riemannian Newton ascent of F on the unit sphere from n (in/out).
// Returns 1 if certified (gradient or step at the rounding floor).
__device__ int newton_sphere(double *n, const double *d, double dnorm, const Sym &Sa, const Sym &Sb, Eval &E) {
    const double gtol = 1e-13 * fmax(1.0, dnorm);
    feval(n, d, Sa, Sb, E);
    for (int it = 0; it < 64; ++it) {
        // tangent frame: t1 from the coordinate axis least aligned with n
        const double ax = fabs(n[0]), ay = fabs(n[1]), az = fabs(n[2]);
        double e[3] = {0.0, 0.0, 0.0};
        if (ax <= ay && ax <= az) e[0] = 1.0; else if (ay <= az) e[1] = 1.0; else e[2] = 1.0;
        const double ne = d3(n, e);
        double t1[3] = {e[0] - ne * n[0], e[1] - ne * n[1], e[2] - ne * n[2]};
        const double il = 1.0 / sqrt(d3(t1, t1));
        t1[0] *= il; t1[1] *= il; t1[2] *= il;
        const double t2[3] = {n[1] * t1[2] - n[2] * t1[1], n[2] * t1[0] - n[0] * t1[2], n[0] * t1[1] - n[1] * t1[0]};
        const double g1 = d3(t1, E.v), g2 = d3(t2, E.v);
        if (sqrt(g1 * g1 + g2 * g2) <= gtol) return 1;
        const double nv = d3(n, E.v);
        // Riemannian Hessian in the (t1, t2) frame: P Hess(F) P - (n . grad F) I
        const double h11 = -hess_form(Sa, E.Sa_n, E.ha, t1, t1) - hess_form(Sb, E.Sb_n, E.hb, t1, t1) - nv;
        const double h22 = -hess_form(Sa, E.Sa_n, E.ha, t2, t2) - hess_form(Sb, E.Sb_n, E.hb, t2, t2) - nv;
        const double h12 = -0.5 * (hess_form(Sa, E.Sa_n, E.ha, t1, t2) + hess_form(Sa, E.Sa_n, E.ha, t2, t1)) -
                           0.5 * (hess_form(Sb, E.Sb_n, E.hb, t1, t2) + hess_form(Sb, E.Sb_n, E.hb, t2, t1));
        const double scale = fabs(h11) + fabs(h12) + fabs(h22) + 1e-300;
        const double lmax = 0.5 * (h11 + h22) + sqrt(0.25 * (h11 - h22) * (h11 - h22) + h12 * h12);
        double mu = lmax > -1e-8 * scale ? lmax + 1e-8 * scale + 1e-12 : 0.0;
        bool accepted = false;
        double step = 0.0;
        Eval En;
        double nn[3];
        for (int tr = 0; tr < 48; ++tr) {
            const double a = h11 - mu, c = h22 - mu;
            const double det = a * c - h12 * h12;
            double x1 = -(c * g1 - h12 * g2) / det;
            double x2 = -(a * g2 - h12 * g1) / det;
            double xl = sqrt(x1 * x1 + x2 * x2);
            if (xl > 0.5) {
                x1 *= 0.5 / xl;
                x2 *= 0.5 / xl;
                xl = 0.5;
            }
            nn[0] = n[0] + x1 * t1[0] + x2 * t2[0];
            nn[1] = n[1] + x1 * t1[1] + x2 * t2[1];
            nn[2] = n[2] + x1 * t1[2] + x2 * t2[2];
            const double inn = 1.0 / sqrt(d3(nn, nn));
            nn[0] *= inn; nn[1] *= inn; nn[2] *= inn;
            feval(nn, d, Sa, Sb, En);
            if (En.f >= E.f - 1e-15 * (1.0 + dnorm)) {
                accepted = true;
                step = xl;
                break;
            }
            mu = 4.0 * mu + scale + 1e-12;
        }
        if (!accepted) return 1;  // no ascent left at rounding level
        n[0] = nn[0]; n[1] = nn[1]; n[2] = nn[2];
        E = En;
        if (step < 1e-14) return 1;
    }
    return 0;
}

__device__ __forceinline__ bool better(double f, const double *n, double fb, const double *nb, const double *dh) {
    if (f > fb) return true;
    if (f < fb) return false;
    const double c1 = d3(n, dh), c0 = d3(nb, dh);
    if (c1 != c0) return c1 > c0;
    if (n[0] != nb[0]) return n[0] < nb[0];
    if (n[1] != nb[1]) return n[1] < nb[1];
    return n[2] < nb[2];
}

#ifndef SNSD_MINB
#define SNSD_MINB 4  // resident blocks per SM for the Newton / multistart stages: 128 registers (some spills)
                     // beats 146-168 at 1-2 blocks: SNSD 66 -> 56.5 ms per cfg5 step (same-box A/B)
#endif

// SNSD status codes (k_snsd_* outputs)
#define SNSD_OK 0
#define SNSD_DEGENERATE 1  // coincident centres (R4)
#define SNSD_NONCONV 2     // Newton not certified
#define SNSD_BOUND 3       // quick reject: Phi >= F(d/|d|) >= reject threshold (phi = that lower bound)
#define SNSD_MULTI 4       // internal: needs the multistart pass

__device__ __forceinline__ void write_out(const Eval &E, const double *nb, double &phi, double *nout, double *ra,
                                          double *rb) {
    phi = E.f;
    const double ia = 1.0 / E.ha, ib = 1.0 / E.hb;
    for (int k = 0; k < 3; ++k) {
        nout[k] = nb[k];
        ra[k] = E.Sa_n[k] * ia;
        rb[k] = -E.Sb_n[k] * ib;
    }
}

// Stage 1 of one pair.  F is concave and 1-homogeneous on R^3, so
// Phi >= F(d/|d|): if that bound is >= reject_above the pair cannot pass any
// threshold below it (generation: cutoff; check: 0 > -eps) -> SNSD_BOUND.
// Otherwise Newton from d/|d|; a maximum with F > 0 is global -> SNSD_OK /
// SNSD_NONCONV.  Overlap / touching (F <= 0): a certified critical point with
// F > -cert is the global maximum (curvature certificate, R29: F(n) =
// n.d - h_K(n) with K = A + B, whose radii of curvature are >= rho = r_min(A)
// + r_min(B); by Blaschke's rolling theorem a ball of radius rho rolls freely
// in K, so a critical point at depth |F| < rho is the unique nearest boundary
// point of d, i.e. F = -dist(d, dK) = Phi; cert = rho / 2) -> SNSD_OK.
// Otherwise SNSD_MULTI (outputs hold the Newton result as the incumbent for
// the stage-2 multistart).
__device__ int snsd_stage1(const double *d, const Sym &Sa, const Sym &Sb, double reject_above, double &phi,
                           double *nout, double *ra, double *rb, double cert = 0.0) {
    const double dn = sqrt(d3(d, d));
    if (!(dn >= 1e-12)) {
        phi = nan("");
        for (int k = 0; k < 3; ++k) nout[k] = ra[k] = rb[k] = nan("");
        return SNSD_DEGENERATE;
    }
    double nb[3] = {d[0] / dn, d[1] / dn, d[2] / dn};
    Eval Eb;
    feval(nb, d, Sa, Sb, Eb);
    if (Eb.f >= reject_above + 1e-12 * fmax(1.0, dn)) {
        write_out(Eb, nb, phi, nout, ra, rb);
        return SNSD_BOUND;
    }
    const int ok = newton_sphere(nb, d, dn, Sa, Sb, Eb);
    feval(nb, d, Sa, Sb, Eb);
    write_out(Eb, nb, phi, nout, ra, rb);
    if (Eb.f > 0.0) return ok ? SNSD_OK : SNSD_NONCONV;
    if (ok && Eb.f > -cert) return SNSD_OK;  // shallow overlap: the curvature certificate
    return ok ? SNSD_MULTI : -SNSD_MULTI;  // sign carries the incumbent's certification
}

// The n_dirs-point Fibonacci sphere of the stage-2 multistart, (3, n_dirs)
// planes: m_i = (r cos(g i), r sin(g i), z), z = 1 - (2i + 1)/n, r = sqrt(1 - z^2),
// g = pi (3 - sqrt 5).  Shared by every pair, so tabulated once per context.
__global__ void k_dirs(int n_dirs, double *__restrict__ dirs, float *__restrict__ dirs32) {
    const double ga = 3.14159265358979323846 * (3.0 - sqrt(5.0));
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_dirs; i += gridDim.x * blockDim.x) {
        const double z = 1.0 - (2.0 * i + 1.0) / n_dirs;
        const double r = sqrt(fmax(0.0, 1.0 - z * z));
        double sn, cs;
        sincos(ga * i, &sn, &cs);
        dirs[i] = r * cs;
        dirs[n_dirs + i] = r * sn;
        dirs[2 * n_dirs + i] = z;
        dirs32[i] = (float)(r * cs);
        dirs32[n_dirs + i] = (float)(r * sn);
        dirs32[2 * n_dirs + i] = (float)z;
    }
}

// fp32 value of F at a sample direction: the stage-2 screening only RANKS the
// samples to pick the Newton starts (refined in fp64 from the fp64 table), so
// single precision is enough there and runs on the fp32 pipe / MUFU
struct Sym32 {
    float xx, xy, xz, yy, yz, zz;
};
__device__ __forceinline__ Sym32 sym32(const Sym &S) {
    return Sym32{(float)S.xx, (float)S.xy, (float)S.xz, (float)S.yy, (float)S.yz, (float)S.zz};
}
__device__ __forceinline__ float fval32(const float *n, const float *d, const Sym32 &A, const Sym32 &B) {
    const float ta0 = A.xx * n[0] + A.xy * n[1] + A.xz * n[2], ta1 = A.xy * n[0] + A.yy * n[1] + A.yz * n[2],
                ta2 = A.xz * n[0] + A.yz * n[1] + A.zz * n[2];
    const float tb0 = B.xx * n[0] + B.xy * n[1] + B.xz * n[2], tb1 = B.xy * n[0] + B.yy * n[1] + B.yz * n[2],
                tb2 = B.xz * n[0] + B.yz * n[1] + B.zz * n[2];
    return n[0] * d[0] + n[1] * d[1] + n[2] * d[2] - sqrtf(n[0] * ta0 + n[1] * ta1 + n[2] * ta2) -
           sqrtf(n[0] * tb0 + n[1] * tb1 + n[2] * tb2);
}

// Stage 2 (overlap / touching): multistart from `n_dirs`-sample directions in
// distinct basins (angular non-maximum suppression, cos > SNSD_SEP_COS = same
// basin) against the incumbent (nb, status st_best) from stage 1.
#ifndef SNSD_SEP_COS
#define SNSD_SEP_COS 0.9  // ~26 deg
#endif
__device__ int snsd_stage2(const double *d, const Sym &Sa, const Sym &Sb, int n_dirs,
                           const double *__restrict__ dirs, const float *__restrict__ dirs32, double *nb,
                           int st_best, double &phi, double *nout, double *ra, double *rb) {
    const double dn = sqrt(d3(d, d));
    const double dh[3] = {d[0] / dn, d[1] / dn, d[2] / dn};
    Eval Eb;
    feval(nb, d, Sa, Sb, Eb);
    double fb = Eb.f;
    {
        // overlap / touching: Newton from up to K sampled directions that lie
        // in DIFFERENT basins.  One pass over the sample keeps K leaders with
        // online non-maximum suppression: a direction within SNSD_SEP_COS of a
        // leader replaces that leader if its value is larger and is dropped
        // otherwise; a direction near no leader enters if it beats the worst.
        // (Leaders hold sample indices; their directions are re-read from the
        // table, which stays in L1.)  Ties keep the earlier sample.
        constexpr int K = 4;
        float topf[K];
        int topi[K];
#pragma unroll
        for (int k = 0; k < K; ++k) { topf[k] = -INFINITY; topi[k] = -1; }
        const float d32[3] = {(float)d[0], (float)d[1], (float)d[2]};
        const Sym32 A32 = sym32(Sa), B32 = sym32(Sb);
        for (int i = 0; i < n_dirs; ++i) {
            // warp-uniform address: one broadcast load per plane
            const float m[3] = {__ldg(dirs32 + i), __ldg(dirs32 + n_dirs + i), __ldg(dirs32 + 2 * n_dirs + i)};
            const float f = fval32(m, d32, A32, B32);
            if (!(f > topf[K - 1]) && topi[K - 1] >= 0) {
                // cannot enter; it may still only replace a nearby leader, which
                // needs f > that leader's value >= the worst: nothing to do
                continue;
            }
            int near = -1;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (near < 0 && topi[k] >= 0) {
                    const int j = topi[k];
                    const float c = m[0] * __ldg(dirs32 + j) + m[1] * __ldg(dirs32 + n_dirs + j) +
                                    m[2] * __ldg(dirs32 + 2 * n_dirs + j);
                    if (c > (float)SNSD_SEP_COS) near = k;
                }
            }
            int p;
            if (near >= 0) {
                if (!(f > topf[near])) continue;
                p = near;  // replace the nearby leader, then restore the order
            } else {
                p = K - 1;  // evict the worst
            }
            while (p > 0 && topf[p - 1] < f) {
                topf[p] = topf[p - 1];
                topi[p] = topi[p - 1];
                --p;
            }
            topf[p] = f;
            topi[p] = i;
        }
        for (int k = 0; k < K; ++k) {
            if (topi[k] < 0) continue;
            const int i = topi[k];
            double m[3] = {dirs[i], dirs[n_dirs + i], dirs[2 * n_dirs + i]};
            Eval Em;
            int ok = newton_sphere(m, d, dn, Sa, Sb, Em);
            if (better(Em.f, m, fb, nb, dh)) {
                fb = Em.f;
                nb[0] = m[0]; nb[1] = m[1]; nb[2] = m[2];
                Eb = Em;
                st_best = ok ? SNSD_OK : SNSD_NONCONV;
            }
        }
    }
    feval(nb, d, Sa, Sb, Eb);
    write_out(Eb, nb, phi, nout, ra, rb);
    return st_best;
}

// ---- tori: Phi = min over the two centreline circles of their
// distance, minus the minor radii.  The nearest point of ring b to a point has
// a closed form, so the search is over theta_a only: 64 samples, the two best
// sampled local minima refined by bisection on df/dtheta (envelope theorem),
// ties within 1e-13 max(1, D) -> smaller theta_a in [0, 2 pi) (R23).
struct Ring {
    double c[3], e1[3], e2[3], ax[3], R;
};
__device__ __forceinline__ void ring_make(const double *c, const double *g, double Rr, Ring &o) {
    for (int k = 0; k < 3; ++k) {
        o.c[k] = c[k];
        o.e1[k] = g[k];
        o.ax[k] = g[3 + k];
    }
    o.e2[0] = o.ax[1] * o.e1[2] - o.ax[2] * o.e1[1];
    o.e2[1] = o.ax[2] * o.e1[0] - o.ax[0] * o.e1[2];
    o.e2[2] = o.ax[0] * o.e1[1] - o.ax[1] * o.e1[0];
    o.R = Rr;
}
__device__ __forceinline__ void ring_pt(const Ring &g, double th, double *p, double *dp) {
    double sn, cs;
    sincos(th, &sn, &cs);
    for (int k = 0; k < 3; ++k) {
        p[k] = g.c[k] + g.R * (cs * g.e1[k] + sn * g.e2[k]);
        dp[k] = g.R * (-sn * g.e1[k] + cs * g.e2[k]);
    }
}
// nearest point q of ring b to p (axis points: along e1); returns |p - q|^2
__device__ __forceinline__ double ring_near(const Ring &b, const double *p, double *q) {
    const double v[3] = {p[0] - b.c[0], p[1] - b.c[1], p[2] - b.c[2]};
    const double h = v[0] * b.ax[0] + v[1] * b.ax[1] + v[2] * b.ax[2];
    const double w[3] = {v[0] - h * b.ax[0], v[1] - h * b.ax[1], v[2] - h * b.ax[2]};
    const double l = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    const bool ok = l > 1e-14 * (1.0 + b.R);
    double r2 = 0.0;
    for (int k = 0; k < 3; ++k) {
        q[k] = b.c[k] + (ok ? b.R * w[k] / l : b.R * b.e1[k]);
        r2 += (q[k] - p[k]) * (q[k] - p[k]);
    }
    return r2;
}
__device__ __forceinline__ double ring_df(const Ring &a, const Ring &b, double th) {
    double p[3], dp[3], q[3];
    ring_pt(a, th, p, dp);
    ring_near(b, p, q);
    return 2.0 * ((p[0] - q[0]) * dp[0] + (p[1] - q[1]) * dp[1] + (p[2] - q[2]) * dp[2]);
}

__device__ int torus_pair(const double *d, const double *ga, const double *gb, double Ra, double rra, double Rb,
                          double rrb, double &phi, double *nout, double *ra, double *rb) {
    const double zero[3] = {0.0, 0.0, 0.0};
    Ring A, B;
    ring_make(zero, ga, Ra, A);
    ring_make(d, gb, Rb, B);
    constexpr int NS = 64;
    const double two_pi = 6.283185307179586476925;
    double f[NS];
    for (int i = 0; i < NS; ++i) {
        double p[3], dp[3], q[3];
        ring_pt(A, two_pi * i / NS, p, dp);
        f[i] = ring_near(B, p, q);
    }
    // the two best sampled local minima
    int i1 = -1, i2 = -1;
    for (int i = 0; i < NS; ++i) {
        const double fm = f[(i + NS - 1) % NS], fp = f[(i + 1) % NS];
        if (!(f[i] <= fm && f[i] <= fp)) continue;
        if (i1 < 0 || f[i] < f[i1]) {
            i2 = i1;
            i1 = i;
        } else if (i2 < 0 || f[i] < f[i2]) {
            i2 = i;
        }
    }
    double best_th = 0.0, best_D = INFINITY;
    for (int c = 0; c < 2; ++c) {
        const int i = c == 0 ? i1 : i2;
        if (i < 0) continue;
        double lo = two_pi * (i - 1) / NS, hi = two_pi * (i + 1) / NS, th = two_pi * i / NS;
        const bool strict = f[i] < f[(i + NS - 1) % NS] && f[i] < f[(i + 1) % NS];  // plateau: keep the sample
        if (strict && ring_df(A, B, lo) <= 0.0 && ring_df(A, B, hi) >= 0.0) {
            for (int it = 0; it < 64; ++it) {
                const double mid = 0.5 * (lo + hi);
                if (ring_df(A, B, mid) < 0.0) lo = mid; else hi = mid;
            }
            th = 0.5 * (lo + hi);
        }
        th = fmod(th, two_pi);
        if (th < 0.0) th += two_pi;
        double p[3], dp[3], q[3];
        ring_pt(A, th, p, dp);
        const double D = sqrt(ring_near(B, p, q));
        const double tie = 1e-13 * fmax(1.0, fmin(D, best_D));
        if (D < best_D - tie || (fabs(D - best_D) <= tie && th < best_th)) {
            best_D = D;
            best_th = th;
        }
    }
    double pa[3], dp[3], pb[3];
    ring_pt(A, best_th, pa, dp);
    ring_near(B, pa, pb);
    const double v[3] = {pb[0] - pa[0], pb[1] - pa[1], pb[2] - pa[2]};
    const double D = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    if (!(D >= 1e-12)) {
        phi = nan("");
        for (int k = 0; k < 3; ++k) nout[k] = ra[k] = rb[k] = nan("");
        return 1;
    }
    phi = D - rra - rrb;
    for (int k = 0; k < 3; ++k) {
        const double nk = v[k] / D;
        nout[k] = nk;
        ra[k] = pa[k] + rra * nk;
        rb[k] = pb[k] - d[k] - rrb * nk;
    }
    return 0;
}

__device__ __forceinline__ void min_image(const double *xa, const double *xb, const double *box, double *d) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double t = xb[k] - xa[k];
        if (box[k] > 0.0) t -= box[k] * rint(t / box[k]);
        d[k] = t;
    }
}

struct Box3 {
    double v[3];
};

__device__ __forceinline__ void pair_geom(int64_t k, const int *__restrict__ pi, const int *__restrict__ pj,
                                          const double *__restrict__ pos, const double *__restrict__ Sig,
                                          const Box3 &box, double *d, Sym &Sa, Sym &Sb) {
    const int a = pi[k], b = pj[k];
    min_image(pos + 3 * (int64_t)a, pos + 3 * (int64_t)b, box.v, d);
    Sa = load_sym(Sig + 6 * (int64_t)a);
    Sb = load_sym(Sig + 6 * (int64_t)b);
}

__device__ __forceinline__ void store_pair(int64_t k, int64_t planes, double f, const double *n, const double *r1,
                                           const double *r2, double *__restrict__ phi, double *__restrict__ nrm,
                                           double *__restrict__ ra, double *__restrict__ rb) {
    phi[k] = f;
    for (int c = 0; c < 3; ++c) {
        nrm[c * planes + k] = n[c];
        ra[c * planes + k] = r1[c];
        rb[c * planes + k] = r2[c];
    }
}

// Append k to a device list when `push`, one atomic per warp (the list order
// is scheduling dependent; every consumer's per-pair result is not).
__device__ __forceinline__ void list_push(bool push, int64_t k, int *list, unsigned *count) {
    const unsigned act = __activemask();
    const unsigned bal = __ballot_sync(act, push);
    if (!bal) return;
    const int lane = threadIdx.x & 31, leader = __ffs(act) - 1;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(count, (unsigned)__popc(bal));
    base = __shfl_sync(act, base, leader);
    if (push) list[base + __popc(bal & ((1u << lane) - 1u))] = (int)k;
}

// K3/K10 stage 0 over all pairs: spherocylinder / torus / mixed pairs in full;
// ellipsoid pairs get the lower bound Phi >= F(d/|d|) (snsd_stage1) and, when
// it does not reject them, go to the Newton list, so that the Newton stage
// runs with full warps (most pairs of a check are rejected by the bound).
// SHAPES: the bodies carry a shape array (rods / tori possible); without it
// every pair is an ellipsoid pair and the rod / torus code is compiled out.
template <bool SHAPES>
__global__ void __launch_bounds__(128) k_snsd_stage0(int64_t np, const int *__restrict__ pi,
                                                     const int *__restrict__ pj, const double *__restrict__ pos,
                                                     const double *__restrict__ Sig, Box3 box, double reject_above,
                                                     double *__restrict__ phi, double *__restrict__ nrm,
                                                     double *__restrict__ ra, double *__restrict__ rb,
                                                     int *__restrict__ status, int64_t planes, int *nlist,
                                                     unsigned *n_nlist, const int32_t *__restrict__ shape,
                                                     const double *__restrict__ axes) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < np; k += (int64_t)gridDim.x * blockDim.x) {
        double d[3];
        Sym Sa, Sb;
        pair_geom(k, pi, pj, pos, Sig, box, d, Sa, Sb);
        double f, n[3], r1[3], r2[3];
        int st = -1;  // >= 0: outputs final here; -1: bound (phi only) or Newton list
        bool newton = false;
        const int sha = SHAPES ? shape[pi[k]] : 0, shb = SHAPES ? shape[pj[k]] : 0;
        if (SHAPES && sha == RELCP_SHAPE_SPHEROCYLINDER && shb == RELCP_SHAPE_SPHEROCYLINDER) {
            const double ga[6] = {Sa.xx, Sa.xy, Sa.xz, Sa.yy, Sa.yz, Sa.zz};
            const double gb[6] = {Sb.xx, Sb.xy, Sb.xz, Sb.yy, Sb.yz, Sb.zz};
            st = rod_pair(d, ga, gb, f, n, r1, r2);
        } else if (SHAPES && sha == RELCP_SHAPE_TORUS && shb == RELCP_SHAPE_TORUS) {
            const double ga[6] = {Sa.xx, Sa.xy, Sa.xz, Sa.yy, Sa.yz, Sa.zz};
            const double gb[6] = {Sb.xx, Sb.xy, Sb.xz, Sb.yy, Sb.yz, Sb.zz};
            const int64_t a = pi[k], b = pj[k];
            st = torus_pair(d, ga, gb, axes[3 * a], axes[3 * a + 1], axes[3 * b], axes[3 * b + 1], f, n, r1, r2);
        } else if (SHAPES && sha != shb) {  // mixed ellipsoid-rod pairs are not defined (include/relcp.h)
            f = nan("");
            for (int c = 0; c < 3; ++c) n[c] = r1[c] = r2[c] = nan("");
            st = SNSD_DEGENERATE;
        } else {
            const double dn = sqrt(d3(d, d));
            if (!(dn >= 1e-12)) {
                f = nan("");
                for (int c = 0; c < 3; ++c) n[c] = r1[c] = r2[c] = nan("");
                st = SNSD_DEGENERATE;
            } else {
                const double nb[3] = {d[0] / dn, d[1] / dn, d[2] / dn};
                f = fval(nb, d, Sa, Sb);
                if (f >= reject_above + 1e-12 * fmax(1.0, dn)) {
                    // phi = the bound; only phi and the status are consumed (k_flag)
                    phi[k] = f;
                    status[k] = SNSD_BOUND;
                } else {
                    newton = true;
                }
            }
        }
        list_push(newton, k, nlist, n_nlist);
        if (st >= 0) {
            store_pair(k, planes, f, n, r1, r2, phi, nrm, ra, rb);
            status[k] = st;
        }
    }
}

// Stage 1 over the Newton list (ellipsoid pairs under the bound): Newton from
// d/|d|; pairs needing the multistart are listed for stage 2.
__global__ void __launch_bounds__(128, SNSD_MINB) k_snsd_stage1(const int *__restrict__ nlist, const unsigned *__restrict__ n_nlist,
                                                     const int *__restrict__ pi, const int *__restrict__ pj,
                                                     const double *__restrict__ pos, const double *__restrict__ Sig,
                                                     Box3 box, double *__restrict__ phi, double *__restrict__ nrm,
                                                     double *__restrict__ ra, double *__restrict__ rb,
                                                     int *__restrict__ status, int64_t planes, int *multi,
                                                     unsigned *n_multi, const double *__restrict__ axes) {
    const int64_t m = *n_nlist;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = nlist[i];
        double d[3];
        Sym Sa, Sb;
        pair_geom(k, pi, pj, pos, Sig, box, d, Sa, Sb);
        double f, n[3], r1[3], r2[3];
        // curvature certificate depth (R29): half the smallest radius of
        // curvature of K = A + B; an ellipsoid's is min(e)^2 / max(e)
        double cert = 0.0;
        if (axes) {
            auto rmin = [&](int64_t b) {
                const double e0 = axes[3 * b], e1 = axes[3 * b + 1], e2 = axes[3 * b + 2];
                const double lo = fmin(e0, fmin(e1, e2)), hi = fmax(e0, fmax(e1, e2));
                return hi > 0.0 ? lo * lo / hi : 0.0;
            };
            cert = 0.5 * (rmin(pi[k]) + rmin(pj[k]));
        }
        // reject_above = +inf: the bound was tested in stage 0
        const int st = snsd_stage1(d, Sa, Sb, INFINITY, f, n, r1, r2, cert);
        store_pair(k, planes, f, n, r1, r2, phi, nrm, ra, rb);
        const bool mult = st == SNSD_MULTI || st == -SNSD_MULTI;
        list_push(mult, k, multi, n_multi);
        status[k] = mult ? (st == SNSD_MULTI ? SNSD_OK : SNSD_NONCONV) : st;  // incumbent's certification
    }
}

// Stage 2 over the listed (overlapping / touching) pairs: uniform work per thread.
__global__ void __launch_bounds__(128, SNSD_MINB) k_snsd_stage2(const int *__restrict__ multi, const unsigned *__restrict__ n_multi,
                                                     const int *__restrict__ pi, const int *__restrict__ pj,
                                                     const double *__restrict__ pos, const double *__restrict__ Sig,
                                                     Box3 box, int n_dirs, const double *__restrict__ dirs,
                                                     const float *__restrict__ dirs32, double *__restrict__ phi,
                                                     double *__restrict__ nrm, double *__restrict__ ra,
                                                     double *__restrict__ rb, int *__restrict__ status,
                                                     int64_t planes) {
    const int64_t m = *n_multi;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = multi[i];
        double d[3];
        Sym Sa, Sb;
        pair_geom(k, pi, pj, pos, Sig, box, d, Sa, Sb);
        double nb[3] = {nrm[k], nrm[planes + k], nrm[2 * planes + k]};
        double f, n[3], r1[3], r2[3];
        const int st = snsd_stage2(d, Sa, Sb, n_dirs, dirs, dirs32, nb, status[k], f, n, r1, r2);
        store_pair(k, planes, f, n, r1, r2, phi, nrm, ra, rb);
        status[k] = st;
    }
}

__global__ void k_count_add(const unsigned *c, long long *acc) { *acc += *c; }

int geo_snsd(relcp_ctx *ctx, int64_t np, const int *pi, const int *pj, const double *pos, const double *Sig,
             double *phi, double *nrm, double *ra, double *rb, int *status, int64_t planes, double reject_above,
             const int32_t *shape, const double *axes) {
    if (np <= 0) return RELCP_OK;
    Box3 bx;
    for (int k = 0; k < 3; ++k) bx.v[k] = ctx->p.box[k];
    int nd = ctx->p.n_dirs > 0 ? ctx->p.n_dirs : 256;
    if (nd > RELCP_MAX_DIRS) nd = RELCP_MAX_DIRS;
    CK(ctx->multi.grow(np));
    CK(ctx->nlist.grow(np));
    if (ctx->dirs_n != nd) {
        CK(ctx->dirs.grow(3 * nd));
        CK(ctx->dirs32.grow(3 * nd));
        k_dirs<<<(nd + 127) / 128, 128, 0, ctx->stream>>>(nd, ctx->dirs.p, ctx->dirs32.p);
        CKL();
        ctx->dirs_n = nd;
    }
    // counter[1] = stage-2 list length, counter[2] = Newton list length
    CK(cudaMemsetAsync(ctx->counter.p + 1, 0, 2 * sizeof(unsigned), ctx->stream));
    int64_t g = (np + 127) / 128;
    if (g > 148 * 64) g = 148 * 64;
    if (shape)
        k_snsd_stage0<true><<<(unsigned)g, 128, 0, ctx->stream>>>(np, pi, pj, pos, Sig, bx, reject_above, phi, nrm, ra,
                                                                  rb, status, planes, ctx->nlist.p, ctx->counter.p + 2,
                                                                  shape, axes);
    else
        k_snsd_stage0<false><<<(unsigned)g, 128, 0, ctx->stream>>>(np, pi, pj, pos, Sig, bx, reject_above, phi, nrm,
                                                                   ra, rb, status, planes, ctx->nlist.p,
                                                                   ctx->counter.p + 2, shape, axes);
    CKL();
    k_snsd_stage1<<<148 * 8, 128, 0, ctx->stream>>>(ctx->nlist.p, ctx->counter.p + 2, pi, pj, pos, Sig, bx, phi, nrm,
                                                    ra, rb, status, planes, ctx->multi.p, ctx->counter.p + 1,
                                                    ctx->p.snsd_cert ? axes : nullptr);
    CKL();
    k_snsd_stage2<<<148 * 8, 128, 0, ctx->stream>>>(ctx->multi.p, ctx->counter.p + 1, pi, pj, pos, Sig, bx, nd,
                                                    ctx->dirs.p, ctx->dirs32.p, phi, nrm, ra, rb, status, planes);
    CKL();
    if (!ctx->dstat.p) {
        CK(ctx->dstat.grow(4));
        CK(cudaMemsetAsync(ctx->dstat.p, 0, 4 * sizeof(long long), ctx->stream));
    }
    k_count_add<<<1, 1, 0, ctx->stream>>>(ctx->counter.p + 1, ctx->dstat.p);
    CKL();
    return RELCP_OK;
}

// ------------------------------------------------------------ broadphase
struct Grid {
    int nc[3];
    double lo[3];
    double cs[3];     // cell edge per axis
    double box[3];    // > 0: periodic
};

__device__ __forceinline__ int cell_coord(double x, const Grid &G, int k) {
    int c;
    if (G.box[k] > 0.0) {
        double u = x / G.box[k];
        u -= floor(u);
        c = (int)(u * G.nc[k]);
    } else {
        c = (int)floor((x - G.lo[k]) / G.cs[k]);
    }
    return c < 0 ? 0 : (c >= G.nc[k] ? G.nc[k] - 1 : c);
}

// body -> cell; per-cell counts (integer atomics: exact counts)
__global__ void k_cell_assign(int64_t nb, const double *__restrict__ pos, Grid G, int *__restrict__ body_cell,
                              int *__restrict__ cell_count) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        int cx = cell_coord(pos[3 * b], G, 0), cy = cell_coord(pos[3 * b + 1], G, 1), cz = cell_coord(pos[3 * b + 2], G, 2);
        int c = (cz * G.nc[1] + cy) * G.nc[0] + cx;
        body_cell[b] = c;
        atomicAdd(cell_count + c, 1);
    }
}

__global__ void k_cell_fill(int64_t nb, const int *__restrict__ body_cell, const int *__restrict__ cell_start,
                            int *__restrict__ cell_fill, int *__restrict__ items) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        int c = body_cell[b];
        items[cell_start[c] + atomicAdd(cell_fill + c, 1)] = (int)b;
    }
}

// Unique neighbour cells along one axis (periodic wrap or clipped).
__device__ __forceinline__ int axis_neighbours(int c, int k, const Grid &G, int *out) {
    int m = 0;
    for (int o = -1; o <= 1; ++o) {
        int v = c + o;
        if (G.box[k] > 0.0) {
            v = (v % G.nc[k] + G.nc[k]) % G.nc[k];
        } else if (v < 0 || v >= G.nc[k]) {
            continue;
        }
        bool dup = false;
        for (int t = 0; t < m; ++t) dup |= out[t] == v;
        if (!dup) out[m++] = v;
    }
    return m;
}

__device__ __forceinline__ bool near_pair(const double *__restrict__ pos, const double *__restrict__ rad,
                                          const Grid &G, double margin, int i, int j) {
    double d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double t = pos[3 * (int64_t)j + k] - pos[3 * (int64_t)i + k];
        if (G.box[k] > 0.0) t -= G.box[k] * rint(t / G.box[k]);
        d[k] = t;
    }
    const double r = rad[i] + rad[j] + margin;
    return d[0] * d[0] + d[1] * d[1] + d[2] * d[2] < r * r;
}

// pass 0: count pairs (i < j) per body; pass 1: write them, sorted by j.
template <int PASS>
__global__ void __launch_bounds__(128) k_pairs2(int64_t nb, const double *__restrict__ pos,
                                                const double *__restrict__ rad, Grid G, double margin,
                                                const int *__restrict__ body_cell, const int *__restrict__ cell_start,
                                                const int *__restrict__ cell_count, const int *__restrict__ items,
                                                long long *__restrict__ cnt_or_off, int *__restrict__ pi,
                                                int *__restrict__ pj) {
    for (int64_t ib = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ib < nb; ib += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)ib;
        const int c = body_cell[i];
        const int cx = c % G.nc[0], cy = (c / G.nc[0]) % G.nc[1], cz = c / (G.nc[0] * G.nc[1]);
        int nx[3], ny[3], nz[3];
        const int mx = axis_neighbours(cx, 0, G, nx), my = axis_neighbours(cy, 1, G, ny),
                  mz = axis_neighbours(cz, 2, G, nz);
        long long m = 0;
        const long long base = PASS == 1 ? cnt_or_off[i] : 0;
        for (int a = 0; a < mz; ++a)
            for (int b2 = 0; b2 < my; ++b2)
                for (int e = 0; e < mx; ++e) {
                    const int cc = (nz[a] * G.nc[1] + ny[b2]) * G.nc[0] + nx[e];
                    const int s = cell_start[cc], t = s + cell_count[cc];
                    for (int q = s; q < t; ++q) {
                        const int j = items[q];
                        if (j <= i) continue;
                        if (!near_pair(pos, rad, G, margin, i, j)) continue;
                        if (PASS == 1) {
                            pi[base + m] = i;
                            pj[base + m] = j;
                        }
                        ++m;
                    }
                }
        if (PASS == 0) {
            cnt_or_off[i] = m;
        } else {
            // insertion sort of this body's partners: lexicographic (i, j) order
            for (long long u = base + 1; u < base + m; ++u) {
                int k = pj[u];
                long long v = u - 1;
                while (v >= base && pj[v] > k) {
                    pj[v + 1] = pj[v];
                    --v;
                }
                pj[v + 1] = k;
            }
        }
    }
}

// Single pass (the common case): each body's partners j > i go to a
// fixed-capacity slot row tmp[i * cap ...] (sorted there), the count to
// cnt[i]; a body with more than `cap` partners sets *ovf and the caller reruns
// the two-pass kernel above.  cap comes from the previous broadphase's
// largest per-body count (ctx->bp_cap), so the neighbour search runs once.
__global__ void __launch_bounds__(128) k_pairs_one(int64_t nb, const double *__restrict__ pos,
                                                   const double *__restrict__ rad, Grid G, double margin,
                                                   const int *__restrict__ body_cell, const int *__restrict__ cell_start,
                                                   const int *__restrict__ cell_count, const int *__restrict__ items,
                                                   long long *__restrict__ cnt, int *__restrict__ tmp, int cap,
                                                   int *__restrict__ ovf) {
    for (int64_t ib = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ib < nb; ib += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)ib;
        const int c = body_cell[i];
        const int cx = c % G.nc[0], cy = (c / G.nc[0]) % G.nc[1], cz = c / (G.nc[0] * G.nc[1]);
        int nx[3], ny[3], nz[3];
        const int mx = axis_neighbours(cx, 0, G, nx), my = axis_neighbours(cy, 1, G, ny),
                  mz = axis_neighbours(cz, 2, G, nz);
        int *row = tmp + (int64_t)i * cap;
        long long m = 0;
        for (int a = 0; a < mz; ++a)
            for (int b2 = 0; b2 < my; ++b2)
                for (int e = 0; e < mx; ++e) {
                    const int cc = (nz[a] * G.nc[1] + ny[b2]) * G.nc[0] + nx[e];
                    const int s = cell_start[cc], t = s + cell_count[cc];
                    for (int q = s; q < t; ++q) {
                        const int j = items[q];
                        if (j <= i) continue;
                        if (!near_pair(pos, rad, G, margin, i, j)) continue;
                        if (m < cap) row[m] = j;
                        ++m;
                    }
                }
        cnt[i] = m;
        if (m > cap) {
            *ovf = 1;
            continue;
        }
        for (long long u = 1; u < m; ++u) {  // lexicographic (i, j) order
            const int k = row[u];
            long long v = u - 1;
            while (v >= 0 && row[v] > k) {
                row[v + 1] = row[v];
                --v;
            }
            row[v + 1] = k;
        }
    }
}

__global__ void k_max_count(int64_t nb, const long long *__restrict__ cnt, int *mx) {
    int m = 0;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
        m = max(m, (int)min(cnt[b], (long long)1 << 30));
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
}

// slot rows -> the packed pair list at the scanned offsets
__global__ void k_pairs_pack(int64_t nb, const long long *__restrict__ off, const int *__restrict__ tmp, int cap,
                             int *__restrict__ pi, int *__restrict__ pj) {
    const int64_t nw = (nb + 31) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nw;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        // a warp packs 32 consecutive bodies' rows, one body after the other
        const int64_t b0 = w << 5;
        const int64_t bl = b0 + 32 < nb ? b0 + 32 : nb;
        for (int64_t i = b0; i < bl; ++i) {
            const long long o = off[i], m = off[i + 1] - o;
            for (long long u = lane; u < m; u += 32) {
                pi[o + u] = (int)i;
                pj[o + u] = tmp[i * cap + u];
            }
        }
    }
}

// bounds: min pos (3), max pos (3), max rad
__global__ void __launch_bounds__(RELCP_NT) k_bounds(int64_t nb, const double *__restrict__ pos,
                                                     const double *__restrict__ rad, double *part,
                                                     unsigned *counter, double *out) {
    __shared__ double sh[7 * 32];
    double v[7] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY, 0.0};
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        for (int k = 0; k < 3; ++k) {
            v[k] = fmin(v[k], pos[3 * b + k]);
            v[3 + k] = fmax(v[3 + k], pos[3 * b + k]);
        }
        v[6] = fmax(v[6], rad[b]);
    }
    const int ops[7] = {2, 2, 2, 1, 1, 1, 1};
    if (grid_reduce_last<7>(v, ops, part, counter, sh) && threadIdx.x == 0)
        for (int k = 0; k < 7; ++k) out[k] = v[k];
}

int geo_broadphase(relcp_ctx *ctx, int64_t nb, const double *pos, const double *rad, double margin) {
    cudaStream_t st = ctx->stream;
    k_bounds<<<grid_for(nb), RELCP_NT, 0, st>>>(nb, pos, rad, ctx->partials.p, ctx->counter.p, ctx->red.p);
    CKL();
    CK(cudaMemcpyAsync(ctx->red_host, ctx->red.p, 7 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    PHASE(ctx, "bp.bounds");
    double lo[3], hi[3], rmax = ctx->red_host[6];
    for (int k = 0; k < 3; ++k) {
        lo[k] = ctx->red_host[k];
        hi[k] = ctx->red_host[3 + k];
    }
    if (!(rmax > 0.0) || !isfinite(rmax)) return set_err(ctx, RELCP_E_ARG, "broadphase: bad radii / positions");
    double csize = 2.0 * rmax + margin;
    Grid G;
    for (;;) {
        double ncell = 1.0;
        for (int k = 0; k < 3; ++k) {
            G.box[k] = ctx->p.box[k];
            if (G.box[k] > 0.0) {
                int n = (int)floor(G.box[k] / csize);
                G.nc[k] = n < 1 ? 1 : n;
                G.lo[k] = 0.0;
                G.cs[k] = G.box[k] / G.nc[k];
            } else {
                double ext = hi[k] - lo[k];
                int n = (int)floor(ext / csize);
                G.nc[k] = n < 1 ? 1 : n;
                G.lo[k] = lo[k];
                G.cs[k] = n < 1 ? fmax(ext, csize) : ext / n;
                if (G.cs[k] < csize) G.cs[k] = csize;
            }
            ncell *= G.nc[k];
        }
        if (ncell <= 4.0 * (double)nb + 64.0) break;
        csize *= 1.5;
    }
    const int64_t ncell = (int64_t)G.nc[0] * G.nc[1] * G.nc[2];
    CK(ctx->cell_count.grow(ncell + 1));
    CK(ctx->cell_start.grow(ncell + 1));
    CK(ctx->cell_fill.grow(ncell + 1));
    CK(ctx->cell_items.grow(nb));
    CK(ctx->body_cell.grow(nb));
    CK(ctx->pair_cnt.grow(nb + 1));
    CK(cudaMemsetAsync(ctx->cell_count.p, 0, sizeof(int) * (ncell + 1), st));
    CK(cudaMemsetAsync(ctx->cell_fill.p, 0, sizeof(int) * (ncell + 1), st));
    k_cell_assign<<<grid_for(nb), RELCP_NT, 0, st>>>(nb, pos, G, ctx->body_cell.p, ctx->cell_count.p);
    CKL();
    CKS(scan_exclusive_int(ctx, ctx->cell_count.p, ctx->cell_start.p, ncell + 1, nullptr));
    k_cell_fill<<<grid_for(nb), RELCP_NT, 0, st>>>(nb, ctx->body_cell.p, ctx->cell_start.p, ctx->cell_fill.p,
                                                    ctx->cell_items.p);
    CKL();
    PHASE(ctx, "bp.cells");
    const int gp = grid_for(nb, 128, 32);
    long long total = 0;
    CK(ctx->scan_ll.grow(nb + 1));
    if (ctx->bp_cap > 0 && (double)ctx->bp_cap * (double)nb <= 2.0e9) {
        // one neighbour search into slot rows of the last search's largest count (+ slack)
        const int cap = ctx->bp_cap;
        CK(ctx->bp_tmp.grow((size_t)cap * nb));
        CK(cudaMemsetAsync(ctx->counter.p + 3, 0, sizeof(unsigned), st));
        k_pairs_one<<<gp, 128, 0, st>>>(nb, pos, rad, G, margin, ctx->body_cell.p, ctx->cell_start.p,
                                        ctx->cell_count.p, ctx->cell_items.p, ctx->pair_cnt.p, ctx->bp_tmp.p, cap,
                                        (int *)(ctx->counter.p + 3));
        CKL();
        CK(cudaMemsetAsync(ctx->pair_cnt.p + nb, 0, sizeof(long long), st));
        CKS(scan_exclusive_ll(ctx, ctx->pair_cnt.p, ctx->scan_ll.p, nb + 1, &total));  // synchronises
        int ovf = 0;
        CK(cudaMemcpyAsync(&ovf, ctx->counter.p + 3, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (!ovf) {
            PHASE(ctx, "bp.count_scan");
            CK(ctx->pi.grow(total > 0 ? total : 1));
            CK(ctx->pj.grow(total > 0 ? total : 1));
            k_pairs_pack<<<grid_for(32 * ((nb + 31) / 32), 256, 8), 256, 0, st>>>(nb, ctx->scan_ll.p, ctx->bp_tmp.p,
                                                                               cap, ctx->pi.p, ctx->pj.p);
            CKL();
            ctx->npairs = total;
            PHASE(ctx, "bp.pairs");
            return RELCP_OK;
        }
    }
    k_pairs2<0><<<gp, 128, 0, st>>>(nb, pos, rad, G, margin, ctx->body_cell.p, ctx->cell_start.p, ctx->cell_count.p,
                                    ctx->cell_items.p, ctx->pair_cnt.p, nullptr, nullptr);
    CKL();
    CK(cudaMemsetAsync(ctx->pair_cnt.p + nb, 0, sizeof(long long), st));
    CKS(scan_exclusive_ll(ctx, ctx->pair_cnt.p, ctx->scan_ll.p, nb + 1, &total));
    PHASE(ctx, "bp.count_scan");
    // the largest per-body count sizes the next search's slot rows (+ 25 % + 8 slack)
    CK(cudaMemsetAsync(ctx->counter.p + 3, 0, sizeof(unsigned), st));
    k_max_count<<<grid_for(nb), RELCP_NT, 0, st>>>(nb, ctx->pair_cnt.p, (int *)(ctx->counter.p + 3));
    CKL();
    CK(ctx->pi.grow(total > 0 ? total : 1));
    CK(ctx->pj.grow(total > 0 ? total : 1));
    k_pairs2<1><<<gp, 128, 0, st>>>(nb, pos, rad, G, margin, ctx->body_cell.p, ctx->cell_start.p, ctx->cell_count.p,
                                    ctx->cell_items.p, ctx->scan_ll.p, ctx->pi.p, ctx->pj.p);
    CKL();
    int mx = 0;
    CK(cudaMemcpyAsync(&mx, ctx->counter.p + 3, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ctx->bp_cap = mx + mx / 4 + 8;
    ctx->npairs = total;
    PHASE(ctx, "bp.pairs");
    return RELCP_OK;
}
