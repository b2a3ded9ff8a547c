/*
 * relcp_oracle.c -- plain, slow, obviously-correct CPU oracle for the ReLCP
 * hot path of arXiv 2506.14097 ("Smooth-Rigid-Body Contact as a ReLCP").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path in
 * paper_2506_14097_b200/csrc/, and the CUDA path never calls it.
 *
 * Single-threaded C99, fp64 values, `long double` (x87 80-bit) accumulators
 * for every sum.  Citations: P:Lnnn = /root/reference/PAPER.md line.
 *
 *  orc_snsd_pair      shared-normal signed distance of two ellipsoids
 *                     (definition O1 of
 *                     Phi = max_{|n|=1} n.d - h_a(n) - h_b(n)).
 *  orc_snsd_batch     the same over a pair list.
 *  orc_broadphase_*   candidate pairs |d| < R_a + R_b + margin (P:L147,
 *                     P:L532 "near-contacting pairs"), O(N^2) and cell list.
 *  orc_delassus_apply y = s D^T W D x, plain definition (P:L154-157 force
 *                     map F = D gamma; P:L207-211 rows of D^T;
 *                     P:L627 A_n = dt D^T M D; P:L553 inertial dt^2).
 *  orc_bbpgd          Barzilai-Borwein projected gradient for the monotone
 *                     LCP 0 <= A x + q  _|_  x >= 0 (P:L280-299, P:L205
 *                     "projected gradient"; reading R1).
 *  orc_pgs_csr        projected Gauss-Seidel on the assembled A (CSR), the
 *                     independent LCP cross-check.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_DEGENERATE 1
#define ORC_NONCONV 2

/* ---------------------------------------------------------------- helpers */

/* Rotation matrix of the unit quaternion q = (s, w), row-major,
 * R = I + 2 s [w]x + 2 [w]x^2 after normalising q. */
/* Timing-only OpenMP build (bench.py cpu_baseline, "-fopenmp" -> liboracle_omp.so):
 * the independent per-body / per-row loops of the apply and of the BB vector
 * updates run on all host cores; in the apply's wrench scatter each thread
 * adds the terms of its own body range in the serial alpha order.  The test
 * oracle (liboracle.so) is compiled WITHOUT -fopenmp, so these pragmas are
 * empty there and its arithmetic is the serial code below. */
#ifdef _OPENMP
#define ORC_OMP_FOR _Pragma("omp parallel for schedule(static)")
#define ORC_OMP_FOR_REDUCE _Pragma("omp parallel for schedule(static) reduction(+ : ss, sy, yy) reduction(max : r)")
#else
#define ORC_OMP_FOR
#define ORC_OMP_FOR_REDUCE
#endif

static void quat_to_rot(const double q_in[4], double R[9]) {
    double nq = sqrt(q_in[0] * q_in[0] + q_in[1] * q_in[1] + q_in[2] * q_in[2] +
                     q_in[3] * q_in[3]);
    double s = q_in[0] / nq, x = q_in[1] / nq, y = q_in[2] / nq, z = q_in[3] / nq;
    R[0] = 1.0 - 2.0 * (y * y + z * z);
    R[1] = 2.0 * (x * y - s * z);
    R[2] = 2.0 * (x * z + s * y);
    R[3] = 2.0 * (x * y + s * z);
    R[4] = 1.0 - 2.0 * (x * x + z * z);
    R[5] = 2.0 * (y * z - s * x);
    R[6] = 2.0 * (x * z - s * y);
    R[7] = 2.0 * (y * z + s * x);
    R[8] = 1.0 - 2.0 * (x * x + y * y);
}

/* Sigma = R diag(e^2) R^T : the quadratic form of the ellipsoid's support
 * function h(n) = sqrt(n^T Sigma n). */
static void shape_matrix(const double q[4], const double e[3], double S[9]) {
    double R[9];
    quat_to_rot(q, R);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0.0;
            for (int k = 0; k < 3; ++k) acc += R[3 * i + k] * e[k] * e[k] * R[3 * j + k];
            S[3 * i + j] = acc;
        }
}

static void matvec3(const double S[9], const double v[3], double out[3]) {
    for (int i = 0; i < 3; ++i) out[i] = S[3 * i] * v[0] + S[3 * i + 1] * v[1] + S[3 * i + 2] * v[2];
}

static double dot3(const double a[3], const double b[3]) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

static void normalize3(double v[3]) {
    double n = sqrt(dot3(v, v));
    v[0] /= n; v[1] /= n; v[2] /= n;
}

/* Minimum-image offset b - a in a periodic box (box[k] == 0: not periodic). */
static void min_image(const double xa[3], const double xb[3], const double box[3], double d[3]) {
    for (int k = 0; k < 3; ++k) {
        d[k] = xb[k] - xa[k];
        if (box && box[k] > 0.0) d[k] -= box[k] * rint(d[k] / box[k]);
    }
}

/* ------------------------------------------------------------------ SNSD */

/* f(n) = n.d - h_a(n) - h_b(n) and its Euclidean gradient
 * v = d - Sa n / h_a - Sb n / h_b  (= y_b - y_a, the shared-normal gap vector). */
typedef struct {
    double f, v[3], ha, hb, San[3], Sbn[3];
} eval_t;

static void snsd_eval(const double n[3], const double d[3], const double Sa[9], const double Sb[9],
                      eval_t *E) {
    matvec3(Sa, n, E->San);
    matvec3(Sb, n, E->Sbn);
    E->ha = sqrt(dot3(n, E->San));
    E->hb = sqrt(dot3(n, E->Sbn));
    E->f = dot3(n, d) - E->ha - E->hb;
    for (int k = 0; k < 3; ++k) E->v[k] = d[k] - E->San[k] / E->ha - E->Sbn[k] / E->hb;
}

/* Riemannian Newton ascent of f on the unit sphere with Levenberg damping. */
static int snsd_newton(double n[3], const double d[3], const double Sa[9], const double Sb[9],
                       double *f_out, int *iters) {
    const double dn = sqrt(dot3(d, d));
    const double gtol = 1e-13 * (dn > 1.0 ? dn : 1.0);
    eval_t E;
    snsd_eval(n, d, Sa, Sb, &E);
    int converged = 0, it;
    for (it = 0; it < 100; ++it) {
        double nv = dot3(n, E.v);
        double g[3] = {E.v[0] - nv * n[0], E.v[1] - nv * n[1], E.v[2] - nv * n[2]};
        if (sqrt(dot3(g, g)) <= gtol) { converged = 1; break; }
        /* tangent basis t1, t2 */
        double a0 = fabs(n[0]), a1 = fabs(n[1]), a2 = fabs(n[2]);
        double e[3] = {0, 0, 0};
        if (a0 <= a1 && a0 <= a2) e[0] = 1; else if (a1 <= a2) e[1] = 1; else e[2] = 1;
        double ne = dot3(n, e);
        double t1[3] = {e[0] - ne * n[0], e[1] - ne * n[1], e[2] - ne * n[2]};
        normalize3(t1);
        double t2[3] = {n[1] * t1[2] - n[2] * t1[1], n[2] * t1[0] - n[0] * t1[2], n[0] * t1[1] - n[1] * t1[0]};
        /* Euclidean Hessian Hf = -(Sa/ha - San San^T/ha^3) - (Sb/hb - Sbn Sbn^T/hb^3) */
        const double *T[2] = {t1, t2};
        double H2[2][2];
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) {
                double Sat[3], Sbt[3];
                matvec3(Sa, T[j], Sat);
                matvec3(Sb, T[j], Sbt);
                double hij = -(dot3(T[i], Sat) / E.ha - dot3(T[i], E.San) * dot3(T[j], E.San) / (E.ha * E.ha * E.ha))
                             - (dot3(T[i], Sbt) / E.hb - dot3(T[i], E.Sbn) * dot3(T[j], E.Sbn) / (E.hb * E.hb * E.hb));
                H2[i][j] = hij - (i == j ? nv : 0.0);
            }
        double hs = 0.5 * (H2[0][1] + H2[1][0]);
        double A = H2[0][0], B = hs, C = H2[1][1];
        double g2[2] = {dot3(t1, E.v), dot3(t2, E.v)};
        double lam_max = 0.5 * (A + C) + sqrt(0.25 * (A - C) * (A - C) + B * B);
        double hscale = fabs(A) + fabs(B) + fabs(C) + 1e-300;
        double mu = lam_max > -1e-8 * hscale ? lam_max + 1e-8 * hscale + 1e-12 : 0.0;
        int accepted = 0;
        double xi_norm = 0.0, n_new[3];
        eval_t En;
        for (int tries = 0; tries < 60; ++tries) {
            double a = A - mu, c = C - mu;
            double det = a * c - B * B;
            double xi0 = -(c * g2[0] - B * g2[1]) / det;
            double xi1 = -(-B * g2[0] + a * g2[1]) / det;
            double xn = sqrt(xi0 * xi0 + xi1 * xi1);
            if (xn > 0.5) { xi0 *= 0.5 / xn; xi1 *= 0.5 / xn; xn = 0.5; }
            for (int k = 0; k < 3; ++k) n_new[k] = n[k] + xi0 * t1[k] + xi1 * t2[k];
            normalize3(n_new);
            snsd_eval(n_new, d, Sa, Sb, &En);
            if (En.f >= E.f - 1e-15 * (1.0 + dn)) { accepted = 1; xi_norm = xn; break; }
            mu = 4.0 * mu + hscale + 1e-12;
        }
        if (!accepted) { converged = 1; break; } /* no ascent direction left at rounding level */
        n[0] = n_new[0]; n[1] = n_new[1]; n[2] = n_new[2];
        E = En;
        if (xi_norm < 1e-14) { converged = 1; ++it; break; }
    }
    *f_out = E.f;
    if (iters) *iters = it;
    return converged ? ORC_OK : ORC_NONCONV;
}

/* Shared-normal signed distance of two ellipsoids.
 * out: phi, n[3] (outward normal of a), ra[3] = y_a - x_a, rb[3] = y_b - x_b.
 * Multi-start: the best n_fib Fibonacci-sphere directions and d/|d| seed
 * Newton; the largest converged maximum wins (ties: larger n.d/|d|, then the
 * lexicographically smaller n; reading R4). */
int orc_snsd_pair(const double xa[3], const double qa[4], const double ea[3],
                  const double xb[3], const double qb[4], const double eb[3],
                  const double box[3], int n_fib, double out[10], int *iters_out) {
    double d[3], Sa[9], Sb[9];
    min_image(xa, xb, box, d);
    double dn = sqrt(dot3(d, d));
    if (dn < 1e-12) return ORC_DEGENERATE;
    shape_matrix(qa, ea, Sa);
    shape_matrix(qb, eb, Sb);
    enum { K = 4 };
    double best_dir[K + 1][3];
    double best_f[K];
    int nb = 0;
    const double golden = M_PI * (3.0 - sqrt(5.0));
    for (int i = 0; i < n_fib; ++i) {
        double z = 1.0 - (2.0 * i + 1.0) / n_fib;
        double r = sqrt(1.0 - z * z);
        double ph = golden * i;
        double n[3] = {r * cos(ph), r * sin(ph), z};
        eval_t E;
        snsd_eval(n, d, Sa, Sb, &E);
        /* insertion into the top-K list */
        int pos = nb;
        while (pos > 0 && best_f[pos - 1] < E.f) --pos;
        if (pos < K) {
            int last = nb < K ? nb : K - 1;
            for (int m = last; m > pos; --m) {
                best_f[m] = best_f[m - 1];
                memcpy(best_dir[m], best_dir[m - 1], sizeof(best_dir[m]));
            }
            best_f[pos] = E.f;
            memcpy(best_dir[pos], n, sizeof(n));
            if (nb < K) ++nb;
        }
    }
    double dhat[3] = {d[0] / dn, d[1] / dn, d[2] / dn};
    memcpy(best_dir[nb], dhat, sizeof(dhat));
    int nstart = nb + 1;
    double fb = -INFINITY, nbest[3] = {0, 0, 0};
    int status_best = ORC_NONCONV, it_total = 0;
    for (int s = 0; s < nstart; ++s) {
        double n[3] = {best_dir[s][0], best_dir[s][1], best_dir[s][2]};
        double f;
        int it;
        int st = snsd_newton(n, d, Sa, Sb, &f, &it);
        it_total += it;
        int better = 0;
        if (f > fb) better = 1;
        else if (f == fb) {
            double c1 = dot3(n, dhat), c0 = dot3(nbest, dhat);
            if (c1 > c0) better = 1;
            else if (c1 == c0 && (n[0] < nbest[0] || (n[0] == nbest[0] && (n[1] < nbest[1] || (n[1] == nbest[1] && n[2] < nbest[2])))))
                better = 1;
        }
        if (better) { fb = f; memcpy(nbest, n, sizeof(n)); status_best = st; }
    }
    eval_t E;
    snsd_eval(nbest, d, Sa, Sb, &E);
    out[0] = E.f;
    out[1] = nbest[0]; out[2] = nbest[1]; out[3] = nbest[2];
    for (int k = 0; k < 3; ++k) {
        out[4 + k] = E.San[k] / E.ha;   /* y_a - x_a : support point of a along n   */
        out[7 + k] = -E.Sbn[k] / E.hb;  /* y_b - x_b : support point of b along -n  */
    }
    if (iters_out) *iters_out = it_total;
    return status_best;
}

/* Batched SNSD over pairs (pi[k], pj[k]).  Bodies: pos (N,3), quat (N,4),
 * axes (N,3), row-major.  Outputs phi (P), nrm (P,3), ra (P,3), rb (P,3),
 * status (P).  Returns the number of non-OK pairs. */
int64_t orc_snsd_batch(int64_t n_pairs, const int32_t *pi, const int32_t *pj, const double *pos,
                       const double *quat, const double *axes, const double *box, int n_fib,
                       double *phi, double *nrm, double *ra, double *rb, int32_t *status) {
    int64_t bad = 0;
    for (int64_t k = 0; k < n_pairs; ++k) {
        int a = pi[k], b = pj[k];
        double out[10];
        int st = orc_snsd_pair(pos + 3 * a, quat + 4 * a, axes + 3 * a, pos + 3 * b, quat + 4 * b,
                               axes + 3 * b, box, n_fib, out, NULL);
        status[k] = st;
        if (st != ORC_OK) ++bad;
        if (st == ORC_DEGENERATE) { for (int m = 0; m < 10; ++m) out[m] = NAN; }
        phi[k] = out[0];
        for (int m = 0; m < 3; ++m) {
            nrm[3 * k + m] = out[1 + m];
            ra[3 * k + m] = out[4 + m];
            rb[3 * k + m] = out[7 + m];
        }
    }
    return bad;
}

/* ----------------------------------------------------- spherocylinders */

/* Shared-normal signed distance of two spherocylinders ("the
 * minimum-distance problem between the two centerline segments ... after
 * which the cap radii were subtracted").  Body frame: centerline along body x
 * from -h to +h (h = half-length), radius r.  Plain definition: minimise the
 * convex quadratic f(s, t) = |d + t u_b - s u_a|^2 over the rectangle
 * [-h_a, h_a] x [-h_b, h_b] by enumerating every face of the rectangle
 * (interior stationary point, the four edges with their exact 1-D minimiser,
 * the four corners) and keeping the smallest f.  Parallel axes (|u_a x u_b|
 * below 1e-12): the minimisers form a segment; the tie is broken by the
 * midpoint of the overlap of the two projections on u_a (DESIGN R22).
 * out: phi, n (3), ra = y_a - x_a (3), rb = y_b - x_b (3).  Returns
 * ORC_DEGENERATE when the centrelines intersect (no normal). */
static double seg_f(const double d[3], const double ua[3], const double ub[3], double s, double t) {
    double v[3];
    for (int k = 0; k < 3; ++k) v[k] = d[k] + t * ub[k] - s * ua[k];
    return dot3(v, v);
}

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

int orc_rod_pair(const double xa[3], const double qa[4], double ha, double rra, const double xb[3],
                 const double qb[4], double hb, double rrb, const double box[3], double out[10]) {
    double d[3], Ra[9], Rb[9];
    min_image(xa, xb, box, d);
    quat_to_rot(qa, Ra);
    quat_to_rot(qb, Rb);
    const double ua[3] = {Ra[0], Ra[3], Ra[6]}, ub[3] = {Rb[0], Rb[3], Rb[6]};  /* body x axis */
    const double c = dot3(ua, ub), da = dot3(ua, d), db = dot3(ub, d);
    double cr[3] = {ua[1] * ub[2] - ua[2] * ub[1], ua[2] * ub[0] - ua[0] * ub[2], ua[0] * ub[1] - ua[1] * ub[0]};
    double s, t;
    if (sqrt(dot3(cr, cr)) < 1e-12) {
        /* parallel: projections of A and B on u_a, midpoint of their overlap */
        const double sg = c > 0.0 ? 1.0 : -1.0;
        const double lo = fmax(-ha, da - hb), hi = fmin(ha, da + hb);
        if (lo <= hi) s = 0.5 * (lo + hi);
        else s = (da > 0.0) ? ha : -ha;
        const double proj_b = clampd(s, da - hb, da + hb); /* B's projection closest to s */
        t = sg * (proj_b - da);
    } else {
        double bs = 0.0, bt = 0.0, bf = INFINITY;
        /* interior stationary point */
        const double den = 1.0 - c * c;
        double cand[9][2];
        int m = 0;
        cand[m][0] = (da - c * db) / den; cand[m][1] = (c * da - db) / den; ++m;
        /* edges: s = +-ha with the best t, t = +-hb with the best s */
        for (int e = -1; e <= 1; e += 2) {
            cand[m][0] = e * ha; cand[m][1] = clampd(-db + e * ha * c, -hb, hb); ++m;
            cand[m][1] = e * hb; cand[m][0] = clampd(da + e * hb * c, -ha, ha); ++m;
        }
        for (int e = -1; e <= 1; e += 2)
            for (int g = -1; g <= 1; g += 2) { cand[m][0] = e * ha; cand[m][1] = g * hb; ++m; }
        for (int k = 0; k < m; ++k) {
            double cs = cand[k][0], ct = cand[k][1];
            if (cs < -ha || cs > ha || ct < -hb || ct > hb) continue;  /* infeasible interior point */
            double f = seg_f(d, ua, ub, cs, ct);
            if (f < bf) { bf = f; bs = cs; bt = ct; }
        }
        s = bs; t = bt;
    }
    double v[3];
    for (int k = 0; k < 3; ++k) v[k] = d[k] + t * ub[k] - s * ua[k];
    const double dist = sqrt(dot3(v, v));
    if (dist < 1e-12) return ORC_DEGENERATE;
    out[0] = dist - rra - rrb;
    for (int k = 0; k < 3; ++k) {
        const double nk = v[k] / dist;
        out[1 + k] = nk;
        out[4 + k] = s * ua[k] + rra * nk;  /* y_a - x_a */
        out[7 + k] = t * ub[k] - rrb * nk;  /* y_b - x_b */
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ tori */

/* Torus = tube of radius r around the centreline circle of radius R in the
 * body x-y plane (ring axis = body z).  SNSD of two tori (P:L1080 / S:L56:
 * "two-dimensional minimization" of the centreline distance minus the minor
 * radii): Phi = min_{theta_a, theta_b} |c_b(theta_b) - c_a(theta_a)| - r_a - r_b.
 * The inner minimum over theta_b has a closed form (nearest point of circle b
 * to a point: project into b's plane and scale to R_b), so the oracle samples
 * theta_a densely (4096), refines EVERY sampled local minimum by golden
 * section (200 iterations) and keeps the global one.  Set-valued minima
 * ("deterministic selection rule", DESIGN R23): values within
 * 1e-13 max(1, D) count as ties; the smallest theta_a in [0, 2 pi) wins.
 * A point on b's axis has no unique nearest point: b's body x direction. */
typedef struct {
    double c[3], e1[3], e2[3], ax[3], R;
} ring_t;

static void ring_of(const double x[3], const double q[4], double R, ring_t *g) {
    double M[9];
    quat_to_rot(q, M);
    for (int k = 0; k < 3; ++k) {
        g->c[k] = x[k];
        g->e1[k] = M[3 * k];
        g->e2[k] = M[3 * k + 1];
        g->ax[k] = M[3 * k + 2];
    }
    g->R = R;
}

static void ring_point(const ring_t *g, double th, double p[3]) {
    const double cs = cos(th), sn = sin(th);
    for (int k = 0; k < 3; ++k) p[k] = g->c[k] + g->R * (cs * g->e1[k] + sn * g->e2[k]);
}

/* nearest point of ring b to p; returns the squared distance */
static double ring_nearest(const ring_t *b, const double p[3], double out[3]) {
    double q[3], qp[3];
    for (int k = 0; k < 3; ++k) q[k] = p[k] - b->c[k];
    const double h = dot3(q, b->ax);
    for (int k = 0; k < 3; ++k) qp[k] = q[k] - h * b->ax[k];
    const double l = sqrt(dot3(qp, qp));
    for (int k = 0; k < 3; ++k)
        out[k] = b->c[k] + (l > 1e-14 * (1.0 + b->R) ? b->R * qp[k] / l : b->R * b->e1[k]);
    double v[3] = {out[0] - p[0], out[1] - p[1], out[2] - p[2]};
    return dot3(v, v);
}

static double ring_fa(const ring_t *a, const ring_t *b, double th) {
    double p[3], o[3];
    ring_point(a, th, p);
    return ring_nearest(b, p, o);
}

/* d/dtheta of ring_fa (envelope theorem: the inner nearest point is stationary):
 * 2 (p - q) . p'(theta), p'(theta) = R (-sin e1 + cos e2) */
static double ring_dfa(const ring_t *a, const ring_t *b, double th) {
    double p[3], q[3];
    ring_point(a, th, p);
    ring_nearest(b, p, q);
    const double cs = cos(th), sn = sin(th);
    double acc = 0.0;
    for (int k = 0; k < 3; ++k) acc += (p[k] - q[k]) * a->R * (-sn * a->e1[k] + cs * a->e2[k]);
    return 2.0 * acc;
}

int orc_torus_pair(const double xa[3], const double qa[4], double Ra, double rra, const double xb[3],
                   const double qb[4], double Rb, double rrb, const double box[3], double out[10]) {
    double d[3], xa0[3] = {0, 0, 0};
    min_image(xa, xb, box, d);
    ring_t A, B;
    ring_of(xa0, qa, Ra, &A);
    ring_of(d, qb, Rb, &B); /* frame centred on a */
    enum { NS = 4096 };
    static const double TWO_PI = 6.283185307179586476925;
    double fs[NS];
    for (int i = 0; i < NS; ++i) fs[i] = ring_fa(&A, &B, TWO_PI * i / NS);
    double best_th = 0.0, best_f = INFINITY;
    for (int i = 0; i < NS; ++i) {
        const double fm = fs[(i + NS - 1) % NS], fp = fs[(i + 1) % NS];
        if (!(fs[i] <= fm && fs[i] <= fp)) continue; /* not a sampled local minimum */
        /* bisection on the sign change of d f / d theta inside the bracket */
        double lo = TWO_PI * (i - 1) / NS, hi = TWO_PI * (i + 1) / NS, th = TWO_PI * i / NS;
        /* a flat (set-valued) neighbourhood keeps the exact sample angle */
        const int strict = fs[i] < fm && fs[i] < fp;
        if (strict && ring_dfa(&A, &B, lo) <= 0.0 && ring_dfa(&A, &B, hi) >= 0.0) {
            for (int it = 0; it < 100; ++it) {
                const double mid = 0.5 * (lo + hi);
                if (ring_dfa(&A, &B, mid) < 0.0) lo = mid; else hi = mid;
            }
            th = 0.5 * (lo + hi);
        }
        double f = ring_fa(&A, &B, th);
        th = fmod(th, TWO_PI);
        if (th < 0) th += TWO_PI;
        const double tie = 1e-13 * fmax(1.0, sqrt(fmax(f, best_f == INFINITY ? f : best_f)));
        if (sqrt(f) < sqrt(best_f) - tie || (fabs(sqrt(f) - sqrt(best_f)) <= tie && th < best_th)) {
            best_f = f;
            best_th = th;
        }
    }
    double pa[3], pb[3];
    ring_point(&A, best_th, pa);
    ring_nearest(&B, pa, pb);
    double v[3] = {pb[0] - pa[0], pb[1] - pa[1], pb[2] - pa[2]};
    const double D = sqrt(dot3(v, v));
    if (D < 1e-12) return ORC_DEGENERATE;
    out[0] = D - rra - rrb;
    for (int k = 0; k < 3; ++k) {
        const double nk = v[k] / D;
        out[1 + k] = nk;
        out[4 + k] = pa[k] + rra * nk;        /* y_a - x_a */
        out[7 + k] = pb[k] - d[k] - rrb * nk; /* y_b - x_b */
    }
    return ORC_OK;
}

/* Batched SNSD with per-body shapes: 0 ellipsoid (axes = semi-axes), 1
 * spherocylinder (axes[0] = half-length, axes[1] = radius), 2 torus (axes[0] =
 * major radius R, axes[1] = minor radius r).  Mixed pairs are not defined by
 * the paper: status ORC_NONCONV + NaN outputs. */
int64_t orc_snsd_batch_shapes(int64_t n_pairs, const int32_t *pi, const int32_t *pj, const double *pos,
                              const double *quat, const double *axes, const int32_t *shape, const double *box,
                              int n_fib, double *phi, double *nrm, double *ra, double *rb, int32_t *status) {
    int64_t bad = 0;
    for (int64_t k = 0; k < n_pairs; ++k) {
        int a = pi[k], b = pj[k];
        double out[10];
        int st;
        if (shape[a] == 0 && shape[b] == 0)
            st = orc_snsd_pair(pos + 3 * a, quat + 4 * a, axes + 3 * a, pos + 3 * b, quat + 4 * b, axes + 3 * b, box,
                               n_fib, out, NULL);
        else if (shape[a] == 1 && shape[b] == 1)
            st = orc_rod_pair(pos + 3 * a, quat + 4 * a, axes[3 * a], axes[3 * a + 1], pos + 3 * b, quat + 4 * b,
                              axes[3 * b], axes[3 * b + 1], box, out);
        else if (shape[a] == 2 && shape[b] == 2)
            st = orc_torus_pair(pos + 3 * a, quat + 4 * a, axes[3 * a], axes[3 * a + 1], pos + 3 * b, quat + 4 * b,
                                axes[3 * b], axes[3 * b + 1], box, out);
        else
            st = ORC_NONCONV;
        status[k] = st;
        if (st != ORC_OK) {
            ++bad;
            for (int m = 0; m < 10; ++m) out[m] = NAN;
        }
        phi[k] = out[0];
        for (int m = 0; m < 3; ++m) {
            nrm[3 * k + m] = out[1 + m];
            ra[3 * k + m] = out[4 + m];
            rb[3 * k + m] = out[7 + m];
        }
    }
    return bad;
}

/* ------------------------------------------------------------ broadphase */

/* Candidate test, written once: |d|^2 < (R_i + R_j + margin)^2, d the
 * minimum-image centre offset, R the bounding radius (largest semi-axis). */
static int near_pair(const double *pos, const double *rad, const double *box, double margin, int i, int j) {
    double d[3];
    min_image(pos + 3 * i, pos + 3 * j, box, d);
    double d2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
    double r = rad[i] + rad[j] + margin;
    return d2 < r * r;
}

/* O(N^2) all-pairs scan; pairs (i < j) in lexicographic order.  Returns the
 * pair count (may exceed cap; only the first cap are written). */
int64_t orc_broadphase_bruteforce(int64_t n, const double *pos, const double *rad, const double *box,
                                  double margin, int32_t *out_i, int32_t *out_j, int64_t cap) {
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = i + 1; j < n; ++j)
            if (near_pair(pos, rad, box, margin, (int)i, (int)j)) {
                if (m < cap) { out_i[m] = (int32_t)i; out_j[m] = (int32_t)j; }
                ++m;
            }
    return m;
}

static int cmp_pair(const void *pa, const void *pb) {
    const int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
    return (a > b) - (a < b);
}

/* Plain cell list for a periodic cube (all box[k] > 0) with at least 3 cells
 * per axis; falls back to the O(N^2) scan otherwise. */
int64_t orc_broadphase_cells(int64_t n, const double *pos, const double *rad, const double *box,
                             double margin, int32_t *out_i, int32_t *out_j, int64_t cap) {
    double rmax = 0.0;
    for (int64_t i = 0; i < n; ++i) if (rad[i] > rmax) rmax = rad[i];
    double csize = 2.0 * rmax + margin;
    int nc[3];
    for (int k = 0; k < 3; ++k) {
        if (!(box && box[k] > 0.0)) return orc_broadphase_bruteforce(n, pos, rad, box, margin, out_i, out_j, cap);
        nc[k] = (int)floor(box[k] / csize);
        if (nc[k] < 3) return orc_broadphase_bruteforce(n, pos, rad, box, margin, out_i, out_j, cap);
    }
    int64_t ncell = (int64_t)nc[0] * nc[1] * nc[2];
    int64_t *head = malloc(sizeof(int64_t) * ncell), *next = malloc(sizeof(int64_t) * n);
    int *cell_of = malloc(sizeof(int) * 3 * n);
    for (int64_t c = 0; c < ncell; ++c) head[c] = -1;
    for (int64_t i = n - 1; i >= 0; --i) {
        int c3[3];
        for (int k = 0; k < 3; ++k) {
            double u = pos[3 * i + k] / box[k];
            u -= floor(u);
            int ci = (int)(u * nc[k]);
            if (ci >= nc[k]) ci = nc[k] - 1;
            if (ci < 0) ci = 0;
            c3[k] = ci;
            cell_of[3 * i + k] = ci;
        }
        int64_t c = ((int64_t)c3[2] * nc[1] + c3[1]) * nc[0] + c3[0];
        next[i] = head[c];
        head[c] = i;
    }
    int64_t m = 0, mcap = 1024;
    int64_t *keys = malloc(sizeof(int64_t) * mcap);
    for (int64_t i = 0; i < n; ++i) {
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    int cx = (cell_of[3 * i] + dx + nc[0]) % nc[0];
                    int cy = (cell_of[3 * i + 1] + dy + nc[1]) % nc[1];
                    int cz = (cell_of[3 * i + 2] + dz + nc[2]) % nc[2];
                    int64_t c = ((int64_t)cz * nc[1] + cy) * nc[0] + cx;
                    for (int64_t j = head[c]; j >= 0; j = next[j]) {
                        if (j <= i) continue;
                        if (near_pair(pos, rad, box, margin, (int)i, (int)j)) {
                            if (m == mcap) { mcap *= 2; keys = realloc(keys, sizeof(int64_t) * mcap); }
                            keys[m++] = (i << 32) | j;
                        }
                    }
                }
    }
    qsort(keys, (size_t)m, sizeof(int64_t), cmp_pair);
    for (int64_t k = 0; k < m && k < cap; ++k) {
        out_i[k] = (int32_t)(keys[k] >> 32);
        out_j[k] = (int32_t)(keys[k] & 0xffffffff);
    }
    free(keys); free(head); free(next); free(cell_of);
    return m;
}

/* ------------------------------------------------------------- Delassus */

/* y = s * D^T W D x, plain definition.
 *   column alpha of D: [-n; -t_a] at body ia, [n; t_b] at body ib
 *   (F_a = -n gamma, T_a = -(y_a - x_a) x n gamma; row of D^T
 *   = [-n^T, -t_a^T, n^T, t_b^T]).
 *   W: per-body dense 6x6 block, row-major (N,36): M^{-1} (inertial) or the
 *   local-drag mobility (overdamped).
 * Wrenches F_b are accumulated over alpha = 0..nc-1 in long double. */
void orc_delassus_apply(int64_t nb, int64_t nc, const int32_t *ia, const int32_t *ib, const double *nrm,
                        const double *ta, const double *tb, const double *W, double s, const double *x,
                        double *y) {
    long double *F = calloc((size_t)(6 * nb), sizeof(long double));
    long double *U = calloc((size_t)(6 * nb), sizeof(long double));
#ifdef _OPENMP
    /* timing build: thread t owns bodies [lo, hi) and adds, in the same
     * alpha order, only the wrench terms of its own bodies (same sums) */
#pragma omp parallel
    {
        const int64_t T = omp_get_num_threads(), t = omp_get_thread_num();
        const int64_t lo = nb * t / T, hi = nb * (t + 1) / T;
        for (int64_t al = 0; al < nc; ++al) {
            long double xa = x[al];
            int a = ia[al], b = ib[al];
            const int own_a = a >= lo && a < hi, own_b = b >= lo && b < hi;
            for (int k = 0; k < 3 && (own_a || own_b); ++k) {
                if (own_a) F[6 * a + k] += -(long double)nrm[3 * al + k] * xa;
                if (own_a) F[6 * a + 3 + k] += -(long double)ta[3 * al + k] * xa;
                if (own_b) F[6 * b + k] += (long double)nrm[3 * al + k] * xa;
                if (own_b) F[6 * b + 3 + k] += (long double)tb[3 * al + k] * xa;
            }
        }
    }
#else
    for (int64_t al = 0; al < nc; ++al) {
        long double xa = x[al];
        int a = ia[al], b = ib[al];
        for (int k = 0; k < 3; ++k) {
            F[6 * a + k] += -(long double)nrm[3 * al + k] * xa;
            F[6 * a + 3 + k] += -(long double)ta[3 * al + k] * xa;
            F[6 * b + k] += (long double)nrm[3 * al + k] * xa;
            F[6 * b + 3 + k] += (long double)tb[3 * al + k] * xa;
        }
    }
#endif
    ORC_OMP_FOR
    for (int64_t b = 0; b < nb; ++b)
        for (int i = 0; i < 6; ++i) {
            long double acc = 0.0L;
            for (int j = 0; j < 6; ++j) acc += (long double)W[36 * b + 6 * i + j] * F[6 * b + j];
            U[6 * b + i] = acc;
        }
    ORC_OMP_FOR
    for (int64_t al = 0; al < nc; ++al) {
        int a = ia[al], b = ib[al];
        long double acc = 0.0L;
        for (int k = 0; k < 3; ++k) {
            acc += -(long double)nrm[3 * al + k] * U[6 * a + k];
            acc += -(long double)ta[3 * al + k] * U[6 * a + 3 + k];
            acc += (long double)nrm[3 * al + k] * U[6 * b + k];
            acc += (long double)tb[3 * al + k] * U[6 * b + 3 + k];
        }
        y[al] = (double)((long double)s * acc);
    }
    free(F);
    free(U);
}

/* Body wrench F = D x (N,6) and U = W F, both in long double then rounded. */
void orc_wrench(int64_t nb, int64_t nc, const int32_t *ia, const int32_t *ib, const double *nrm,
                const double *ta, const double *tb, const double *W, const double *x, double *F_out,
                double *U_out) {
    long double *F = calloc((size_t)(6 * nb), sizeof(long double));
    for (int64_t al = 0; al < nc; ++al) {
        long double xa = x[al];
        int a = ia[al], b = ib[al];
        for (int k = 0; k < 3; ++k) {
            F[6 * a + k] += -(long double)nrm[3 * al + k] * xa;
            F[6 * a + 3 + k] += -(long double)ta[3 * al + k] * xa;
            F[6 * b + k] += (long double)nrm[3 * al + k] * xa;
            F[6 * b + 3 + k] += (long double)tb[3 * al + k] * xa;
        }
    }
    for (int64_t b = 0; b < nb; ++b)
        for (int i = 0; i < 6; ++i) {
            long double acc = 0.0L;
            for (int j = 0; j < 6; ++j) acc += (long double)W[36 * b + 6 * i + j] * F[6 * b + j];
            if (F_out) F_out[6 * b + i] = (double)F[6 * b + i];
            if (U_out) U_out[6 * b + i] = (double)acc;
        }
    free(F);
}

/* ----------------------------------------------------------------- LCP */

static long double ldot(int64_t n, const double *a, const double *b) {
    long double acc = 0.0L;
    for (int64_t i = 0; i < n; ++i) acc += (long double)a[i] * b[i];
    return acc;
}

/* Barzilai-Borwein projected gradient for 0 <= g = A x + q _|_ x >= 0 with
 * A = s D^T W D applied matrix-free (Lemma 3; CQP form P:L195-205).
 *   alpha_0 = 1/L, L from `power_iters` power iterations on A;
 *   x+ = max(0, x - alpha g); g+ = A x+ + q; s = x+ - x; y = g+ - g;
 *   alpha = s.s / s.y (BB1, even k) or s.y / y.y (BB2, odd k); 1/L if s.y <= 0;
 *   stop when r = ||min(x+, g+)||_inf <= tol.
 * x: in = warm start (projected onto x >= 0), out = solution; g out.
 * info[0] = iterations, info[1] = residual, info[2] = converged, info[3] = L. */
void orc_bbpgd(int64_t nb, int64_t nc, const int32_t *ia, const int32_t *ib, const double *nrm,
               const double *ta, const double *tb, const double *W, double s, const double *q, double *x,
               double *g, double tol, int64_t max_iter, int power_iters, double *info) {
    double *v = malloc(sizeof(double) * (nc > 0 ? nc : 1));
    double *Av = malloc(sizeof(double) * (nc > 0 ? nc : 1));
    double *xn = malloc(sizeof(double) * (nc > 0 ? nc : 1));
    double *gn = malloc(sizeof(double) * (nc > 0 ? nc : 1));
    double L = 0.0;
    /* power iteration for the largest eigenvalue of A */
    for (int64_t i = 0; i < nc; ++i) v[i] = 1.0 / sqrt((double)nc);
    for (int it = 0; it < power_iters && nc > 0; ++it) {
        orc_delassus_apply(nb, nc, ia, ib, nrm, ta, tb, W, s, v, Av);
        double nrm2 = sqrt((double)ldot(nc, Av, Av));
        L = nrm2;
        if (nrm2 == 0.0) break;
        for (int64_t i = 0; i < nc; ++i) v[i] = Av[i] / nrm2;
    }
    if (L <= 0.0) L = 1.0;
    double alpha = 1.0 / L;
    for (int64_t i = 0; i < nc; ++i) x[i] = x[i] > 0.0 ? x[i] : 0.0;
    orc_delassus_apply(nb, nc, ia, ib, nrm, ta, tb, W, s, x, g);
    for (int64_t i = 0; i < nc; ++i) g[i] += q[i];
    double r = 0.0;
    for (int64_t i = 0; i < nc; ++i) { double m = fabs(fmin(x[i], g[i])); if (m > r) r = m; }
    int64_t k = 0;
    int conv = r <= tol;
    while (!conv && k < max_iter) {
        ORC_OMP_FOR
        for (int64_t i = 0; i < nc; ++i) { double t = x[i] - alpha * g[i]; xn[i] = t > 0.0 ? t : 0.0; }
        orc_delassus_apply(nb, nc, ia, ib, nrm, ta, tb, W, s, xn, gn);
        ORC_OMP_FOR
        for (int64_t i = 0; i < nc; ++i) gn[i] += q[i];
        long double ss = 0.0L, sy = 0.0L, yy = 0.0L;
        r = 0.0;
        ORC_OMP_FOR_REDUCE
        for (int64_t i = 0; i < nc; ++i) {
            long double si = (long double)xn[i] - x[i], yi = (long double)gn[i] - g[i];
            ss += si * si; sy += si * yi; yy += yi * yi;
            double m = fabs(fmin(xn[i], gn[i]));
            if (m > r) r = m;
        }
        memcpy(x, xn, sizeof(double) * nc);
        memcpy(g, gn, sizeof(double) * nc);
        if (r <= tol) { conv = 1; ++k; break; }
        if (sy <= 0.0L || yy == 0.0L) alpha = 1.0 / L;
        else alpha = (k % 2 == 0) ? (double)(ss / sy) : (double)(sy / yy);
        ++k;
    }
    info[0] = (double)k;
    info[1] = r;
    info[2] = conv;
    info[3] = L;
    free(v); free(Av); free(xn); free(gn);
}

/* Projected Gauss-Seidel on an ASSEMBLED matrix (a
 * cross-check of orc_bbpgd by a different algorithm): A in CSR (indptr[n+1],
 * indices, data), sweeps i = 0..n-1 in order,
 *   x_i <- max(0, x_i - (sum_j A_ij x_j + q_i) / A_ii),
 * stop when r = ||min(x, A x + q)||_inf <= tol after a sweep (g recomputed
 * from the final x).  Rows with A_ii <= 0 are left at 0.  For symmetric PSD
 * A with positive diagonal the sweeps converge to a solution of the LCP.
 * x: in = start (projected), out = solution; g out.
 * info[0] = sweeps, info[1] = residual, info[2] = converged. */
void orc_pgs_csr(int64_t n, const int64_t *indptr, const int32_t *indices, const double *data, const double *q,
                 double *x, double *g, double tol, int64_t max_sweeps, double *info) {
    for (int64_t i = 0; i < n; ++i) x[i] = x[i] > 0.0 ? x[i] : 0.0;
    int64_t k = 0;
    double r = INFINITY;
    while (k < max_sweeps) {
        for (int64_t i = 0; i < n; ++i) {
            long double acc = q[i];
            double aii = 0.0;
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
                acc += (long double)data[p] * x[indices[p]];
                if (indices[p] == i) aii = data[p];
            }
            if (aii <= 0.0) { x[i] = 0.0; continue; }
            double t = x[i] - (double)acc / aii;
            x[i] = t > 0.0 ? t : 0.0;
        }
        ++k;
        r = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            long double acc = q[i];
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) acc += (long double)data[p] * x[indices[p]];
            g[i] = (double)acc;
            double m = fabs(fmin(x[i], g[i]));
            if (m > r) r = m;
        }
        if (r <= tol) break;
    }
    info[0] = (double)k;
    info[1] = r;
    info[2] = r <= tol;
}
