// Row of D^T applied to body velocities (Phi_dot = n.(ydot_b - ydot_a),
// P:L207-211):  row_a . [U_ia; U_ib] = -n.u_a - t_a.w_a + n.u_b + t_b.w_b.
// U is AoS (nb, 6) fp64; each 48-byte row is 16-byte aligned and is read as
// three 128-bit loads (LDG.128) instead of six 64-bit ones.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ void load_u6(const double *__restrict__ U, int64_t b, double (&u)[6]) {
    const double2 *p = reinterpret_cast<const double2 *>(U + 6 * b);
    const double2 a = p[0], c = p[1], d = p[2];
    u[0] = a.x; u[1] = a.y; u[2] = c.x; u[3] = c.y; u[4] = d.x; u[5] = d.y;
}

__device__ __forceinline__ double row_dot_u(int64_t a, int64_t cap, const int32_t *__restrict__ ia,
                                            const int32_t *__restrict__ ib, const double *__restrict__ n,
                                            const double *__restrict__ ta, const double *__restrict__ tb,
                                            const double *__restrict__ U) {
    const int i = ia[a], j = ib[a];
    const double nx = n[a], ny = n[cap + a], nz = n[2 * cap + a];
    const double tax = ta[a], tay = ta[cap + a], taz = ta[2 * cap + a];
    const double tbx = tb[a], tby = tb[cap + a], tbz = tb[2 * cap + a];
    double ua[6], ub[6];
    load_u6(U, i, ua);
    load_u6(U, j, ub);
    double v = nx * (ub[0] - ua[0]) + ny * (ub[1] - ua[1]) + nz * (ub[2] - ua[2]);
    v -= tax * ua[3] + tay * ua[4] + taz * ua[5];
    v += tbx * ub[3] + tby * ub[4] + tbz * ub[5];
    return v;
}

// ---- compact rows: the row's 9 fp64 (n, t_a, t_b) in 6 (built by op_prepare,
// operator.cu k_compact; read by K6, K7 and every other operator pass).
//   n   : octahedral (u, v); decoded by folding the lower hemisphere and
//         normalising (error ~1 ulp).
//   t_a, t_b: t = r x n is orthogonal to n, so with k = argmax_i |n'_i| of the
//         DECODED normal n' only t_j1, t_j2 are stored (j1 = (k+1) % 3,
//         j2 = (k+2) % 3) and t_k = -(t_j1 n'_j1 + t_j2 n'_j2) / n'_k, where
//         |n'_k| >= 1/sqrt(3) keeps it well conditioned (error ~ulp * |r|).
// Planes (stride rs): 0 u, 1 v, 2 t_a,j1, 3 t_a,j2, 4 t_b,j1, 5 t_b,j2.
// 48 + 8 (ids) = 56 bytes per row pass instead of 80.
struct CNormal {
    double n[3];    // decoded unit normal n'
    double n1, n2;  // n'_j1, n'_j2
    double irk;     // -1 / n'_k
    int k;
};

__device__ __forceinline__ CNormal cn_decode(double u, double v) {
    CNormal c;
    const double z = 1.0 - fabs(u) - fabs(v);
    const double t = fmax(-z, 0.0);
    const double x = u >= 0.0 ? u - t : u + t;
    const double y = v >= 0.0 ? v - t : v + t;
    const double r = rsqrt(fma(x, x, fma(y, y, z * z)));
    c.n[0] = x * r;
    c.n[1] = y * r;
    c.n[2] = z * r;
    const double ax = fabs(c.n[0]), ay = fabs(c.n[1]), az = fabs(c.n[2]);
    c.k = (ax >= ay && ax >= az) ? 0 : (ay >= az ? 1 : 2);
    c.n1 = c.k == 0 ? c.n[1] : (c.k == 1 ? c.n[2] : c.n[0]);
    c.n2 = c.k == 0 ? c.n[2] : (c.k == 1 ? c.n[0] : c.n[1]);
    c.irk = -1.0 / (c.k == 0 ? c.n[0] : (c.k == 1 ? c.n[1] : c.n[2]));
    return c;
}

__device__ __forceinline__ void t_expand(const CNormal &c, double a1, double a2, double (&t)[3]) {
    const double tk = fma(a1, c.n1, a2 * c.n2) * c.irk;
    t[0] = c.k == 0 ? tk : (c.k == 1 ? a2 : a1);
    t[1] = c.k == 0 ? a1 : (c.k == 1 ? tk : a2);
    t[2] = c.k == 0 ? a2 : (c.k == 1 ? a1 : tk);
}

// the two stored components (t_j1, t_j2) of t for the decoded normal c
__device__ __forceinline__ void t_pick(const CNormal &c, const double (&t)[3], double &a1, double &a2) {
    a1 = c.k == 0 ? t[1] : (c.k == 1 ? t[2] : t[0]);
    a2 = c.k == 0 ? t[2] : (c.k == 1 ? t[0] : t[1]);
}

__device__ __forceinline__ void oct_encode(double nx, double ny, double nz, double &u, double &v) {
    const double s = 1.0 / (fabs(nx) + fabs(ny) + fabs(nz));
    const double px = nx * s, py = ny * s, pz = nz * s;
    if (pz < 0.0) {
        u = (1.0 - fabs(py)) * (px >= 0.0 ? 1.0 : -1.0);
        v = (1.0 - fabs(px)) * (py >= 0.0 ? 1.0 : -1.0);
    } else {
        u = px;
        v = py;
    }
}

// row_a . [U_ia; U_ib] from the compact planes
__device__ __forceinline__ double row_dot_c(int64_t a, int64_t rs, const int32_t *__restrict__ ia,
                                            const int32_t *__restrict__ ib, const double *__restrict__ rc,
                                            const double *__restrict__ U) {
    const int i = ia[a], j = ib[a];
    const double u = rc[a], v = rc[rs + a];
    const double a1 = rc[2 * rs + a], a2 = rc[3 * rs + a], b1 = rc[4 * rs + a], b2 = rc[5 * rs + a];
    double ua[6], ub[6];
    load_u6(U, i, ua);
    load_u6(U, j, ub);
    const CNormal c = cn_decode(u, v);
    double ta[3], tb[3];
    t_expand(c, a1, a2, ta);
    t_expand(c, b1, b2, tb);
    double r = c.n[0] * (ub[0] - ua[0]) + c.n[1] * (ub[1] - ua[1]) + c.n[2] * (ub[2] - ua[2]);
    r -= ta[0] * ua[3] + ta[1] * ua[4] + ta[2] * ua[5];
    r += tb[0] * ub[3] + tb[1] * ub[4] + tb[2] * ub[5];
    return r;
}
