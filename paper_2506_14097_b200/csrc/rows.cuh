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
