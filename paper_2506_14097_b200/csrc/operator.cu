// The Delassus operator A = s D^T W D, matrix-free.
//
//   column alpha of D (P:L154-157 Eq. collision_ft; P:L174 F = D gamma):
//       wrench -[n; t_a] on body ia, +[n; t_b] on body ib
//   row alpha of D^T (Phi_dot = n.(ydot_b - ydot_a)):
//       [-n, -t_a, n, t_b]
//   W_b = M_b^{-1} or local-drag mobility
//
// B200 layout:
//   * scatter F = D x is a body-major CSR pass: each body owns a contiguous
//     segment of signed 6-double wrench payloads (built once per operator,
//     sorted by (constraint, side) so the per-body sum has a fixed order);
//     a G-lane group of one warp reduces a body's segment with shuffles, then
//     six lanes apply W_b and store U_b.  No floating-point atomics.
//   * gather y = s D^T U is a constraint-major streaming pass over the SoA
//     store (coalesced n / t_a / t_b planes) with U_a, U_b read from L2.
#include "common.cuh"
#include "reduce.cuh"

// ------------------------------------------------------------ W blocks
__global__ void k_build_W(int64_t nb, int dyn, double xi, const double *__restrict__ quat,
                          const double *__restrict__ axes, const double *__restrict__ inv_mass,
                          const double *__restrict__ inv_inertia, const int32_t *__restrict__ kin,
                          double *__restrict__ W) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        double w[7];
        if (dyn == RELCP_INERTIAL) {
            double s = quat[4 * b], x = quat[4 * b + 1], y = quat[4 * b + 2], z = quat[4 * b + 3];
            double inv = 1.0 / sqrt(s * s + x * x + y * y + z * z);
            s *= inv; x *= inv; y *= inv; z *= inv;
            double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - s * z), 2 * (x * z + s * y)},
                              {2 * (x * y + s * z), 1 - 2 * (x * x + z * z), 2 * (y * z - s * x)},
                              {2 * (x * z - s * y), 2 * (y * z + s * x), 1 - 2 * (x * x + y * y)}};
            double d0 = inv_inertia[3 * b], d1 = inv_inertia[3 * b + 1], d2 = inv_inertia[3 * b + 2];
            auto S = [&](int i, int j) { return R[i][0] * d0 * R[j][0] + R[i][1] * d1 * R[j][1] + R[i][2] * d2 * R[j][2]; };
            w[0] = inv_mass[b];
            w[1] = S(0, 0); w[2] = S(0, 1); w[3] = S(0, 2);
            w[4] = S(1, 1); w[5] = S(1, 2); w[6] = S(2, 2);
        } else {
            double L = 2.0 * fmax(axes[3 * b], fmax(axes[3 * b + 1], axes[3 * b + 2]));
            double r = 12.0 / (xi * L * L * L);
            w[0] = 1.0 / (xi * L);
            w[1] = r; w[2] = 0.0; w[3] = 0.0; w[4] = r; w[5] = 0.0; w[6] = r;
        }
        bool k = kin && kin[b] != 0;
#pragma unroll
        for (int i = 0; i < 7; ++i) W[RELCP_WSTRIDE * b + i] = k ? 0.0 : w[i];
        W[RELCP_WSTRIDE * b + 7] = 0.0;
    }
}

int op_build_W(relcp_ctx *ctx, const relcp_bodies *b, double *W) {
    if (ctx->p.dynamics == RELCP_INERTIAL && (!b->inv_mass || !b->inv_inertia || !b->quat))
        return set_err(ctx, RELCP_E_ARG, "inertial dynamics needs quat, inv_mass and inv_inertia");
    if (ctx->p.dynamics == RELCP_OVERDAMPED && !b->axes)
        return set_err(ctx, RELCP_E_ARG, "overdamped dynamics needs axes");
    k_build_W<<<grid_for(b->n), RELCP_NT, 0, ctx->stream>>>(b->n, ctx->p.dynamics, ctx->p.xi, b->quat, b->axes,
                                                            b->inv_mass, b->inv_inertia, b->kinematic, W);
    CKL();
    return RELCP_OK;
}

// ------------------------------------------------------------ CSR of D
__global__ void k_degree(int64_t nc, const int32_t *__restrict__ ia, const int32_t *__restrict__ ib, int *deg,
                         int64_t nb, int *bad) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nc; a += (int64_t)gridDim.x * blockDim.x) {
        int i = ia[a], j = ib[a];
        if (i < 0 || j < 0 || i >= nb || j >= nb || i == j) { atomicExch(bad, 1); continue; }
        atomicAdd(deg + i, 1);
        atomicAdd(deg + j, 1);
    }
}

__global__ void k_fill_slots(int64_t nc, const int32_t *__restrict__ ia, const int32_t *__restrict__ ib,
                             const int *__restrict__ row_ptr, int *fill, int *ekey) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nc; a += (int64_t)gridDim.x * blockDim.x) {
        int i = ia[a], j = ib[a];
        int si = row_ptr[i] + atomicAdd(fill + i, 1);
        int sj = row_ptr[j] + atomicAdd(fill + j, 1);
        ekey[si] = (int)(2 * a);      // side a
        ekey[sj] = (int)(2 * a + 1);  // side b
    }
}

// Sort each body segment by key (constraint, side): fixes the summation order.
__global__ void k_sort_segments(int64_t nb, const int *__restrict__ row_ptr, int *ekey) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        int s = row_ptr[b], e = row_ptr[b + 1];
        for (int i = s + 1; i < e; ++i) {
            int k = ekey[i];
            int j = i - 1;
            while (j >= s && ekey[j] > k) { ekey[j + 1] = ekey[j]; --j; }
            ekey[j + 1] = k;
        }
    }
}

__global__ void k_payload(int64_t E, int64_t cap, const double *__restrict__ n, const double *__restrict__ ta,
                          const double *__restrict__ tb, int *ekey, double *__restrict__ ew) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
        int key = ekey[e];
        int64_t a = key >> 1;
        bool side_b = key & 1;
        double sg = side_b ? 1.0 : -1.0;
        const double *t = side_b ? tb : ta;
        ew[0 * E + e] = sg * n[a];
        ew[1 * E + e] = sg * n[cap + a];
        ew[2 * E + e] = sg * n[2 * cap + a];
        ew[3 * E + e] = sg * t[a];
        ew[4 * E + e] = sg * t[cap + a];
        ew[5 * E + e] = sg * t[2 * cap + a];
        ekey[e] = (int)a;
    }
}

int op_prepare(relcp_ctx *ctx, const relcp_bodies *b, const relcp_constraints *cs) {
    if (!b || !cs || b->n <= 0) return set_err(ctx, RELCP_E_ARG, "prepare: empty bodies");
    const int64_t nb = b->n, nc = cs->count, E = 2 * nc;
    if (nc < 0 || nc > cs->capacity) return set_err(ctx, RELCP_E_ARG, "prepare: count %lld > capacity", (long long)nc);
    if (nc >= (1ll << 30)) return set_err(ctx, RELCP_E_ARG, "prepare: more than 2^30 constraints");
    CK(ctx->W.grow(RELCP_WSTRIDE * nb));
    CK(ctx->row_ptr.grow(nb + 1));
    CK(ctx->deg.grow(nb + 1));
    CK(ctx->fill.grow(nb + 1));
    CK(ctx->U.grow(6 * nb));
    CK(ctx->ecid.grow(E > 0 ? E : 1));
    CK(ctx->ew.grow(6 * (E > 0 ? E : 1)));
    CKS(op_build_W(ctx, b, ctx->W.p));
    CK(cudaMemsetAsync(ctx->deg.p, 0, sizeof(int) * (nb + 1), ctx->stream));
    CK(cudaMemsetAsync(ctx->fill.p, 0, sizeof(int) * (nb + 1), ctx->stream));  // fill[nb] = bad flag
    if (nc > 0) {
        k_degree<<<grid_for(nc), RELCP_NT, 0, ctx->stream>>>(nc, cs->ia, cs->ib, ctx->deg.p, nb, ctx->fill.p + nb);
        CKL();
    }
    int total = 0;
    CKS(scan_exclusive_int(ctx, ctx->deg.p, ctx->row_ptr.p, nb + 1, &total));  // deg[nb] = 0
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, ctx->fill.p + nb, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (bad) return set_err(ctx, RELCP_E_ARG, "prepare: body index out of range or ia == ib");
    if (nc > 0) {
        CK(cudaMemsetAsync(ctx->fill.p, 0, sizeof(int) * nb, ctx->stream));
        k_fill_slots<<<grid_for(nc), RELCP_NT, 0, ctx->stream>>>(nc, cs->ia, cs->ib, ctx->row_ptr.p, ctx->fill.p,
                                                                 ctx->ecid.p);
        CKL();
        k_sort_segments<<<grid_for(nb, 128), 128, 0, ctx->stream>>>(nb, ctx->row_ptr.p, ctx->ecid.p);
        CKL();
        k_payload<<<grid_for(E), RELCP_NT, 0, ctx->stream>>>(E, cs->capacity, cs->n, cs->ta, cs->tb, ctx->ecid.p,
                                                             ctx->ew.p);
        CKL();
    }
    ctx->op_nc = nc;
    ctx->op_nb = nb;
    ctx->op_key_ia = cs->ia;
    return RELCP_OK;
}

// ------------------------------------------------------------ scatter
// U_b = W_b sum_{e in seg(b)} w_e * xeff(cid_e), xeff = proj ? max(0, x - alpha g) : x,
// scaled by *xscale if given.  G lanes per body.
template <int G, bool PROJ>
__global__ void __launch_bounds__(RELCP_NT) k_scatter(int64_t nb, int64_t E, const int *__restrict__ row_ptr,
                                                      const int *__restrict__ ecid, const double *__restrict__ ew,
                                                      const double *__restrict__ x, const double *__restrict__ g,
                                                      const LcpState *__restrict__ st,
                                                      const double *__restrict__ xscale,
                                                      const double *__restrict__ W, double *__restrict__ U,
                                                      double *__restrict__ Fout) {
    constexpr int BPW = 32 / G;
    double alpha = 0.0;
    if (PROJ) {
        if (st->done) return;
        alpha = st->alpha;
    }
    const double sc = xscale ? *xscale : 1.0;
    const int lane = threadIdx.x & 31, lg = lane % G, grp = lane / G;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * BPW; base < nb; base += nwarp * BPW) {
        const int64_t b = base + grp;
        const bool valid = b < nb;
        double f0 = 0, f1 = 0, f2 = 0, f3 = 0, f4 = 0, f5 = 0;
        if (valid) {
            const int s = row_ptr[b], e1 = row_ptr[b + 1];
            for (int e = s + lg; e < e1; e += G) {
                const int c = ecid[e];
                double xv = x[c];
                if (PROJ) xv = fmax(0.0, xv - alpha * g[c]);
                xv *= sc;
                f0 = fma(ew[e], xv, f0);
                f1 = fma(ew[E + e], xv, f1);
                f2 = fma(ew[2 * E + e], xv, f2);
                f3 = fma(ew[3 * E + e], xv, f3);
                f4 = fma(ew[4 * E + e], xv, f4);
                f5 = fma(ew[5 * E + e], xv, f5);
            }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            f0 += __shfl_down_sync(0xffffffffu, f0, o, G);
            f1 += __shfl_down_sync(0xffffffffu, f1, o, G);
            f2 += __shfl_down_sync(0xffffffffu, f2, o, G);
            f3 += __shfl_down_sync(0xffffffffu, f3, o, G);
            f4 += __shfl_down_sync(0xffffffffu, f4, o, G);
            f5 += __shfl_down_sync(0xffffffffu, f5, o, G);
        }
        // broadcast the group's lane-0 totals (one association for all lanes)
        const int src = grp * G;
        f0 = __shfl_sync(0xffffffffu, f0, src);
        f1 = __shfl_sync(0xffffffffu, f1, src);
        f2 = __shfl_sync(0xffffffffu, f2, src);
        f3 = __shfl_sync(0xffffffffu, f3, src);
        f4 = __shfl_sync(0xffffffffu, f4, src);
        f5 = __shfl_sync(0xffffffffu, f5, src);
        if (valid && lg < 6) {
            const double *w = W + RELCP_WSTRIDE * b;
            double u;
            if (lg < 3) {
                u = w[0] * (lg == 0 ? f0 : (lg == 1 ? f1 : f2));
            } else if (lg == 3) {
                u = w[1] * f3 + w[2] * f4 + w[3] * f5;
            } else if (lg == 4) {
                u = w[2] * f3 + w[4] * f4 + w[5] * f5;
            } else {
                u = w[3] * f3 + w[5] * f4 + w[6] * f5;
            }
            U[6 * b + lg] = u;
            if (Fout) {
                double fv = lg == 0 ? f0 : lg == 1 ? f1 : lg == 2 ? f2 : lg == 3 ? f3 : lg == 4 ? f4 : f5;
                Fout[6 * b + lg] = fv;
            }
        }
    }
}

static int scatter_group(const relcp_ctx *ctx) {
    // mean half-entries per body decides the group width
    double mean = ctx->op_nb > 0 ? 2.0 * (double)ctx->op_nc / (double)ctx->op_nb : 0.0;
    return mean > 24.0 ? 32 : (mean > 10.0 ? 16 : 8);
}

template <bool PROJ>
static void launch_scatter(relcp_ctx *ctx, int G, int64_t nb, const double *x, const double *g,
                           const double *xscale, double *U, double *F) {
    const int64_t E = 2 * ctx->op_nc;
    int64_t threads = nb * G;
    int grid = grid_for(threads, RELCP_NT, 16);
    const LcpState *st = ctx->st.p;
    if (G == 8)
        k_scatter<8, PROJ><<<grid, RELCP_NT, 0, ctx->stream>>>(nb, E, ctx->row_ptr.p, ctx->ecid.p, ctx->ew.p, x, g, st,
                                                              xscale, ctx->W.p, U, F);
    else if (G == 16)
        k_scatter<16, PROJ><<<grid, RELCP_NT, 0, ctx->stream>>>(nb, E, ctx->row_ptr.p, ctx->ecid.p, ctx->ew.p, x, g, st,
                                                               xscale, ctx->W.p, U, F);
    else
        k_scatter<32, PROJ><<<grid, RELCP_NT, 0, ctx->stream>>>(nb, E, ctx->row_ptr.p, ctx->ecid.p, ctx->ew.p, x, g, st,
                                                               xscale, ctx->W.p, U, F);
}

int op_scatter(relcp_ctx *ctx, int64_t nb, const double *x, const double *g, int proj, const double *xscale_dev,
               double *U, double *F) {
    int G = scatter_group(ctx);
    if (proj)
        launch_scatter<true>(ctx, G, nb, x, g, xscale_dev, U, F);
    else
        launch_scatter<false>(ctx, G, nb, x, g, xscale_dev, U, F);
    CKL();
    return RELCP_OK;
}

// ------------------------------------------------------------ gather
__device__ __forceinline__ double row_dot(int64_t a, int64_t cap, const int32_t *__restrict__ ia,
                                          const int32_t *__restrict__ ib, const double *__restrict__ n,
                                          const double *__restrict__ ta, const double *__restrict__ tb,
                                          const double *__restrict__ U) {
    const int i = ia[a], j = ib[a];
    const double nx = n[a], ny = n[cap + a], nz = n[2 * cap + a];
    const double *ua = U + 6 * (int64_t)i, *ub = U + 6 * (int64_t)j;
    double v = nx * (ub[0] - ua[0]) + ny * (ub[1] - ua[1]) + nz * (ub[2] - ua[2]);
    v -= ta[a] * ua[3] + ta[cap + a] * ua[4] + ta[2 * cap + a] * ua[5];
    v += tb[a] * ub[3] + tb[cap + a] * ub[4] + tb[2 * cap + a] * ub[5];
    return v;
}

// y = scale * D^T U ; optionally the grid-wide ||y||^2 -> st->pnorm = 1/||y||, st->L = ||y||
__global__ void __launch_bounds__(RELCP_NT) k_gather(int64_t nc, int64_t cap, const int32_t *__restrict__ ia,
                                                     const int32_t *__restrict__ ib, const double *__restrict__ n,
                                                     const double *__restrict__ ta, const double *__restrict__ tb,
                                                     const double *__restrict__ U, double scale,
                                                     double *__restrict__ y, int norm2, double *part,
                                                     unsigned *counter, LcpState *st) {
    __shared__ double sh[32];
    double acc[1] = {0.0};
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nc; a += (int64_t)gridDim.x * blockDim.x) {
        double v = scale * row_dot(a, cap, ia, ib, n, ta, tb, U);
        y[a] = v;
        acc[0] = fma(v, v, acc[0]);
    }
    if (!norm2) return;
    const int ops[1] = {0};
    if (grid_reduce_last<1>(acc, ops, part, counter, sh) && threadIdx.x == 0) {
        double nrm = sqrt(acc[0]);
        st->L = nrm;
        st->pnorm = nrm > 0.0 ? 1.0 / nrm : 0.0;
    }
}

int op_gather_apply(relcp_ctx *ctx, const relcp_constraints *cs, const double *U, double *y, double scale,
                    int norm2) {
    const int64_t nc = cs->count;
    if (nc == 0) return RELCP_OK;
    int grid = grid_for(nc, RELCP_NT, 8);
    k_gather<<<grid, RELCP_NT, 0, ctx->stream>>>(nc, cs->capacity, cs->ia, cs->ib, cs->n, cs->ta, cs->tb, U, scale, y,
                                                 norm2, ctx->partials.p, ctx->counter.p, ctx->st.p);
    CKL();
    return RELCP_OK;
}

// out[a] += coef * row_a . [U_ia; U_ib] for a in [begin, end)
__global__ void k_row_dot_add(int64_t begin, int64_t end, int64_t cap, const int32_t *__restrict__ ia,
                              const int32_t *__restrict__ ib, const double *__restrict__ n,
                              const double *__restrict__ ta, const double *__restrict__ tb,
                              const double *__restrict__ U, double coef, double *out) {
    for (int64_t a = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < end;
         a += (int64_t)gridDim.x * blockDim.x)
        out[a] += coef * row_dot(a, cap, ia, ib, n, ta, tb, U);
}

int op_row_dot_U(relcp_ctx *ctx, const relcp_constraints *cs, int64_t begin, int64_t end, const double *U,
                 double coef, double *out_add) {
    if (end <= begin) return RELCP_OK;
    k_row_dot_add<<<grid_for(end - begin), RELCP_NT, 0, ctx->stream>>>(begin, end, cs->capacity, cs->ia, cs->ib, cs->n,
                                                                       cs->ta, cs->tb, U, coef, out_add);
    CKL();
    return RELCP_OK;
}
