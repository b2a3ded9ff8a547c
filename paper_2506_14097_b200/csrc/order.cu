// Internal spatial body order for relcp_step (params.reorder; DESIGN.md §5
// "Body order").  The operator's performance depends on the body index being
// spatially coherent: K6 sums a warp's 32 consecutive bodies and gathers
// x / g at the rows of each body's lower-index neighbours, K7 gathers U_ib.
// Callers need not provide such an order (colonies grow, bodies get
// relabelled), so the step can run on an internal copy of the bodies in
// cell order and translate back at the end:
//
//   perm  internal index -> caller index: bodies sorted by (cell, caller id),
//         cells of edge ~ the mean spacing (V / N)^(1/3), row-major (x fastest)
//   inv   caller index -> internal index
//
// The step then sees a relabelled but otherwise identical problem (body
// labels are arbitrary, as constraint labels are).  Its store is
// translated back row by row: ids through perm, the row re-oriented when the
// caller's ids come out as ia > ib (n' = -n, t_a' = -t_b, t_b' = -t_a: the
// same constraint, the same Phi, q, lambda and g), and sorted by (ia, ib, gen)
// (R18).  Everything here is integer / permutation work: deterministic (the
// per-cell and per-body insertion sorts fix the order of the atomic fills).
#include "common.cuh"
#include "reduce.cuh"

__global__ void k_ord_bounds(int64_t nb, const double *__restrict__ pos, double *part, unsigned *counter,
                             double *out) {
    __shared__ double sh[6 * 32];
    double v[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
        for (int k = 0; k < 3; ++k) {
            v[k] = fmin(v[k], pos[3 * b + k]);
            v[3 + k] = fmax(v[3 + k], pos[3 * b + k]);
        }
    const int ops[6] = {2, 2, 2, 1, 1, 1};
    if (grid_reduce_last<6>(v, ops, part, counter, sh) && threadIdx.x == 0)
        for (int k = 0; k < 6; ++k) out[k] = v[k];
}

struct OrdGrid {
    int nc[3];
    double lo[3], cs[3], box[3];
};

__global__ void k_ord_cell(int64_t nb, const double *__restrict__ pos, OrdGrid G, int *__restrict__ cell,
                           int *__restrict__ count) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        int c[3];
        for (int k = 0; k < 3; ++k) {
            int v;
            if (G.box[k] > 0.0) {
                double u = pos[3 * b + k] / G.box[k];
                u -= floor(u);
                v = (int)(u * G.nc[k]);
            } else {
                v = (int)floor((pos[3 * b + k] - G.lo[k]) / G.cs[k]);
            }
            c[k] = v < 0 ? 0 : (v >= G.nc[k] ? G.nc[k] - 1 : v);
        }
        const int id = (c[2] * G.nc[1] + c[1]) * G.nc[0] + c[0];
        cell[b] = id;
        atomicAdd(count + id, 1);
    }
}

// fraction of consecutive caller indices (b, b+1) in the same or adjacent cells
__global__ void k_ord_coherence(int64_t nb, const int *__restrict__ cell, OrdGrid G, double *part, unsigned *counter,
                                double *out) {
    __shared__ double sh[32];
    double v[1] = {0.0};
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b + 1 < nb; b += (int64_t)gridDim.x * blockDim.x) {
        const int c0 = cell[b], c1 = cell[b + 1];
        const int dx = c0 % G.nc[0] - c1 % G.nc[0];
        const int dy = (c0 / G.nc[0]) % G.nc[1] - (c1 / G.nc[0]) % G.nc[1];
        const int dz = c0 / (G.nc[0] * G.nc[1]) - c1 / (G.nc[0] * G.nc[1]);
        v[0] += (abs(dx) <= 1 && abs(dy) <= 1 && abs(dz) <= 1) ? 1.0 : 0.0;
    }
    const int ops[1] = {0};
    if (grid_reduce_last<1>(v, ops, part, counter, sh) && threadIdx.x == 0) out[0] = v[0] / (double)(nb > 1 ? nb - 1 : 1);
}

__global__ void k_ord_fill(int64_t nb, const int *__restrict__ cell, const int *__restrict__ start,
                           int *__restrict__ fill, int *__restrict__ perm) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        const int c = cell[b];
        perm[start[c] + atomicAdd(fill + c, 1)] = (int)b;
    }
}

// per-segment insertion sort of int keys (segments are a few entries long)
__global__ void k_ord_sort_segments(int64_t nseg, const int *__restrict__ start, int *__restrict__ v) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nseg; c += (int64_t)gridDim.x * blockDim.x) {
        const int s = start[c], e = start[c + 1];
        for (int i = s + 1; i < e; ++i) {
            const int k = v[i];
            int j = i - 1;
            while (j >= s && v[j] > k) {
                v[j + 1] = v[j];
                --j;
            }
            v[j + 1] = k;
        }
    }
}

__global__ void k_ord_inverse(int64_t nb, const int *__restrict__ perm, int *__restrict__ inv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb; i += (int64_t)gridDim.x * blockDim.x)
        inv[perm[i]] = (int)i;
}

// *coherent (if non-null) = fraction of consecutive caller bodies in the same
// or adjacent cells; the permutation is built only when coherent is null or
// below RELCP_REORDER_COHERENT (the caller's order already follows space)
int ord_body_perm(relcp_ctx *ctx, int64_t nb, const double *pos, double *coherent) {
    cudaStream_t st = ctx->stream;
    CK(ctx->ord_perm.grow(nb));
    CK(ctx->ord_inv.grow(nb));
    CK(ctx->ord_cell.grow(nb));
    k_ord_bounds<<<grid_for(nb), RELCP_NT, 0, st>>>(nb, pos, ctx->partials.p, ctx->counter.p, ctx->red.p);
    CKL();
    CK(cudaMemcpyAsync(ctx->red_host, ctx->red.p, 6 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    OrdGrid G;
    double ext[3], emax = 0.0;
    for (int k = 0; k < 3; ++k) {
        G.box[k] = ctx->p.box[k];
        ext[k] = G.box[k] > 0.0 ? G.box[k] : ctx->red_host[3 + k] - ctx->red_host[k];
        if (!isfinite(ext[k])) return set_err(ctx, RELCP_E_NAN, "reorder: non-finite positions");
        G.lo[k] = G.box[k] > 0.0 ? 0.0 : ctx->red_host[k];
        emax = fmax(emax, ext[k]);
    }
    // cell edge ~ the mean spacing over the extended axes (a planar colony
    // is 2-D: one cell across its thickness)
    double vol = 1.0;
    int dim = 0;
    for (int k = 0; k < 3; ++k)
        if (ext[k] > 1e-9 * emax) {
            vol *= ext[k];
            ++dim;
        }
    double h = dim > 0 ? pow(vol / (double)nb, 1.0 / dim) : 1.0;
    for (;;) {
        double ncell = 1.0;
        for (int k = 0; k < 3; ++k) {
            int n = ext[k] > 1e-9 * emax ? (int)floor(ext[k] / h) : 1;
            n = n < 1 ? 1 : n;
            G.nc[k] = n;
            G.cs[k] = ext[k] > 0.0 ? ext[k] / n : 1.0;
            ncell *= n;
        }
        if (ncell <= 2.0 * (double)nb + 64.0) break;
        h *= 1.25;
    }
    const int64_t ncell = (int64_t)G.nc[0] * G.nc[1] * G.nc[2];
    CK(ctx->ord_cnt.grow(ncell + 1));
    CK(ctx->ord_start.grow(ncell + 1));
    CK(cudaMemsetAsync(ctx->ord_cnt.p, 0, sizeof(int) * (ncell + 1), st));
    k_ord_cell<<<grid_for(nb), RELCP_NT, 0, st>>>(nb, pos, G, ctx->ord_cell.p, ctx->ord_cnt.p);
    CKL();
    if (coherent) {
        k_ord_coherence<<<grid_for(nb), RELCP_NT, 0, st>>>(nb, ctx->ord_cell.p, G, ctx->partials.p, ctx->counter.p,
                                                           ctx->red.p);
        CKL();
        CK(cudaMemcpyAsync(ctx->red_host, ctx->red.p, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        *coherent = ctx->red_host[0];
        if (*coherent >= RELCP_REORDER_COHERENT) return RELCP_OK;
    }
    CKS(scan_exclusive_int(ctx, ctx->ord_cnt.p, ctx->ord_start.p, ncell + 1, nullptr));
    CK(cudaMemsetAsync(ctx->ord_cnt.p, 0, sizeof(int) * (ncell + 1), st));
    k_ord_fill<<<grid_for(nb), RELCP_NT, 0, st>>>(nb, ctx->ord_cell.p, ctx->ord_start.p, ctx->ord_cnt.p,
                                                  ctx->ord_perm.p);
    CKL();
    k_ord_sort_segments<<<grid_for(ncell, 128), 128, 0, st>>>(ncell, ctx->ord_start.p, ctx->ord_perm.p);
    CKL();
    k_ord_inverse<<<grid_for(nb), RELCP_NT, 0, st>>>(nb, ctx->ord_perm.p, ctx->ord_inv.p);
    CKL();
    return RELCP_OK;
}

// dst[i] = src[perm[i]] (gather, to internal order) or dst[perm[i]] = src[i]
// (scatter, back to the caller's order), rows of w values of T
template <typename T>
__global__ void k_ord_rows(int64_t nb, int w, const int *__restrict__ perm, const T *__restrict__ src,
                           T *__restrict__ dst, int to_caller) {
    const int64_t n = nb * w;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / w, k = e - i * w, p = perm[i];
        if (to_caller) dst[p * w + k] = src[e];
        else dst[e] = src[p * w + k];
    }
}

template <typename T>
static int ord_rows(relcp_ctx *ctx, int64_t nb, int w, const T *src, T *dst, int to_caller) {
    if (!src || !dst) return RELCP_OK;
    k_ord_rows<T><<<grid_for(nb * w), RELCP_NT, 0, ctx->stream>>>(nb, w, ctx->ord_perm.p, src, dst, to_caller);
    CKL();
    return RELCP_OK;
}

int ord_bodies_in(relcp_ctx *ctx, const relcp_bodies *b, const double *f_ext, relcp_bodies *bi,
                  const double **f_ext_i) {
    const int64_t nb = b->n;
    *bi = *b;
    CK(ctx->ob_pos.grow(3 * nb));
    CK(ctx->ob_quat.grow(4 * nb));
    CK(ctx->ob_axes.grow(3 * nb));
    bi->pos = ctx->ob_pos.p;
    bi->quat = ctx->ob_quat.p;
    bi->axes = ctx->ob_axes.p;
    CKS(ord_rows(ctx, nb, 3, b->pos, bi->pos, 0));
    CKS(ord_rows(ctx, nb, 4, b->quat, bi->quat, 0));
    CKS(ord_rows(ctx, nb, 3, b->axes, ctx->ob_axes.p, 0));
    if (b->vel) {
        CK(ctx->ob_vel.grow(6 * nb));
        bi->vel = ctx->ob_vel.p;
        CKS(ord_rows(ctx, nb, 6, b->vel, bi->vel, 0));
    }
    if (b->inv_mass) {
        CK(ctx->ob_im.grow(nb));
        bi->inv_mass = ctx->ob_im.p;
        CKS(ord_rows(ctx, nb, 1, b->inv_mass, ctx->ob_im.p, 0));
    }
    if (b->inv_inertia) {
        CK(ctx->ob_ii.grow(3 * nb));
        bi->inv_inertia = ctx->ob_ii.p;
        CKS(ord_rows(ctx, nb, 3, b->inv_inertia, ctx->ob_ii.p, 0));
    }
    if (b->kinematic) {
        CK(ctx->ob_kin.grow(nb));
        bi->kinematic = ctx->ob_kin.p;
        CKS(ord_rows(ctx, nb, 1, b->kinematic, ctx->ob_kin.p, 0));
    }
    if (b->shape) {
        CK(ctx->ob_shape.grow(nb));
        bi->shape = ctx->ob_shape.p;
        CKS(ord_rows(ctx, nb, 1, b->shape, ctx->ob_shape.p, 0));
    }
    *f_ext_i = nullptr;
    if (f_ext) {
        CK(ctx->ob_fext.grow(6 * nb));
        CKS(ord_rows(ctx, nb, 6, f_ext, ctx->ob_fext.p, 0));
        *f_ext_i = ctx->ob_fext.p;
    }
    return RELCP_OK;
}

int ord_bodies_out(relcp_ctx *ctx, const relcp_bodies *bi, relcp_bodies *b) {
    const int64_t nb = b->n;
    CKS(ord_rows(ctx, nb, 3, (const double *)bi->pos, b->pos, 1));
    CKS(ord_rows(ctx, nb, 4, (const double *)bi->quat, b->quat, 1));
    if (b->vel) CKS(ord_rows(ctx, nb, 6, (const double *)bi->vel, b->vel, 1));
    return RELCP_OK;
}

// the internal store (same capacity as the caller's)
int ord_store(relcp_ctx *ctx, const relcp_constraints *cs, relcp_constraints *ci) {
    const int64_t cap = cs->capacity > 0 ? cs->capacity : 1;
    CK(ctx->os_i.grow(3 * cap));
    CK(ctx->os_d.grow(13 * cap));
    *ci = *cs;
    ci->count = 0;
    ci->ia = ctx->os_i.p;
    ci->ib = ctx->os_i.p + cap;
    ci->gen = ctx->os_i.p + 2 * cap;
    double *d = ctx->os_d.p;
    ci->n = d;
    ci->ta = d + 3 * cap;
    ci->tb = d + 6 * cap;
    ci->phi = d + 9 * cap;
    ci->q = d + 10 * cap;
    ci->lambda = d + 11 * cap;
    ci->g = d + 12 * cap;
    return RELCP_OK;
}

// internal row r -> caller key (a = min, b = max of the caller ids), flip flag
__global__ void k_ord_keys(int64_t m, const int *__restrict__ perm, const int32_t *__restrict__ ia,
                           const int32_t *__restrict__ ib, int *__restrict__ ka, int *__restrict__ kb,
                           int *__restrict__ count) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
        const int i = perm[ia[r]], j = perm[ib[r]];
        const int a = i < j ? i : j;
        ka[r] = a;
        kb[r] = i < j ? j : ~i;  // the larger id; ~ marks a re-oriented row (ids >= 0)
        atomicAdd(count + a, 1);
    }
}

__global__ void k_ord_slots(int64_t m, const int *__restrict__ ka, const int *__restrict__ start,
                            int *__restrict__ fill, int *__restrict__ order) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
        const int a = ka[r];
        order[start[a] + atomicAdd(fill + a, 1)] = (int)r;
    }
}

// per caller body a: sort its rows by (b, gen) -- unique keys, so the order is
// deterministic whatever order the atomic fill left
__global__ void k_ord_sort_rows(int64_t nb, const int *__restrict__ start, const int *__restrict__ kb,
                                const int32_t *__restrict__ gen, int *__restrict__ order) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nb; a += (int64_t)gridDim.x * blockDim.x) {
        const int s = start[a], e = start[a + 1];
        auto key = [&](int r) {
            const int b = kb[r] < 0 ? ~kb[r] : kb[r];
            return ((long long)b << 32) | (unsigned)gen[r];
        };
        for (int i = s + 1; i < e; ++i) {
            const int r = order[i];
            const long long k = key(r);
            int j = i - 1;
            while (j >= s && key(order[j]) > k) {
                order[j + 1] = order[j];
                --j;
            }
            order[j + 1] = r;
        }
    }
}

__global__ void k_ord_write(int64_t m, const int *__restrict__ order, const int *__restrict__ ka,
                            const int *__restrict__ kb, const int64_t ci_cap, const int32_t *__restrict__ gen,
                            const double *__restrict__ n, const double *__restrict__ ta,
                            const double *__restrict__ tb, const double *__restrict__ phi,
                            const double *__restrict__ q, const double *__restrict__ lam,
                            const double *__restrict__ g, int64_t cap, int32_t *__restrict__ oia,
                            int32_t *__restrict__ oib, int32_t *__restrict__ ogen, double *__restrict__ on,
                            double *__restrict__ ota, double *__restrict__ otb, double *__restrict__ ophi,
                            double *__restrict__ oq, double *__restrict__ olam, double *__restrict__ og) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m; s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = order[s];
        const bool flip = kb[r] < 0;
        oia[s] = ka[r];
        oib[s] = flip ? ~kb[r] : kb[r];
        ogen[s] = gen[r];
        for (int k = 0; k < 3; ++k) {
            const double nv = n[k * ci_cap + r], av = ta[k * ci_cap + r], bv = tb[k * ci_cap + r];
            on[k * cap + s] = flip ? -nv : nv;
            ota[k * cap + s] = flip ? -bv : av;
            otb[k * cap + s] = flip ? -av : bv;
        }
        ophi[s] = phi[r];
        oq[s] = q[r];
        olam[s] = lam[r];
        if (og) og[s] = g[r];
    }
}

int ord_store_out(relcp_ctx *ctx, int64_t nb, const relcp_constraints *ci, relcp_constraints *cs) {
    const int64_t m = ci->count;
    cs->count = m;
    if (m > cs->capacity) return RELCP_OK;  // the caller reports E_CAPACITY with the needed count
    if (m == 0) return RELCP_OK;
    cudaStream_t st = ctx->stream;
    CK(ctx->ord_key.grow(3 * m));
    CK(ctx->ord_cnt.grow(nb + 1));
    CK(ctx->ord_start.grow(nb + 1));
    int *ka = ctx->ord_key.p, *kb = ka + m, *order = ka + 2 * m;
    CK(cudaMemsetAsync(ctx->ord_cnt.p, 0, sizeof(int) * (nb + 1), st));
    k_ord_keys<<<grid_for(m), RELCP_NT, 0, st>>>(m, ctx->ord_perm.p, ci->ia, ci->ib, ka, kb, ctx->ord_cnt.p);
    CKL();
    CKS(scan_exclusive_int(ctx, ctx->ord_cnt.p, ctx->ord_start.p, nb + 1, nullptr));
    CK(cudaMemsetAsync(ctx->ord_cnt.p, 0, sizeof(int) * (nb + 1), st));
    k_ord_slots<<<grid_for(m), RELCP_NT, 0, st>>>(m, ka, ctx->ord_start.p, ctx->ord_cnt.p, order);
    CKL();
    k_ord_sort_rows<<<grid_for(nb, 128), 128, 0, st>>>(nb, ctx->ord_start.p, kb, ci->gen, order);
    CKL();
    k_ord_write<<<grid_for(m), RELCP_NT, 0, st>>>(m, order, ka, kb, ci->capacity, ci->gen, ci->n, ci->ta, ci->tb,
                                                  ci->phi, ci->q, ci->lambda, ci->g, cs->capacity, cs->ia, cs->ib,
                                                  cs->gen, cs->n, cs->ta, cs->tb, cs->phi, cs->q, cs->lambda, cs->g);
    CKL();
    return RELCP_OK;
}

// pairs (device) in internal ids -> caller ids, oriented i < j
__global__ void k_ord_pairs(int64_t np, const int *__restrict__ perm, const int *__restrict__ pi,
                            const int *__restrict__ pj, int32_t *__restrict__ oi, int32_t *__restrict__ oj) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np; p += (int64_t)gridDim.x * blockDim.x) {
        const int i = perm[pi[p]], j = perm[pj[p]];
        oi[p] = i < j ? i : j;
        oj[p] = i < j ? j : i;
    }
}

int ord_pairs_out(relcp_ctx *ctx, int64_t np, int32_t *oi, int32_t *oj) {
    if (np == 0) return RELCP_OK;
    k_ord_pairs<<<grid_for(np), RELCP_NT, 0, ctx->stream>>>(np, ctx->ord_perm.p, ctx->pi.p, ctx->pj.p, oi, oj);
    CKL();
    return RELCP_OK;
}
