// Constraint-store maintenance: keep the store sorted by (ia, ib, gen).
//
// Constraint order is a labeling ("without loss of generality"); the
// library keeps rows sorted by (ia, ib, gen) (R18) so that the rows
// whose a-side body is b form one contiguous run: K6 then reads them straight
// from the store (coalesced) and only b-side entries go through the CSR.
// Augmentation appends Delta A_n sorted by (ia, ib) behind the sorted old
// rows; k_merge is the stable merge of the two runs (old before new on equal
// (ia, ib): smaller gen first).  Retained rows keep every field, so the
// q-retention identity and the warm start iota(lambda) move with them.
#include "common.cuh"

__device__ __forceinline__ long long row_key(const int32_t *ia, const int32_t *ib, int64_t r) {
    return ((long long)ia[r] << 32) | (unsigned)ib[r];
}

// number of rows in [lo, hi) with key < k (strict) or <= k (!strict); sorted range
__device__ __forceinline__ int64_t rank_in(const int32_t *ia, const int32_t *ib, int64_t lo, int64_t hi, long long k,
                                           bool strict) {
    int64_t a = lo, b = hi;
    while (a < b) {
        const int64_t m = (a + b) >> 1;
        const long long km = row_key(ia, ib, m);
        if (strict ? (km < k) : (km <= k)) a = m + 1; else b = m;
    }
    return a - lo;
}

__global__ void k_merge(int64_t n_old, int64_t total, int64_t cap, const int32_t *__restrict__ ia,
                        const int32_t *__restrict__ ib, const int32_t *__restrict__ gen, const double *__restrict__ n,
                        const double *__restrict__ ta, const double *__restrict__ tb, const double *__restrict__ phi,
                        const double *__restrict__ q, const double *__restrict__ lam, const double *__restrict__ g,
                        int32_t *__restrict__ ti, double *__restrict__ td) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < total; r += (int64_t)gridDim.x * blockDim.x) {
        const long long k = row_key(ia, ib, r);
        int64_t dest;
        if (r < n_old)
            dest = r + rank_in(ia, ib, n_old, total, k, true);  // new rows strictly before
        else
            dest = (r - n_old) + rank_in(ia, ib, 0, n_old, k, false);  // old rows <= before
        ti[dest] = ia[r];
        ti[total + dest] = ib[r];
        ti[2 * total + dest] = gen[r];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            td[(0 + c) * total + dest] = n[c * cap + r];
            td[(3 + c) * total + dest] = ta[c * cap + r];
            td[(6 + c) * total + dest] = tb[c * cap + r];
        }
        td[9 * total + dest] = phi[r];
        td[10 * total + dest] = q[r];
        td[11 * total + dest] = lam[r];
        td[12 * total + dest] = g ? g[r] : 0.0;
    }
}

// bad[0] = 1 if a (ia, ib) key decreases inside [0, n_old) or inside
// [n_old, total) (the two runs the merge assumes sorted)
__global__ void k_check_runs(int64_t n_old, int64_t total, const int32_t *__restrict__ ia,
                             const int32_t *__restrict__ ib, int *bad) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a + 1 < total;
         a += (int64_t)gridDim.x * blockDim.x)
        if (a + 1 != n_old && row_key(ia, ib, a) > row_key(ia, ib, a + 1)) *bad = 1;
}

// Merge rows [n_old, n_old + m) (sorted) into the sorted rows [0, n_old).
// A store whose runs are not (ia, ib)-sorted (a caller's own order, e.g. rows
// loaded or edited out of order) is left as appended: the operator handles
// any row order (general CSR path), only the fast sorted path is lost.
int store_merge_appended(relcp_ctx *ctx, relcp_constraints *cs, int64_t n_old, int64_t m) {
    if (m <= 0 || n_old <= 0) return RELCP_OK;  // already sorted
    const int64_t total = n_old + m, cap = cs->capacity;
    CK(ctx->red.grow(64));
    CK(cudaMemsetAsync(ctx->red.p + 63, 0, sizeof(double), ctx->stream));
    int *bad = reinterpret_cast<int *>(ctx->red.p + 63);
    k_check_runs<<<grid_for(total), RELCP_NT, 0, ctx->stream>>>(n_old, total, cs->ia, cs->ib, bad);
    CKL();
    int bad_h = 0;
    CK(cudaMemcpyAsync(&bad_h, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (bad_h) return RELCP_OK;
    CK(ctx->mi.grow(3 * total));
    CK(ctx->md.grow(13 * total));
    cudaStream_t st = ctx->stream;
    k_merge<<<grid_for(total), RELCP_NT, 0, st>>>(n_old, total, cap, cs->ia, cs->ib, cs->gen, cs->n, cs->ta, cs->tb,
                                                  cs->phi, cs->q, cs->lambda, cs->g, ctx->mi.p, ctx->md.p);
    CKL();
    const size_t bi = sizeof(int32_t) * total, bd = sizeof(double) * total;
    CK(cudaMemcpyAsync(cs->ia, ctx->mi.p, bi, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(cs->ib, ctx->mi.p + total, bi, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(cs->gen, ctx->mi.p + 2 * total, bi, cudaMemcpyDeviceToDevice, st));
    for (int c = 0; c < 3; ++c) {
        CK(cudaMemcpyAsync(cs->n + c * cap, ctx->md.p + (0 + c) * total, bd, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(cs->ta + c * cap, ctx->md.p + (3 + c) * total, bd, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(cs->tb + c * cap, ctx->md.p + (6 + c) * total, bd, cudaMemcpyDeviceToDevice, st));
    }
    CK(cudaMemcpyAsync(cs->phi, ctx->md.p + 9 * total, bd, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(cs->q, ctx->md.p + 10 * total, bd, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(cs->lambda, ctx->md.p + 11 * total, bd, cudaMemcpyDeviceToDevice, st));
    if (cs->g) CK(cudaMemcpyAsync(cs->g, ctx->md.p + 12 * total, bd, cudaMemcpyDeviceToDevice, st));
    return RELCP_OK;
}

// sorted[0] = 1 if ia is non-decreasing over [0, nc) (device flag, pre-set to 1)
__global__ void k_check_sorted(int64_t nc, const int32_t *__restrict__ ia, int *sorted) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a + 1 < nc; a += (int64_t)gridDim.x * blockDim.x)
        if (ia[a] > ia[a + 1]) *sorted = 0;
}

int store_is_sorted_by_ia(relcp_ctx *ctx, const relcp_constraints *cs, int *sorted_host) {
    *sorted_host = 1;
    if (cs->count < 2) return RELCP_OK;
    int one = 1;
    CK(cudaMemcpyAsync(ctx->fill.p, &one, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    k_check_sorted<<<grid_for(cs->count), RELCP_NT, 0, ctx->stream>>>(cs->count, cs->ia, ctx->fill.p);
    CKL();
    CK(cudaMemcpyAsync(sorted_host, ctx->fill.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return RELCP_OK;
}
