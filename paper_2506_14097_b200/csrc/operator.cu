// The Delassus operator A = s D^T W D, matrix-free.
//
//   column alpha of D (P:L154-157 Eq. collision_ft; P:L174 F = D gamma):
//       wrench -[n; t_a] on body ia, +[n; t_b] on body ib
//   row alpha of D^T (Phi_dot = n.(ydot_b - ydot_a)):
//       [-n, -t_a, n, t_b]
//   W_b = M_b^{-1} or local-drag mobility
//
// B200 layout:
//   * scatter U = W D x (K6) is a body-major pass.  One warp owns 32 bodies
//     (one per lane).  With the library's sorted store (R18) the a-side rows
//     of those bodies are one contiguous store range, read in place (n, t_a,
//     x, g planes); the b-side entries come from a CSR (constraint id +
//     signed [n; t_b] payload, built once per operator, sorted by constraint).
//     An unsorted caller store puts both sides in the CSR.  Entries are
//     streamed in coalesced 64-entry tiles into shared memory and each lane
//     sums its own body's entries in order (fixed association: bitwise
//     deterministic, no atomics), then applies W_b (SoA planes) and stores U_b
//     through a shared-memory transpose (coalesced).  The kernel reaches 78 %
//     of the copy bandwidth on its bytes and is limited by load latency (the
//     dependent chains pa -> rows, row_ptr -> ecid -> x / g gathers); see
//     profiles/README.md for the variants measured against it.
//   * gather y = s D^T U (K7, k_gather) is a constraint-major streaming pass
//     with U_a, U_b read from L2.  When every row has t . n ~ 0 (t = r x n),
//     the row passes read a compact copy of the rows built here (k_compact,
//     rows.cuh: 6 instead of 9 fp64 per row); otherwise the store's planes.
//   * k_fused_rows: the fused-APGD row pass (lcp.cu solver 2).
#include "common.cuh"
#include "reduce.cuh"
#include "rows.cuh"
#include "k6k7.cuh"
#include "k6pipe.cuh"
#ifndef K6_PIPE
#define K6_PIPE 1
#endif
#ifndef K6_PIPE_MIN_BODIES
#define K6_PIPE_MIN_BODIES 65536
#endif

#ifndef SCATTER_WPB
#define SCATTER_WPB 4    // warps per block (same-box A/B: 4 x 8 blocks beats 8 x 4)
#endif
#ifndef K6_REVERSE
#define K6_REVERSE 1
#endif
#ifndef SCATTER_WAVES
#define SCATTER_WAVES 8  // grid cap = 148 * SCATTER_MINB * waves (grid-stride over 32-body groups)
#endif
#ifndef SCATTER_MINB
#define SCATTER_MINB 8   // resident blocks per SM the register budget must allow (64 regs at 4 warps)
#endif
#ifndef SCATTER_MINB32
#define SCATTER_MINB32 9  // the same for the 32-bodies-per-warp CSR kernel (large stores): 56 registers, 36 warps
#endif                    // per SM.  Same-box A/B, BB K6 on cfg5 A_0 / the relaxed cfg5 store (us): 4 warps x 8
                          // blocks (64 regs) 173.4 / 212.7; 4 x 9 162.7 / 198.7; 3 x 11 161.7 / 198.1; 3 x 12
                          // 161.9 / 197.9; 2 x 18 161.0 / 197.3; 6 x 6 165.3 / 201.2; 5 x 7 166.0 / 203.4 (all
                          // 56 regs); 3 x 10 and 5 x 6 (64 regs, 30 warps) 176.7 / 217.7 and 179.4 / 219.9.
                          // The 8- / 16-body kernels of the small stores keep 8 blocks (cfg2 18.0 vs 18.5 us).

// ------------------------------------------------------------ W blocks (SoA planes)
__global__ void k_build_W(int64_t nb, int dyn, double xi, const double *__restrict__ quat,
                          const double *__restrict__ axes, const double *__restrict__ inv_mass,
                          const double *__restrict__ inv_inertia, const int32_t *__restrict__ kin,
                          const int32_t *__restrict__ shape, double *__restrict__ W) {
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
            // drag length: 2 r_3 (ellipsoid), l + b (rod, R22)
            double L = (shape && (shape[b] == RELCP_SHAPE_SPHEROCYLINDER || shape[b] == RELCP_SHAPE_TORUS))
                           ? 2.0 * (axes[3 * b] + axes[3 * b + 1])
                           : 2.0 * fmax(axes[3 * b], fmax(axes[3 * b + 1], axes[3 * b + 2]));
            double r = 12.0 / (xi * L * L * L);
            w[0] = 1.0 / (xi * L);
            w[1] = r; w[2] = 0.0; w[3] = 0.0; w[4] = r; w[5] = 0.0; w[6] = r;
        }
        bool k = kin && kin[b] != 0;
#pragma unroll
        for (int i = 0; i < 7; ++i) W[i * nb + b] = k ? 0.0 : w[i];  // SoA planes
    }
}

int op_build_W(relcp_ctx *ctx, const relcp_bodies *b, double *W) {
    if (ctx->p.dynamics == RELCP_INERTIAL && (!b->inv_mass || !b->inv_inertia || !b->quat))
        return set_err(ctx, RELCP_E_ARG, "inertial dynamics needs quat, inv_mass and inv_inertia");
    if (ctx->p.dynamics == RELCP_OVERDAMPED && !b->axes)
        return set_err(ctx, RELCP_E_ARG, "overdamped dynamics needs axes");
    k_build_W<<<grid_for(b->n), RELCP_NT, 0, ctx->stream>>>(b->n, ctx->p.dynamics, ctx->p.xi, b->quat, b->axes,
                                                            b->inv_mass, b->inv_inertia, b->kinematic, b->shape, W);
    CKL();
    return RELCP_OK;
}

// ------------------------------------------------------------ CSR of D
// per-body counts of a-side rows (degA) and b-side rows (degB); may alias
__global__ void k_degree(int64_t nc, const int32_t *__restrict__ ia, const int32_t *__restrict__ ib, int *degA,
                         int *degB, int64_t nb, int *bad) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nc; a += (int64_t)gridDim.x * blockDim.x) {
        int i = ia[a], j = ib[a];
        if (i < 0 || j < 0 || i >= nb || j >= nb || i == j) { atomicExch(bad, 1); continue; }
        atomicAdd(degA + i, 1);
        atomicAdd(degB + j, 1);
    }
}

// entry key = side << 30 | constraint (side 0 = a, 1 = b); nc < 2^30
#define EKEY_SIDE (1 << 30)
__global__ void k_fill_slots(int64_t nc, const int32_t *__restrict__ ia, const int32_t *__restrict__ ib,
                             const int *__restrict__ row_ptr, int *fill, int *ekey, int b_only) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nc; a += (int64_t)gridDim.x * blockDim.x) {
        int i = ia[a], j = ib[a];
        if (!b_only) {
            int si = row_ptr[i] + atomicAdd(fill + i, 1);
            ekey[si] = (int)a;  // side a
        }
        int sj = row_ptr[j] + atomicAdd(fill + j, 1);
        ekey[sj] = (int)a | EKEY_SIDE;  // side b
    }
}

// Sort each body segment by key (side, constraint): fixes the summation order.
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
        const int key = ekey[e];
        const int64_t a = key & (EKEY_SIDE - 1);
        const bool side_b = (key & EKEY_SIDE) != 0;
        const double sg = side_b ? 1.0 : -1.0;
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

// Compact rows (rows.cuh) for the constraint-major row passes (K7, the apply
// gather): n, t_a, t_b -> 6 planes, stride rs.  The encoding assumes t . n = 0
// (t = r x n); a row with |t . n| > 1e-13 (1 + |t|) sets *nonorth and
// the operator keeps reading the full rows.
__global__ void k_compact(int64_t nc, int64_t cap, const double *__restrict__ n, const double *__restrict__ ta,
                          const double *__restrict__ tb, int64_t rs, double *__restrict__ rc, int *nonorth) {
    bool bad = false;
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nc; a += (int64_t)gridDim.x * blockDim.x) {
        const double nv[3] = {n[a], n[cap + a], n[2 * cap + a]};
        const double tav[3] = {ta[a], ta[cap + a], ta[2 * cap + a]};
        const double tbv[3] = {tb[a], tb[cap + a], tb[2 * cap + a]};
        double u, v;
        oct_encode(nv[0], nv[1], nv[2], u, v);
        const CNormal c = cn_decode(u, v);
        double a1, a2, b1, b2;
        t_pick(c, tav, a1, a2);
        t_pick(c, tbv, b1, b2);
        rc[a] = u;
        rc[rs + a] = v;
        rc[2 * rs + a] = a1;
        rc[3 * rs + a] = a2;
        rc[4 * rs + a] = b1;
        rc[5 * rs + a] = b2;
        const double da = fabs(tav[0] * nv[0] + tav[1] * nv[1] + tav[2] * nv[2]);
        const double db = fabs(tbv[0] * nv[0] + tbv[1] * nv[1] + tbv[2] * nv[2]);
        const double la = sqrt(tav[0] * tav[0] + tav[1] * tav[1] + tav[2] * tav[2]);
        const double lb = sqrt(tbv[0] * tbv[0] + tbv[1] * tbv[1] + tbv[2] * tbv[2]);
        bad |= !(da <= 1e-13 * (1.0 + la)) || !(db <= 1e-13 * (1.0 + lb));
    }
    if (__any_sync(__activemask(), bad) && (threadIdx.x & 31) == 0) atomicOr(nonorth, 1);
}

// ------------------------------------------------------------ JDS layout (params.layout)
// Per 32-body group (one warp of K6): the group's a-side rows are the store
// range [pa[b0], pa[b0 + 32]) and its b-side entries the CSR range
// [row_ptr[b0], row_ptr[b0 + 32]).  Each range is laid out as a jagged
// diagonal: lanes sorted by degree (descending, ties by body), column j holds
// the j-th entry of every lane with degree > j, so column j is lanes
// 0 .. h_j - 1 at offset base + sum_{j' < j} h_j' (h_j = popc(ballot(deg > j)),
// nothing stored).  meta[32 w + rank] = degree << 5 | local body.  A lane's
// entries keep their order (its rows in store order, its b-side entries
// sorted by constraint), so the summation order of every body is fixed.
//   a-side: perm[slot] = store row, iperm[row] = slot;
//   b-side: bcid[pos] = slot of the entry's row, bpay = (u, v, t_b,j1, t_b,j2)
//           of that row from the slot-order compact planes.
template <bool ASIDE>
__global__ void k_jds_side(int64_t nb, const int *__restrict__ ptr, int *__restrict__ meta, int *__restrict__ perm,
                           int *__restrict__ iperm, const int *__restrict__ ecid, const int *__restrict__ jiperm,
                           const double *__restrict__ rcs, int64_t rs, int *__restrict__ bcid,
                           double *__restrict__ bpay) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarp = (nb + 31) >> 5;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nwarp; w += wstride) {
        const int64_t b0 = w << 5, b = b0 + lane;
        const int s0 = b < nb ? ptr[b] : 0;
        const int deg = b < nb ? ptr[b + 1] - s0 : 0;
        int r = 0;
        for (int m = 0; m < 32; ++m) {
            const int dm = __shfl_sync(0xffffffffu, deg, m);
            r += (dm > deg) || (dm == deg && m < lane);
        }
        meta[b0 + r] = deg << 5 | lane;
        const int maxd = __reduce_max_sync(0xffffffffu, deg);
        int off = ptr[b0];
        for (int j = 0; j < maxd; ++j) {
            const int h = __popc(__ballot_sync(0xffffffffu, deg > j));
            if (j < deg) {
                const int pos = off + r, src = s0 + j;
                if (ASIDE) {
                    perm[pos] = src;
                    iperm[src] = pos;
                } else {
                    const int row = ecid[src] & (EKEY_SIDE - 1);
                    const int slot = jiperm[row];
                    bcid[pos] = slot;
                    bpay[pos] = rcs[slot];
                    bpay[rs + pos] = rcs[rs + slot];
                    bpay[2 * rs + pos] = rcs[4 * rs + slot];
                    bpay[3 * rs + pos] = rcs[5 * rs + slot];
                }
            }
            off += h;
        }
    }
}

// slot-order copies of the compact rows and the ids
__global__ void k_perm_rows(int64_t nc, const int *__restrict__ perm, const double *__restrict__ rc,
                            double *__restrict__ rc2, const int32_t *__restrict__ ia, const int32_t *__restrict__ ib,
                            int32_t *__restrict__ pia, int32_t *__restrict__ pib) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nc; s += (int64_t)gridDim.x * blockDim.x) {
        const int r = perm[s];
#pragma unroll
        for (int k = 0; k < 6; ++k) rc2[k * nc + s] = rc[k * nc + r];
        pia[s] = ia[r];
        pib[s] = ib[r];
    }
}

// out[s] = in[perm[s]] (store order -> slot order)
__global__ void k_perm_gather(int64_t nc, const int *__restrict__ perm, const double *__restrict__ in,
                              double *__restrict__ out) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nc; s += (int64_t)gridDim.x * blockDim.x)
        out[s] = in[perm[s]];
}

static int op_prepare_jds(relcp_ctx *ctx, int64_t nb, int64_t nc, const relcp_constraints *cs) {
    const int64_t nwarp = (nb + 31) / 32;
    CK(ctx->jperm.grow(nc));
    CK(ctx->jiperm.grow(nc));
    CK(ctx->jameta.grow(32 * nwarp));
    CK(ctx->jbmeta.grow(32 * nwarp));
    CK(ctx->jbcid.grow(nc));
    CK(ctx->jbpay.grow(4 * nc));
    CK(ctx->jia.grow(nc));
    CK(ctx->jib.grow(nc));
    CK(ctx->rc2.grow(6 * nc));
    const unsigned gw = (unsigned)grid_for(32 * nwarp, 256, 8);
    // a-side: slot order of the rows
    k_jds_side<true><<<gw, 256, 0, ctx->stream>>>(nb, ctx->pa.p, ctx->jameta.p, ctx->jperm.p, ctx->jiperm.p, nullptr,
                                                  nullptr, nullptr, 0, nullptr, nullptr);
    CKL();
    k_perm_rows<<<grid_for(nc), RELCP_NT, 0, ctx->stream>>>(nc, ctx->jperm.p, ctx->rc.p, ctx->rc2.p, cs->ia, cs->ib,
                                                            ctx->jia.p, ctx->jib.p);
    CKL();
    ctx->rc.swap(ctx->rc2);  // rc: slot order from here on
    // b-side: CSR of the b-side entries (sorted by constraint), then its JDS
    CK(cudaMemsetAsync(ctx->fill.p, 0, sizeof(int) * nb, ctx->stream));
    k_fill_slots<<<grid_for(nc), RELCP_NT, 0, ctx->stream>>>(nc, cs->ia, cs->ib, ctx->row_ptr.p, ctx->fill.p,
                                                             ctx->ecid.p, 1);
    CKL();
    k_sort_segments<<<grid_for(nb, 128), 128, 0, ctx->stream>>>(nb, ctx->row_ptr.p, ctx->ecid.p);
    CKL();
    k_jds_side<false><<<gw, 256, 0, ctx->stream>>>(nb, ctx->row_ptr.p, ctx->jbmeta.p, nullptr, nullptr, ctx->ecid.p,
                                                   ctx->jiperm.p, ctx->rc.p, nc, ctx->jbcid.p, ctx->jbpay.p);
    CKL();
    return RELCP_OK;
}

int op_prepare(relcp_ctx *ctx, const relcp_bodies *b, const relcp_constraints *cs) {
    if (!b || !cs || b->n <= 0) return set_err(ctx, RELCP_E_ARG, "prepare: empty bodies");
    const int64_t nb = b->n, nc = cs->count, E = 2 * nc;
    if (nc < 0 || nc > cs->capacity) return set_err(ctx, RELCP_E_ARG, "prepare: count %lld > capacity", (long long)nc);
    if (nc >= (1ll << 30)) return set_err(ctx, RELCP_E_ARG, "prepare: more than 2^30 constraints");
    CK(ctx->W.grow(RELCP_WSTRIDE * nb));
    CK(ctx->row_ptr.grow(nb + 1));
    CK(ctx->deg.grow(nb + 1));
    CK(ctx->fill.grow(nb + 2));
    CK(ctx->U.grow(6 * nb));
    CK(ctx->ecid.grow(E > 0 ? E : 1));
    CK(ctx->ew.grow(6 * (E > 0 ? E : 1)));
    CK(ctx->pa.grow(nb + 1));
    CK(ctx->rc.grow(6 * (nc > 0 ? nc : 1)));
    CKS(op_build_W(ctx, b, ctx->W.p));
    int sorted = 0;
    CKS(store_is_sorted_by_ia(ctx, cs, &sorted));
    CK(cudaMemsetAsync(ctx->deg.p, 0, sizeof(int) * (nb + 1), ctx->stream));
    CK(cudaMemsetAsync(ctx->pa.p, 0, sizeof(int) * (nb + 1), ctx->stream));
    CK(cudaMemsetAsync(ctx->fill.p, 0, sizeof(int) * (nb + 2), ctx->stream));  // fill[nb] bad, [nb+1] non-orthogonal
    if (nc > 0) {
        k_degree<<<grid_for(nc), RELCP_NT, 0, ctx->stream>>>(nc, cs->ia, cs->ib, sorted ? ctx->pa.p : ctx->deg.p,
                                                             ctx->deg.p, nb, ctx->fill.p + nb);
        CKL();
        k_compact<<<grid_for(nc), RELCP_NT, 0, ctx->stream>>>(nc, cs->capacity, cs->n, cs->ta, cs->tb, nc, ctx->rc.p,
                                                              ctx->fill.p + nb + 1);
        CKL();
    }
    int total = 0;
    CKS(scan_exclusive_int(ctx, ctx->deg.p, ctx->row_ptr.p, nb + 1, &total));  // deg[nb] = 0
    if (sorted) CKS(scan_exclusive_int(ctx, ctx->pa.p, ctx->pa.p, nb + 1, nullptr));  // in place
    int flags[2] = {0, 0};
    CK(cudaMemcpyAsync(flags, ctx->fill.p + nb, 2 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (flags[0]) return set_err(ctx, RELCP_E_ARG, "prepare: body index out of range or ia == ib");
    ctx->op_compact = nc > 0 && !flags[1];
    const int lay = ctx->p.layout;
    const bool jds = ctx->jds_enable && sorted && ctx->op_compact && ctx->p.solver != RELCP_SOLVER_APGD_FUSED &&
                     (lay == RELCP_LAYOUT_JDS || (lay == RELCP_LAYOUT_AUTO && nb >= RELCP_LAYOUT_JDS_MIN_BODIES &&
                                                  nc <= RELCP_LAYOUT_JDS_MAX_ROWS));
    ctx->op_jds = jds;
    if (jds) CKS(op_prepare_jds(ctx, nb, nc, cs));
    const int64_t Ee = sorted ? nc : E;  // CSR entries: b-side only when sorted
    if (nc > 0 && !jds) {
        CK(cudaMemsetAsync(ctx->fill.p, 0, sizeof(int) * nb, ctx->stream));
        k_fill_slots<<<grid_for(nc), RELCP_NT, 0, ctx->stream>>>(nc, cs->ia, cs->ib, ctx->row_ptr.p, ctx->fill.p,
                                                                 ctx->ecid.p, sorted);
        CKL();
        k_sort_segments<<<grid_for(nb, 128), 128, 0, ctx->stream>>>(nb, ctx->row_ptr.p, ctx->ecid.p);
        CKL();
        k_payload<<<grid_for(Ee), RELCP_NT, 0, ctx->stream>>>(Ee, cs->capacity, cs->n, cs->ta, cs->tb, ctx->ecid.p,
                                                              ctx->ew.p);
        CKL();
    }
    // per-group records of the TMA-staged K6 (k6pipe.cuh; params.k6_pipe)
    ctx->op_k6r = 0;
    if (K6_PIPE && nc > 0 && !jds && sorted && ctx->p.k6_pipe && nb >= K6_PIPE_MIN_BODIES) {
        const int64_t nw = (nb + 31) / 32;
        CK(ctx->k6r_sz.grow(nw + 1));
        CK(ctx->k6r_off.grow(nw + 1));
        CK(cudaMemsetAsync(ctx->k6r_sz.p + nw, 0, sizeof(long long), ctx->stream));
        k_k6r_size<<<grid_for(nw), RELCP_NT, 0, ctx->stream>>>(nb, ctx->pa.p, ctx->row_ptr.p, ctx->k6r_sz.p);
        CKL();
        long long tot = 0;
        CKS(scan_exclusive_ll(ctx, ctx->k6r_sz.p, ctx->k6r_off.p, nw + 1, &tot));
        CK(ctx->k6r_rec.grow((size_t)tot + 16));
        k_k6r_fill<<<grid_for(32 * nw, 256, 8), 256, 0, ctx->stream>>>(nb, ctx->pa.p, ctx->row_ptr.p, ctx->k6r_off.p,
                                                                       cs->n, cs->ta, cs->capacity, ctx->ecid.p,
                                                                       ctx->ew.p, nc, ctx->W.p, ctx->k6r_rec.p);
        CKL();
        ctx->op_k6r = 1;
    }
    ctx->op_sorted = sorted;
    ctx->op_cap = cs->capacity;
    ctx->op_rs = nc;
    ctx->op_n = cs->n;
    ctx->op_ta = cs->ta;
    ctx->op_nc = nc;
    ctx->op_nb = nb;
    ctx->op_key_ia = cs->ia;
    return RELCP_OK;
}

// ------------------------------------------------------------ scatter (K6)
// U_b = W_b sum_{e in seg(b)} w_e * xeff(cid_e), xeff = proj ? max(0, x - alpha g) : x,
// scaled by *xscale if given; optionally F_b = the raw sum.
//
// SORTED (store sorted by ia, the library's own order, R18): body b's a-side
// rows are the store rows [pa[b], pa[b+1]) and contribute -[n; t_a] x_eff read
// straight from the store planes; row_ptr / ecid / ew then hold only the
// b-side entries (+[n; t_b]).  Otherwise row_ptr / ecid / ew hold both sides.
// Per-body order: a-side rows, then CSR entries -- fixed, deterministic.
// the U / F transpose reuses a warp's staging area: 2 x 32 x 6 doubles


// MODE: 0 apply (x_eff = x), 1 BB step (x_eff = max(0, x - alpha g)),
// 2 APGD step (y = x + beta (x - x'), g_y likewise, x_eff = max(0, y - t g_y);
// (x, g) / (x', g') are (x, g) / (xb, gb) or swapped by the device parity bit).
template <int MODE, bool SORTED, int GB = 32>
__global__ void __launch_bounds__(32 * SCATTER_WPB, GB == 32 ? SCATTER_MINB32 : SCATTER_MINB) k_scatter(
    K6Op o, const double *__restrict__ x, const double *__restrict__ g, const double *__restrict__ xb,
    const double *__restrict__ gb, const LcpState *__restrict__ st, const double *__restrict__ xscale,
    double *__restrict__ U, double *__restrict__ Fout, const double *__restrict__ Fa) {
    // contributions staged as 3 planes of double2 (components 01, 23, 45):
    // 128-bit shared loads in the per-lane segment sums
    __shared__ double2 sm[SCATTER_WPB][K6_SMEM_D2];
    pdl_wait();
    pdl_open();
    if (MODE != 0 && st->done) return;
    const XEff xe = xeff_setup<MODE>(st, x, g, xb, gb, xscale);
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int64_t nwarp = (o.nb + GB - 1) / GB;
    for (int64_t wi = blockIdx.x * (int64_t)SCATTER_WPB + wl; wi < nwarp; wi += (int64_t)gridDim.x * SCATTER_WPB) {
        // K6_REVERSE: sweep bodies high -> low, so K6 starts on the rows, x and g
        // K7 (ascending) touched last (still in L2) and ends on the bodies whose
        // U / rows K7 touches first
        const int64_t w = K6_REVERSE ? nwarp - 1 - wi : wi;
        k6_group<MODE, SORTED, GB>(w, o, xe, reinterpret_cast<double2(*)[SCATTER_TILE + 1]>(sm[wl]), lane, U, Fout,
                                   Fa);
    }
}

// ------------------------------------------------------------ scatter, JDS layout (K6)
// Same operator as k_scatter (U_b = W_b sum_e w_e x_eff, MODE 0 / 1 / 2) on the
// JDS layout (op_prepare_jds): one warp per 32-body group.  The warp's
// entries are streamed in chunks of whole columns (<= JT_TILE entries), one
// entry per lane and trip with every lane active (coalesced loads, x_eff and
// the row decode done once per entry), the 6-vector contributions staged in
// shared memory as three double2 planes in entry order; then lane r sums its
// column entries, which sit at consecutive positions across lanes (column j:
// lanes 0 .. h_j - 1), so the shared-memory reads are conflict-free.
#ifndef JDS_WPB
#define JDS_WPB 4
#endif
#ifndef JT_TILE
#define JT_TILE 64
#endif
#ifndef JT_MINB
#define JT_MINB 8
#endif
template <int MODE>
__global__ void __launch_bounds__(32 * JDS_WPB, JT_MINB) k_scatter_jt(
    int64_t nb, int64_t rs, const int *__restrict__ pa, const int *__restrict__ row_ptr,
    const int *__restrict__ ameta, const int *__restrict__ bmeta, const double *__restrict__ rc,
    const int *__restrict__ bcid, const double *__restrict__ bpay, const double *__restrict__ x,
    const double *__restrict__ g, const double *__restrict__ xb, const double *__restrict__ gb,
    const LcpState *__restrict__ st, const double *__restrict__ xscale, const double *__restrict__ W,
    double *__restrict__ U, double *__restrict__ Fout) {
    __shared__ double2 sm[JDS_WPB][3][JT_TILE];
    __shared__ double sa_[JDS_WPB][6][32];
    pdl_wait();
    pdl_open();
    double alpha = 0.0, beta = 0.0, tl = 1.0;
    bool fix = false;
    const double *xc = x, *gc = g, *xp = xb, *gp = gb;
    if (MODE != 0) {
        if (st->done) return;
        alpha = st->alpha;
    }
    if (MODE == 1) {
        if (st->par) {
            xc = xb; gc = gb; xp = x; gp = g;
        }
        fix = st->fix != 0;
        tl = st->t_ls;
    }
    if (MODE == 2) {
        beta = st->beta;
        if (st->par) {
            xc = xb; gc = gb; xp = x; gp = g;
        }
    }
    const double sc = xscale ? *xscale : 1.0;
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    double2(*c6)[JT_TILE] = sm[wl];
    double(*sa)[32] = sa_[wl];
    auto xeff = [&](int c) {
        double xv;
        if (MODE == 0) {
            xv = xc[c];
        } else if (MODE == 1) {
            double x0 = xc[c], g0 = gc[c];
            if (fix) {
                const double xq = xp[c], gq = gp[c];
                x0 = fma(tl, x0 - xq, xq);
                g0 = fma(tl, g0 - gq, gq);
            }
            xv = fmax(0.0, x0 - alpha * g0);
        } else {
            const double x0 = xc[c], g0 = gc[c];
            const double y = x0 + beta * (x0 - xp[c]), gy = g0 + beta * (g0 - gp[c]);
            xv = fmax(0.0, y - alpha * gy);
        }
        return xv * sc;
    };
    // one side of the warp's group: entries [base, base + sum_j h_j) in JDS
    // order, lane degree deg; fetch(pos, v[6]) forms one entry's contribution
    auto side = [&](int base, int deg, double (&f)[6], auto &&fetch) {
        const int maxd = __reduce_max_sync(0xffffffffu, deg);
        int j = 0, off = base;
        while (j < maxd) {
            int j1 = j, tot = 0;
            while (j1 < maxd) {  // whole columns, <= JT_TILE entries
                const int h = __popc(__ballot_sync(0xffffffffu, deg > j1));
                if (tot + h > JT_TILE) break;
                tot += h;
                ++j1;
            }
#pragma unroll
            for (int i = 0; i < JT_TILE / 32; ++i) {
                const int p = lane + 32 * i;
                if (p < tot) {
                    double v[6];
                    fetch(off + p, v);
#pragma unroll
                    for (int k = 0; k < 3; ++k) c6[k][p] = make_double2(v[2 * k], v[2 * k + 1]);
                }
            }
            __syncwarp();
            int o = 0;
            for (int jj = j; jj < j1; ++jj) {
                const int h = __popc(__ballot_sync(0xffffffffu, deg > jj));
                if (lane < h) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        const double2 c = c6[k][o + lane];
                        f[2 * k] += c.x;
                        f[2 * k + 1] += c.y;
                    }
                }
                o += h;
            }
            __syncwarp();
            off += tot;
            j = j1;
        }
    };
    auto contrib = [](double u, double v, double t1, double t2, double xe, double (&o)[6]) {
        const CNormal c = cn_decode(u, v);
        double t[3];
        t_expand(c, t1, t2, t);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            o[k] = c.n[k] * xe;
            o[3 + k] = t[k] * xe;
        }
    };
    const int64_t nwarp = (nb + 31) >> 5;
    const int64_t wstep = (int64_t)gridDim.x * JDS_WPB;
    for (int64_t w = blockIdx.x * (int64_t)JDS_WPB + wl; w < nwarp; w += wstep) {
        const int64_t b0 = w << 5;
        const int64_t b = b0 + lane;
        const bool own = b < nb;
        const int last = nb - b0 < 32 ? (int)(nb - b0 - 1) : 31;
        const int am = ameta[b0 + lane], bm = bmeta[b0 + lane];
        const int cA0 = pa[b0], cB0 = row_ptr[b0];
        double f[6] = {0, 0, 0, 0, 0, 0};
        // a-side: -[n; t_a] x_eff at consecutive slots
        side(cA0, am >> 5, f, [&](int s, double (&v)[6]) {
            contrib(rc[s], rc[rs + s], rc[2 * rs + s], rc[3 * rs + s], -xeff(s), v);
        });
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            sa[k][am & 31] = f[k];
            f[k] = 0.0;
        }
        // b-side: +[n; t_b] x_eff, x / g gathered at the entries' slots
        side(cB0, bm >> 5, f, [&](int e, double (&v)[6]) {
            const int c = bcid[e];
            contrib(bpay[e], bpay[rs + e], bpay[2 * rs + e], bpay[3 * rs + e], xeff(c), v);
        });
        double *flat = &c6[0][0].x;  // 3 x JT_TILE double2 >= 2 x 192 doubles
        static_assert(6 * JT_TILE >= 384, "JT_TILE too small for the U / F staging");
#pragma unroll
        for (int k = 0; k < 6; ++k) flat[k * 32 + (bm & 31)] = f[k];
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 6; ++k) f[k] = sa[k][lane] + flat[k * 32 + lane];
        __syncwarp();
        double u[6] = {0, 0, 0, 0, 0, 0};
        if (own) {
            const double w0 = W[b], s00 = W[nb + b], s01 = W[2 * nb + b], s02 = W[3 * nb + b], s11 = W[4 * nb + b],
                         s12 = W[5 * nb + b], s22 = W[6 * nb + b];
            u[0] = w0 * f[0];
            u[1] = w0 * f[1];
            u[2] = w0 * f[2];
            u[3] = s00 * f[3] + s01 * f[4] + s02 * f[5];
            u[4] = s01 * f[3] + s11 * f[4] + s12 * f[5];
            u[5] = s02 * f[3] + s12 * f[4] + s22 * f[5];
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            flat[6 * lane + k] = u[k];
            flat[192 + 6 * lane + k] = f[k];
        }
        __syncwarp();
        const int64_t nvals = 6 * (int64_t)(last + 1);
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            const int m = lane + 32 * i;
            if (m < nvals) {
                U[6 * b0 + m] = flat[m];
                if (Fout) Fout[6 * b0 + m] = flat[192 + m];
            }
        }
        __syncwarp();
    }
}

K6Op op_k6(const relcp_ctx *ctx) {
    return K6Op{ctx->op_nb, ctx->op_sorted ? ctx->op_nc : 2 * ctx->op_nc, ctx->op_cap, ctx->row_ptr.p, ctx->ecid.p,
                ctx->pa.p, ctx->ew.p, ctx->op_n, ctx->op_ta, ctx->W.p};
}

int op_scatter(relcp_ctx *ctx, int64_t nb, const double *x, const double *g, int mode, const double *xscale_dev,
               double *U, double *F, const double *xb, const double *gb, int slots) {
    if (ctx->op_jds) {
        const int64_t nc = ctx->op_nc;
        if (!slots) {  // caller's store order: apply / wrench / the check's U_c
            if (mode != 0) return set_err(ctx, RELCP_E_STATE, "JDS scatter: store-order input is apply-only");
            CK(ctx->jtmp.grow(nc));
            k_perm_gather<<<grid_for(nc), RELCP_NT, 0, ctx->stream>>>(nc, ctx->jperm.p, x, ctx->jtmp.p);
            CKL();
            x = ctx->jtmp.p;
        }
        const int64_t nwarp = (nb + 31) / 32;
        const int minb = JT_MINB;
        int64_t grid = (nwarp + JDS_WPB - 1) / JDS_WPB;
        if (grid > (int64_t)RELCP_SM_COUNT * minb * SCATTER_WAVES) grid = (int64_t)RELCP_SM_COUNT * minb * SCATTER_WAVES;
        if (grid < 1) grid = 1;
#define JDS_ARGS nb, nc, ctx->pa.p, ctx->row_ptr.p, ctx->jameta.p, ctx->jbmeta.p, ctx->rc.p, ctx->jbcid.p, \
                 ctx->jbpay.p, x, g, xb, gb, ctx->st.p, xscale_dev, ctx->W.p, U, F
        if (mode < 0 || mode > 2) return set_err(ctx, RELCP_E_STATE, "JDS scatter: mode %d unsupported", mode);
        if (mode == 1) CK(launch_k(ctx->pdl, k_scatter_jt<1>, (unsigned)grid, 32 * JDS_WPB, 0, ctx->stream, JDS_ARGS));
        else if (mode == 2) CK(launch_k(ctx->pdl, k_scatter_jt<2>, (unsigned)grid, 32 * JDS_WPB, 0, ctx->stream, JDS_ARGS));
        else k_scatter_jt<0><<<(unsigned)grid, 32 * JDS_WPB, 0, ctx->stream>>>(JDS_ARGS);
#undef JDS_ARGS
        CKL();
        return RELCP_OK;
    }
    if (K6_PIPE && ctx->op_k6r && mode >= 0 && mode <= 2) {
        // TMA-staged K6 (k6pipe.cuh): persistent CTAs, K6P_MINB per SM
        if (!ctx->k6p_attr) {
            CK(cudaFuncSetAttribute(k_scatter_pipe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, k6p::SMEM));
            CK(cudaFuncSetAttribute(k_scatter_pipe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, k6p::SMEM));
            CK(cudaFuncSetAttribute(k_scatter_pipe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, k6p::SMEM));
            ctx->k6p_attr = 1;
        }
        const int64_t nwarp = (nb + 31) / 32;
        int64_t grid = (int64_t)RELCP_SM_COUNT * K6P_MINB;
        if (grid > nwarp) grid = nwarp;
        const K6Op o = op_k6(ctx);
        if (mode == 1)
            k_scatter_pipe<1><<<(unsigned)grid, K6P_NT, k6p::SMEM, ctx->stream>>>(
                o, ctx->k6r_rec.p, ctx->k6r_off.p, x, g, xb, gb, ctx->st.p, xscale_dev, U, F);
        else if (mode == 2)
            k_scatter_pipe<2><<<(unsigned)grid, K6P_NT, k6p::SMEM, ctx->stream>>>(
                o, ctx->k6r_rec.p, ctx->k6r_off.p, x, g, xb, gb, ctx->st.p, xscale_dev, U, F);
        else
            k_scatter_pipe<0><<<(unsigned)grid, K6P_NT, k6p::SMEM, ctx->stream>>>(
                o, ctx->k6r_rec.p, ctx->k6r_off.p, x, g, xb, gb, ctx->st.p, xscale_dev, U, F);
        CKL();
        return RELCP_OK;
    }
    const int64_t E = ctx->op_sorted ? ctx->op_nc : 2 * ctx->op_nc;
    // bodies per warp (params.k6_bpw): 32, or RELCP_K6_BPW_SMALL for stores with
    // few 32-body groups per SM, where the per-warp chain of dependent tile
    // loads is the floor (same-box A/B, profiles/README: cfg2 iteration 14.6 ->
    // 13.2 us with 8; cfg5 A_0 loses with 8 or 16: 0.28 -> 0.38 / 0.30 ms)
    int bpw = ctx->p.k6_bpw ? ctx->p.k6_bpw : (nb <= RELCP_K6_SMALL_N ? RELCP_K6_BPW_SMALL : 32);
    if (!ctx->op_sorted) bpw = 32;
    const int64_t nwarp = (nb + bpw - 1) / bpw;
    int64_t grid = (nwarp + SCATTER_WPB - 1) / SCATTER_WPB;
    const int64_t gcap = (int64_t)RELCP_SM_COUNT * (bpw == 32 ? SCATTER_MINB32 : SCATTER_MINB) * SCATTER_WAVES;
    if (grid > gcap) grid = gcap;
    if (grid < 1) grid = 1;
    const unsigned G = (unsigned)grid, T = 32 * SCATTER_WPB;
    const int *pa = ctx->pa.p;
    const int64_t cap = ctx->op_cap;
    const double *cn = ctx->op_n, *cta = ctx->op_ta;
    const K6Op o{nb, E, cap, ctx->row_ptr.p, ctx->ecid.p, pa, ctx->ew.p, cn, cta, ctx->W.p};
#define SCATTER_ARGS o, x, g, xb, gb, ctx->st.p, xscale_dev, U, F, ctx->Fa.p
    if (mode == 3) {
        if (!ctx->op_sorted) return set_err(ctx, RELCP_E_STATE, "fused solver needs a store sorted by ia");
        k_scatter<3, true><<<G, T, 0, ctx->stream>>>(SCATTER_ARGS);
    } else if (ctx->op_sorted && bpw == 8) {
        if (mode == 1) CK(launch_k(ctx->pdl, k_scatter<1, true, 8>, G, T, 0, ctx->stream, SCATTER_ARGS));
        else if (mode == 2) CK(launch_k(ctx->pdl, k_scatter<2, true, 8>, G, T, 0, ctx->stream, SCATTER_ARGS));
        else k_scatter<0, true, 8><<<G, T, 0, ctx->stream>>>(SCATTER_ARGS);
    } else if (ctx->op_sorted && bpw == 16) {
        if (mode == 1) CK(launch_k(ctx->pdl, k_scatter<1, true, 16>, G, T, 0, ctx->stream, SCATTER_ARGS));
        else if (mode == 2) CK(launch_k(ctx->pdl, k_scatter<2, true, 16>, G, T, 0, ctx->stream, SCATTER_ARGS));
        else k_scatter<0, true, 16><<<G, T, 0, ctx->stream>>>(SCATTER_ARGS);
    } else if (ctx->op_sorted) {
        if (mode == 1) CK(launch_k(ctx->pdl, k_scatter<1, true>, G, T, 0, ctx->stream, SCATTER_ARGS));
        else if (mode == 2) CK(launch_k(ctx->pdl, k_scatter<2, true>, G, T, 0, ctx->stream, SCATTER_ARGS));
        else k_scatter<0, true><<<G, T, 0, ctx->stream>>>(SCATTER_ARGS);
    } else {
        if (mode == 1) k_scatter<1, false><<<G, T, 0, ctx->stream>>>(SCATTER_ARGS);
        else if (mode == 2) k_scatter<2, false><<<G, T, 0, ctx->stream>>>(SCATTER_ARGS);
        else k_scatter<0, false><<<G, T, 0, ctx->stream>>>(SCATTER_ARGS);
    }
#undef SCATTER_ARGS
    CKL();
    return RELCP_OK;
}

// ------------------------------------------------------------ fused BB row pass
#include "rows.cuh"
#define row_dot row_dot_u

// Fused APGD iteration (solver RELCP_SOLVER_APGD_FUSED), row pass of iteration k.
// APGD's extrapolation weight beta_k is fixed by the previous pass's restart
// test, so every row can finish, from data already in registers,
//   g_k = A x_k + q,  y = x_k + beta (x_k - x_{k-1}),  g_y = g_k + beta (g_k - g_{k-1}),
//   x_{k+1} = max(0, y - t g_y)   and the restart dot g_y . (x_{k+1} - x_k),
// AND form the a-side wrench sums of x_{k+1} (K6's a-side re-read of the rows
// disappears; K6 mode 3 adds the b-side).  Same iterates as solver APGD up to
// rounding.  Body-major over the sorted store: warp = 32 bodies, their a-side
// rows are one contiguous range, streamed in coalesced tiles; shared-memory
// segment sums (fixed order).
//   in : x_k (cur slot), x_{k-1} (prev slot), g_{k-1} (g), U = W D x_k
//   out: g_k (g, in place), x_{k+1} (prev slot), Fa = a-side sums of x_{k+1}
#ifndef FUSED_MINB
#define FUSED_MINB 5  // register budget ~100 (the row work + staging would spill at 64)
#endif
__global__ void __launch_bounds__(32 * SCATTER_WPB, FUSED_MINB) k_fused_rows(
    int64_t nb, int64_t cap, const int *__restrict__ pa, const int32_t *__restrict__ ia,
    const int32_t *__restrict__ ib, const double *__restrict__ n, const double *__restrict__ ta,
    const double *__restrict__ tb, const double *__restrict__ U, double s, const double *__restrict__ q,
    double *xA, double *xB, double *g, double *__restrict__ Fa, double *part, unsigned *counter, LcpState *st) {
    __shared__ double2 sm[SCATTER_WPB][3][SCATTER_TILE + 1];
    __shared__ double shr[3 * 32];
    if (st->done) return;
    const double t = st->alpha, beta = st->beta;
    double *xc = xA, *xp = xB;
    if (st->par) {
        xc = xB; xp = xA;
    }
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    double2(*c6)[SCATTER_TILE + 1] = sm[wl];
    const int64_t nwarp = (nb + 31) >> 5;
    double acc[3] = {0.0, 0.0, 0.0};  // restart dot, residual, non-finite flag
    for (int64_t w = blockIdx.x * (int64_t)SCATTER_WPB + wl; w < nwarp; w += (int64_t)gridDim.x * SCATTER_WPB) {
        const int64_t b0 = w << 5;
        const int64_t b = b0 + lane;
        const bool own = b < nb;
        const int last = nb - b0 < 32 ? (int)(nb - b0 - 1) : 31;
        const int sa = own ? pa[b] : 0, tA = own ? pa[b + 1] : 0;
        const int e0 = __shfl_sync(0xffffffffu, sa, 0);
        const int e1 = __shfl_sync(0xffffffffu, tA, last);
        double f[6] = {0, 0, 0, 0, 0, 0};
        for (int base = e0; base < e1; base += SCATTER_TILE) {
#pragma unroll
            for (int i = 0; i < SCATTER_TILE / 32; ++i) {
                const int e = base + lane + 32 * i;
                if (e < e1) {
                    const double x1 = xc[e], x0 = xp[e], g0 = g[e];  // x_k, x_{k-1}, g_{k-1}
                    const double g1 = fma(s, row_dot(e, cap, ia, ib, n, ta, tb, U), q[e]);  // g_k
                    const double y = x1 + beta * (x1 - x0), gy = g1 + beta * (g1 - g0);
                    const double x2 = fmax(0.0, y - t * gy);  // x_{k+1}
                    xp[e] = x2;
                    g[e] = g1;
                    acc[0] = fma(gy, x2 - x1, acc[0]);
                    acc[1] = fmax(acc[1], fabs(fmin(x1, g1)));
                    acc[2] = fmax(acc[2], isfinite(g1) ? 0.0 : 1.0);
                    const double nx = n[e], ny = n[cap + e], nz = n[2 * cap + e];
                    const double tx = ta[e], ty = ta[cap + e], tz = ta[2 * cap + e];
                    c6[0][lane + 32 * i] = make_double2(-nx * x2, -ny * x2);
                    c6[1][lane + 32 * i] = make_double2(-nz * x2, -tx * x2);
                    c6[2][lane + 32 * i] = make_double2(-ty * x2, -tz * x2);
                }
            }
            __syncwarp();
            const int lo = max(sa, base) - base, hi = min(tA, base + SCATTER_TILE) - base;
            for (int j = lo; j < hi; ++j)
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const double2 c = c6[k][j];
                    f[2 * k] += c.x;
                    f[2 * k + 1] += c.y;
                }
            __syncwarp();
        }
        if (own)
#pragma unroll
            for (int k = 0; k < 6; ++k) Fa[k * nb + b] = f[k];
    }
    const int ops[3] = {0, 1, 1};
    if (grid_reduce_last<3>(acc, ops, part, counter, shr) && threadIdx.x == 0) {
        const long long k = st->iter;
        st->resid = acc[1];  // residual of (x_k, g_k)
        if (acc[2] > 0.0 || !isfinite(acc[0])) {
            st->nan = 1;
            st->done = 1;
            return;
        }
        if (acc[1] <= st->tol) {  // (x_k, g_k) solve the LCP: x_k stays current
            st->conv = 1;
            st->done = 1;
            return;
        }
        if (k >= st->max_iter) {  // stop on the consistent pair (x_k, g_k)
            st->done = 1;
            return;
        }
        st->iter = k + 1;
        const double th = st->theta;
        if (acc[0] > 0.0) {  // adaptive restart
            st->theta = 1.0;
            st->beta = 0.0;
        } else {
            const double th1 = 0.5 * (th * sqrt(th * th + 4.0) - th * th);
            st->beta = th * (1.0 - th) / (th * th + th1);
            st->theta = th1;
        }
        st->par ^= 1;  // x_{k+1} becomes current
    }
}

int op_fused_rows(relcp_ctx *ctx, const relcp_constraints *cs, int64_t nb, double s, double *xA, double *xB) {
    CK(ctx->Fa.grow(6 * nb));
    const int64_t nwarp = (nb + 31) / 32;
    int64_t grid = (nwarp + SCATTER_WPB - 1) / SCATTER_WPB;
    if (grid > (int64_t)RELCP_SM_COUNT * FUSED_MINB) grid = (int64_t)RELCP_SM_COUNT * FUSED_MINB;
    if (grid < 1) grid = 1;
    k_fused_rows<<<(unsigned)grid, 32 * SCATTER_WPB, 0, ctx->stream>>>(
        nb, cs->capacity, ctx->pa.p, cs->ia, cs->ib, cs->n, cs->ta, cs->tb, ctx->U.p, s, cs->q, xA, xB, cs->g,
        ctx->Fa.p, ctx->partials.p, ctx->counter.p, ctx->st.p);
    CKL();
    return RELCP_OK;
}

// ------------------------------------------------------------ gather
#ifndef GATHER_ILP
#define GATHER_ILP 2  // rows per thread per trip in the apply gather (store rows; same-box A/B: 2 beats 4)
#endif
#ifndef GATHER_ILP_CR
#define GATHER_ILP_CR 1  // with compact rows: 1 row x 4 blocks (64 registers).  Same-box A/B, whole apply on cfg5
#endif                   // A_0 / the relaxed store (us): 227.8 / 285.0 against 232.6 / 293.1 (2 rows x 3 blocks,
                         // 72 registers), 233.7 / 294.4 (1 x 3), 244.0 / 309.6 (2 x 2)
#ifndef GATHER_MINB_CR
#define GATHER_MINB_CR 4  // resident blocks per SM with compact rows
#endif

// y = scale * D^T U ; optionally the grid-wide ||y||^2 -> st->pnorm = 1/||y||, st->L = ||y||
// (or, with acc_out, the block-reduced ||y||^2 of this part for dd.cu)
// CR: rows from the compact planes rc (stride rs) instead of the store.
template <bool CR>
__global__ void __launch_bounds__(RELCP_NT, CR ? GATHER_MINB_CR : 4) k_gather(int64_t nc, int64_t cap, const int32_t *__restrict__ ia,
                                                     const int32_t *__restrict__ ib, const double *__restrict__ n,
                                                     const double *__restrict__ ta, const double *__restrict__ tb,
                                                     int64_t rs, const double *__restrict__ rc,
                                                     const double *__restrict__ U, double scale,
                                                     double *__restrict__ y, int norm2, double *part,
                                                     unsigned *counter, LcpState *st, double *acc_out,
                                                     const int *__restrict__ yperm) {
    __shared__ double sh[32];
    constexpr int ILP = CR ? GATHER_ILP_CR : GATHER_ILP;
    double acc[1] = {0.0};
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t a0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a0 < nc; a0 += ILP * stride) {
        double v[ILP];
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            const int64_t a = a0 + u * stride;
            const int64_t ac = a < nc ? a : a0;
            v[u] = scale * (CR ? row_dot_c(ac, rs, ia, ib, rc, U) : row_dot(ac, cap, ia, ib, n, ta, tb, U));
        }
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            const int64_t a = a0 + u * stride;
            if (a >= nc) continue;
            y[yperm ? yperm[a] : a] = v[u];  // JDS operator, caller's store order: slot -> row
            acc[0] = fma(v[u], v[u], acc[0]);
        }
    }
    if (!norm2) return;
    const int ops[1] = {0};
    if (grid_reduce_last<1>(acc, ops, part, counter, sh) && threadIdx.x == 0) {
        if (acc_out) {  // domain decomposition: combined over parts first (dd.cu)
            acc_out[0] = acc[0];
            return;
        }
        power_finalize(st, acc);
    }
}

int op_gather_apply(relcp_ctx *ctx, const relcp_constraints *cs, const double *U, double *y, double scale,
                    int norm2, double *acc_out) {
    const int64_t nc = cs->count;
    if (nc == 0) return RELCP_OK;
    const int grid = grid_for(nc, RELCP_NT, ctx->op_compact ? GATHER_MINB_CR : 4);
    const int32_t *ia = cs->ia, *ib = cs->ib;
    const int *yperm = nullptr;
    if (ctx->op_jds && cs->ia != ctx->jia.p) {  // caller's store: rows from the slot order, y through perm
        ia = ctx->jia.p;
        ib = ctx->jib.p;
        yperm = ctx->jperm.p;
    }
    if (ctx->op_compact)
        k_gather<true><<<grid, RELCP_NT, 0, ctx->stream>>>(nc, cs->capacity, ia, ib, cs->n, cs->ta, cs->tb,
                                                           ctx->op_rs, ctx->rc.p, U, scale, y, norm2, ctx->partials.p,
                                                           ctx->counter.p, ctx->st.p, acc_out, yperm);
    else
        k_gather<false><<<grid, RELCP_NT, 0, ctx->stream>>>(nc, cs->capacity, ia, ib, cs->n, cs->ta, cs->tb,
                                                            ctx->op_rs, ctx->rc.p, U, scale, y, norm2, ctx->partials.p,
                                                            ctx->counter.p, ctx->st.p, acc_out, yperm);
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
