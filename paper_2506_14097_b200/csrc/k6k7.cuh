// Bodies of the two LCP-iteration passes, shared by the
// per-pass kernels (operator.cu k_scatter, lcp.cu k_lcp_iter) and the
// single-cluster BB loop for small stores (lcp.cu k_bb_cluster):
//   k6_group : U_b = W_b sum_e w_e x_eff(e) for the 32 bodies of one warp
//              (CSR layout; DESIGN.md §5 K6);
//   k7_rows  : x+ = max(0, x - alpha g), g+ = s row . [U_a; U_b] + q and the
//              six BB partials for a strided range of rows (K7).
#pragma once
#include "common.cuh"
#include "rows.cuh"

#ifndef SCATTER_TILE
#define SCATTER_TILE 64  // entries staged per warp per tile
#endif
#ifndef K6_CL
#define K6_CL 0  // 1 / 2: component-lane segment sums (k6_group), per-round loops / one merged loop
#endif

struct V6 {
    double v[6];
};
// double2 per warp for k6_group's staging: 3 planes of SCATTER_TILE + 1 entries,
// and at least 192 (the U / F transpose: 2 x 192 doubles)
#define K6_SMEM_D2 (3 * (SCATTER_TILE + 1) > 192 ? 3 * (SCATTER_TILE + 1) : 192)

// CSR operator of a prepared context (op_prepare)
struct K6Op {
    int64_t nb, E, cap;
    const int *row_ptr, *ecid, *pa;
    const double *ew, *cn, *cta, *W;
};

K6Op op_k6(const relcp_ctx *ctx);  // the prepared CSR operator (operator.cu)

// x_eff of one iteration.  MODE: 0 apply (x), 1 BB step max(0, x - alpha g)
// (after a shortened step the iterate is the blend xp + t (xc - xp) of the two
// slots), 2 APGD step from (x, g) / (x', g'), 3 fused BB (x of the current slot)
struct XEff {
    double alpha = 0.0, beta = 0.0, tl = 1.0, sc = 1.0;
    bool fix = false;
    const double *xc, *gc, *xp, *gp;
};

template <int MODE>
__device__ __forceinline__ XEff xeff_setup(const LcpState *st, const double *x, const double *g, const double *xb,
                                           const double *gb, const double *xscale) {
    XEff e;
    e.xc = x; e.gc = g; e.xp = xb; e.gp = gb;
    if (MODE != 0) e.alpha = st->alpha;
    if (MODE == 1) {
        if (st->par) {
            e.xc = xb; e.gc = gb; e.xp = x; e.gp = g;
        }
        e.fix = st->fix != 0;
        e.tl = st->t_ls;
    }
    if (MODE == 2) {
        e.beta = st->beta;
        if (st->par) {
            e.xc = xb; e.gc = gb; e.xp = x; e.gp = g;
        }
    }
    if (MODE == 3 && st->par) e.xc = xb;
    e.sc = xscale ? *xscale : 1.0;
    return e;
}

template <int MODE>
__device__ __forceinline__ double xeff_at(const XEff &e, int c) {
    double xv;
    if (MODE == 0 || MODE == 3) {
        xv = e.xc[c];
    } else if (MODE == 1) {
        double x0 = e.xc[c], g0 = e.gc[c];
        if (e.fix) {
            const double xq = e.xp[c], gq = e.gp[c];
            x0 = fma(e.tl, x0 - xq, xq);
            g0 = fma(e.tl, g0 - gq, gq);
        }
        xv = fmax(0.0, x0 - e.alpha * g0);
    } else {
        const double x0 = e.xc[c], g0 = e.gc[c];
        const double y = x0 + e.beta * (x0 - e.xp[c]), gy = g0 + e.beta * (g0 - e.gp[c]);
        xv = fmax(0.0, y - e.alpha * gy);
    }
    return xv * e.sc;
}

// One warp: bodies 32 w .. 32 w + 31 (lane = body).  SORTED (store sorted by
// ia, R18): the a-side rows of the warp's bodies are the store range
// [pa[b0], pa[b0 + 32]), read in place (-[n; t_a] x_eff); row_ptr / ecid / ew
// hold the b-side entries (+[n; t_b]).  Otherwise the CSR holds both sides.
// Entries are streamed in coalesced SCATTER_TILE-entry tiles into shared
// memory (c6: 3 double2 planes of SCATTER_TILE + 1) and each lane sums its own
// body's entries in order (a-side rows, then CSR entries: fixed association,
// bitwise deterministic), then U_b = W_b F_b is stored through a shared-memory
// transpose (coalesced).  Fout: the raw sums F_b; Fa (MODE 3): a-side sums
// formed by the fused row pass.
//
// GB (bodies per warp, 32 / 16 / 8): lanes 0..GB-1 own bodies GB w .. GB w +
// GB - 1; all 32 lanes stream the tiles.  Each body's summation order does not
// depend on GB (bitwise identical U), only the number of dependent tile
// round trips per warp does: small stores (few groups per SM) run GB < 32 so
// that a warp's chain covers fewer entries and more warps are in flight.
template <int MODE, bool SORTED, int GB = 32>
__device__ __forceinline__ void k6_group(int64_t w, const K6Op &o, const XEff &xe, double2 (*c6)[SCATTER_TILE + 1],
                                         int lane, double *__restrict__ U, double *__restrict__ Fout,
                                         const double *__restrict__ Fa) {
    static_assert(GB == 32 || GB == 16 || GB == 8, "bodies per warp");
    const int64_t nb = o.nb;
    const int64_t b0 = w * GB;
    const int64_t b = b0 + lane;
    const bool own = lane < GB && b < nb;
    const int last = nb - b0 < GB ? (int)(nb - b0 - 1) : GB - 1;
    double f[6] = {0, 0, 0, 0, 0, 0};
    // stream [e0, e1) of the warp in coalesced tiles; lane sums its [s, t)
    auto tiles = [&](int s, int t, auto &&fetch) {
        const int e0 = __shfl_sync(0xffffffffu, s, 0);
        const int e1 = __shfl_sync(0xffffffffu, t, last);
        for (int base = e0; base < e1; base += SCATTER_TILE) {
#pragma unroll
            for (int i = 0; i < SCATTER_TILE / 32; ++i) {
                const int e = base + lane + 32 * i;
                if (e < e1) {  // slots past e1 are never read
                    const V6 v = fetch(e);
#pragma unroll
                    for (int k = 0; k < 3; ++k) c6[k][lane + 32 * i] = make_double2(v.v[2 * k], v.v[2 * k + 1]);
                }
            }
            __syncwarp();
            const int lo = max(s, base) - base, hi = min(t, base + SCATTER_TILE) - base;
            for (int j = lo; j < hi; ++j)
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const double2 c = c6[k][j];
                    f[2 * k] += c.x;
                    f[2 * k + 1] += c.y;
                }
            __syncwarp();
        }
    };
#if K6_CL
    // Component lanes (K6_CL, GB = 32, MODE != 3): the 192 sums (body, k) of the
    // group are held one per lane and round, pair p = 32 r + lane = 6 body + k
    // (the AoS order of U / F).  Entries are staged AoS (6 doubles each,
    // conflict-free 16-byte stores); a lane adds ONE double per entry of its
    // pair's body, so a warp-wide shared load serves 32 pairs of ~5 bodies
    // (8-byte accesses, 2-3 wavefronts) instead of 32 bodies x 16 bytes at
    // lane-dependent offsets.  Per-pair order = the per-body order above:
    // bitwise the same sums.
    constexpr bool CL = GB == 32 && MODE != 3;
    double *st6 = &c6[0][0].x;
    auto tiles_cl = [&](int s, int t, auto &&fetch) {
        const int e0 = __shfl_sync(0xffffffffu, s, 0);
        const int e1 = __shfl_sync(0xffffffffu, t, last);
        int sr[6], tr[6];
#pragma unroll
        for (int r = 0; r < 6; ++r) {
            sr[r] = __shfl_sync(0xffffffffu, s, (32 * r + lane) / 6);
            tr[r] = __shfl_sync(0xffffffffu, t, (32 * r + lane) / 6);
        }
        double2 *st2 = reinterpret_cast<double2 *>(st6);
        for (int base = e0; base < e1; base += SCATTER_TILE) {
#pragma unroll
            for (int i = 0; i < SCATTER_TILE / 32; ++i) {
                const int e = base + lane + 32 * i;
                if (e < e1) {
                    const V6 v = fetch(e);
#pragma unroll
                    for (int k = 0; k < 3; ++k) st2[3 * (lane + 32 * i) + k] = make_double2(v.v[2 * k], v.v[2 * k + 1]);
                }
            }
            __syncwarp();
#if K6_CL == 2
            int lo[6], nn[6], mx = 0;
#pragma unroll
            for (int r = 0; r < 6; ++r) {
                lo[r] = max(sr[r], base) - base;
                nn[r] = min(tr[r], base + SCATTER_TILE) - base - lo[r];
                mx = max(mx, nn[r]);
                lo[r] = 6 * lo[r] + (32 * r + lane) % 6;
            }
            for (int jj = 0; jj < mx; ++jj)
#pragma unroll
                for (int r = 0; r < 6; ++r)
                    if (jj < nn[r]) f[r] += st6[lo[r] + 6 * jj];
#else
#pragma unroll
            for (int r = 0; r < 6; ++r) {
                const int lo = max(sr[r], base) - base, hi = min(tr[r], base + SCATTER_TILE) - base;
                const double *pr = st6 + (32 * r + lane) % 6;
                for (int j = lo; j < hi; ++j) f[r] += pr[6 * j];
            }
#endif
            __syncwarp();
        }
    };
#else
    constexpr bool CL = false;
    auto tiles_cl = [&](int, int, auto &&) {};
#endif
    if (MODE == 3) {
        if (own)
#pragma unroll
            for (int k = 0; k < 6; ++k) f[k] = Fa[k * nb + b];
    } else if (SORTED) {
        const int sa = own ? o.pa[b] : 0, ta_ = own ? o.pa[b + 1] : 0;
        auto fa = [&](int e) {
            const double xv = xeff_at<MODE>(xe, e);
            V6 v;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                v.v[k] = -o.cn[k * o.cap + e] * xv;
                v.v[3 + k] = -o.cta[k * o.cap + e] * xv;
            }
            return v;
        };
        if (CL) tiles_cl(sa, ta_, fa);
        else tiles(sa, ta_, fa);
    }
    const int s = own ? o.row_ptr[b] : 0, t = own ? o.row_ptr[b + 1] : 0;
    auto fb = [&](int e) {
        const double xv = xeff_at<MODE>(xe, o.ecid[e]);
        V6 v;
#pragma unroll
        for (int k = 0; k < 6; ++k) v.v[k] = o.ew[k * o.E + e] * xv;
        return v;
    };
    if (CL) tiles_cl(s, t, fb);
    else tiles(s, t, fb);
    double *flat = &c6[0][0].x;  // 3 * 65 double2 >= 2 * 192 doubles
    if (CL) {  // pair sums -> the owning lane's f[0..5]
#pragma unroll
        for (int r = 0; r < 6; ++r) flat[192 + 32 * r + lane] = f[r];
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 6; ++k) f[k] = flat[192 + 6 * lane + k];
        __syncwarp();
    }
    // U_b = W_b F_b ; staged through shared memory for a coalesced AoS store
    const double *W = o.W;
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
    for (int i = 0; i < (6 * GB + 31) / 32; ++i) {
        const int m = lane + 32 * i;
        if (m < nvals) {
            U[6 * b0 + m] = flat[m];
            if (Fout) Fout[6 * b0 + m] = flat[192 + m];
        }
    }
    __syncwarp();
}

// Rows of the LCP in one pass of K7 (constraint-major)
struct K7Rows {
    int64_t nc, cap, rs;
    const int32_t *ia, *ib;
    const double *n, *ta, *tb, *rc, *q;
    double s;
};

// row . [U_a; U_b]: compact planes (CR) or the store's planes
template <bool CR>
__device__ __forceinline__ double k7_row_dot(const K7Rows &r, int64_t a, const double *__restrict__ U) {
    return CR ? row_dot_c(a, r.rs, r.ia, r.ib, r.rc, U) : row_dot_u(a, r.cap, r.ia, r.ib, r.n, r.ta, r.tb, U);
}

// BB update of rows a0, a0 + stride, ... (ILP rows per thread and trip):
// reads the current slot (xc, gc; FIX: the blend with the other slot), writes
// x+, g+ into the other slot (xw, gw), accumulates
// acc = [s.s, s.y, y.y, max |min(x+, g+)|, non-finite flag, g.s].
template <bool CR, int ILP, bool FIX>
__device__ __forceinline__ void k7_rows(int64_t a_first, int64_t stride, const K7Rows &r,
                                        const double *__restrict__ U, double alpha, double tl, const double *xc,
                                        const double *gc, double *xw, double *gw, double (&acc)[6]) {
    const int64_t nc = r.nc;
    for (int64_t a0 = a_first; a0 < nc; a0 += ILP * stride) {
        double xo[ILP], go[ILP], qv[ILP], rd[ILP];
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            const int64_t a = a0 + u * stride;
            const bool ok = a < nc;
            const int64_t ac = ok ? a : a0;
            xo[u] = xc[ac];
            go[u] = gc[ac];
            if (FIX) {  // current iterate = blend of the two slots
                const double xp = xw[ac], gp = gw[ac];
                xo[u] = fma(tl, xo[u] - xp, xp);
                go[u] = fma(tl, go[u] - gp, gp);
            }
            qv[u] = r.q[ac];
            rd[u] = k7_row_dot<CR>(r, ac, U);
        }
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            const int64_t a = a0 + u * stride;
            if (a >= nc) continue;
            const double xn = fmax(0.0, xo[u] - alpha * go[u]);
            const double gn = fma(r.s, rd[u], qv[u]);
            xw[a] = xn;
            gw[a] = gn;
            const double sd = xn - xo[u], yd = gn - go[u];
            acc[0] = fma(sd, sd, acc[0]);
            acc[1] = fma(sd, yd, acc[1]);
            acc[2] = fma(yd, yd, acc[2]);
            acc[3] = fmax(acc[3], fabs(fmin(xn, gn)));
            acc[4] = fmax(acc[4], isfinite(gn) ? 0.0 : 1.0);
            acc[5] = fma(go[u], sd, acc[5]);
        }
    }
}
