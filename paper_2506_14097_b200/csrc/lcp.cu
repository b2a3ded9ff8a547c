// LCP solve 0 <= g = A x + q  _|_  x >= 0, A = s D^T W D (Lemma 3,
// P:L280-299; CQP form P:L195-205) by Barzilai-Borwein projected gradient
// (the paper names only the family; reading R1):
//   alpha_0 = 1/L, L = ||A|| from power iterations;
//   x+ = max(0, x - alpha g);  g+ = A x+ + q;  s = x+ - x;  y = g+ - g;
//   alpha = s.s/s.y (BB1, even k) or s.y/y.y (BB2, odd k); 1/L if s.y <= 0;
//   stop when r = ||min(x+, g+)||_inf <= tol (R2).
//
// One iteration = two streaming kernels:
//   K6 scatter: U = W D max(0, x - alpha g)          (operator.cu, PROJ)
//   K7 gather : x+, g+ = s D^T U + q, s.s, s.y, y.y, r partials; the last
//               block finalizes alpha / convergence on the device.
// Kernels early-exit once LcpState.done is set, so the host enqueues
// `check_every` iterations blindly and reads the state once per batch.
#include <type_traits>

#include "common.cuh"
#include "reduce.cuh"

#include "rows.cuh"
#include "k6k7.cuh"
// row . [U_a; U_b]: compact planes when the operator holds them (CR), else the store
#define ROW_DOT(a) (CR ? row_dot_c((a), rs, ia, ib, rc, U) : row_dot_u((a), cap, ia, ib, n, ta, tb, U))
#ifndef ITER_MINB
#define ITER_MINB 4  // resident K7 blocks per SM (register budget); grid = 148 * ITER_MINB
#endif
#ifndef ITER_MINB_CR
#define ITER_MINB_CR 3  // K7 with compact rows: 1 row per thread and trip x 3 blocks of 256 (80 registers, 24
#endif                  // warps per SM).  Same-box A/B, K7 on cfg5 A_0 / the relaxed cfg5 store (us): ILP 1 x 3
                        // blocks 111.0 / 146.5; ILP 3 x 2 (round-2 default until the last session) 116.2 / 153.5;
                        // ILP 1 x 4 x 192 threads 111.3 / 146.7, 1 x 6 x 128 112.0 / 147.4, 1 x 5 x 128 (96 regs)
                        // 114.5 / 150.6, 1 x 7 x 128 115.3 / 151.5, 1 x 4 x 256 (64 regs, spills) 124.9 / 164.3,
                        // 2 x 3 127.2 / 168.6, 2 x 2 116.2 / 154.5, 4 x 2 139.5 / 186.4; ids one trip ahead
                        // (K7_IDPRE) +4 %.  cfg3 iteration 31.6 -> 31.7 us, cfg2 18.8 -> 18.0 us.
#ifndef APGD_MINB_CR
#define APGD_MINB_CR 2  // k_apgd_iter keeps 128 registers
#endif
#ifndef ITER_ILP_CR
#define ITER_ILP_CR 1
#endif
#ifndef ITER_ILP
#define ITER_ILP 2   // rows per thread per trip in K7
#endif
#ifndef ITER_NT_CR
#define ITER_NT_CR RELCP_NT  // threads per K7 block with compact rows
#endif
#define K7_NT(CR) ((CR) ? ITER_NT_CR : RELCP_NT)

__global__ void k_project(int64_t nc, double *x) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nc; a += (int64_t)gridDim.x * blockDim.x)
        x[a] = x[a] > 0.0 ? x[a] : 0.0;
}

__global__ void k_fill(int64_t n, double *v, double val) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x)
        v[a] = val;
}

__global__ void k_state_init(LcpState *st, int64_t nc, double tol, long long max_iter) {
    st->alpha = 0.0;
    st->L = 0.0;
    st->resid = 0.0;
    st->ss = st->sy = st->yy = 0.0;
    st->obj = 0.0;
    st->pnorm = nc > 0 ? 1.0 / sqrt((double)nc) : 0.0;
    st->tol = tol;
    st->iter = 0;
    st->max_iter = max_iter;
    st->done = 0;
    st->conv = 0;
    st->nan = 0;
    st->par = 0;
    st->theta = 1.0;
    st->beta = 0.0;
    st->f_cur = 0.0;
    for (int k = 0; k < RELCP_GLL_M; ++k) st->fhist[k] = -INFINITY;
    st->t_ls = 1.0;
    st->fix = 0;
    st->n_ls = 0;
}

// ---- finalize steps of the grid reductions (also applied by the domain-
// decomposed solve, dd.cu, to partials combined over all parts)
// acc = [max |min(x, g)|, nan flag, x^T (g + q)]
__device__ void lcp_init_finalize(LcpState *st, const double *acc) {
    double L = st->L > 0.0 && isfinite(st->L) ? st->L : 1.0;
    st->L = L;
    st->alpha = 1.0 / L;
    st->resid = acc[0];
    st->iter = 0;
    st->f_cur = 0.5 * acc[2];
    st->fhist[0] = st->f_cur;
    if (acc[1] > 0.0) {
        st->nan = 1;
        st->done = 1;
    } else if (acc[0] <= st->tol) {
        st->conv = 1;
        st->done = 1;
    } else if (st->max_iter <= 0) {
        st->done = 1;
    }
}

// g = s D^T U + q for the (projected) warm start; r_0; alpha_0 = 1/L.
template <bool CR>
__global__ void __launch_bounds__(RELCP_NT) k_lcp_init(int64_t nc, int64_t cap, const int32_t *__restrict__ ia,
                                                       const int32_t *__restrict__ ib, const double *__restrict__ n,
                                                       const double *__restrict__ ta, const double *__restrict__ tb,
                                                       int64_t rs, const double *__restrict__ rc,
                                                       const double *__restrict__ U, double s,
                                                       const double *__restrict__ q, const double *__restrict__ x,
                                                       double *__restrict__ g, double *part, unsigned *counter,
                                                       LcpState *st, double *acc_out) {
    __shared__ double sh[3 * 32];
    double acc[3] = {0.0, 0.0, 0.0};
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nc; a += (int64_t)gridDim.x * blockDim.x) {
        const double qa = q[a], xa = x[a];
        double gv = fma(s, ROW_DOT(a), qa);
        g[a] = gv;
        acc[0] = fmax(acc[0], fabs(fmin(xa, gv)));
        acc[1] = fmax(acc[1], isfinite(gv) ? 0.0 : 1.0);
        acc[2] = fma(xa, gv + qa, acc[2]);  // 2 f(x) = x^T (A x + 2 q)
    }
    const int ops[3] = {1, 1, 0};
    if (grid_reduce_last<3>(acc, ops, part, counter, sh) && threadIdx.x == 0) {
        if (acc_out) {  // domain decomposition: partials combined across parts first
            for (int k = 0; k < 3; ++k) acc_out[k] = acc[k];
            return;
        }
        lcp_init_finalize(st, acc);
    }
}

// acc = [s.s, s.y, y.y, max |min(x+, g+)|, nan flag, g.d]: BB step, GLL line
// search, convergence (see k_lcp_iter)
__device__ void bb_iter_finalize(LcpState *st, const double *acc) {
    const long long k = st->iter;
    st->ss = acc[0];
    st->sy = acc[1];
    st->yy = acc[2];
    st->resid = acc[3];
    st->iter = k + 1;
    if (acc[4] > 0.0 || !isfinite(acc[0]) || !isfinite(acc[1]) || !isfinite(acc[2]) || !isfinite(acc[5])) {
        st->nan = 1;
        st->done = 1;
        return;
    }
    st->par ^= 1;  // (x+, g+) is the written slot
    if (acc[3] <= st->tol) {  // the full step solves the LCP
        st->fix = 0;
        st->conv = 1;
        st->done = 1;
        return;
    }
    // nonmonotone line search along d = x+ - x (closed form, f quadratic)
    const double gd = acc[5], dAd = acc[1];
    double fmaxh = st->f_cur;
#pragma unroll
    for (int m = 0; m < RELCP_GLL_M; ++m) fmaxh = fmax(fmaxh, st->fhist[m]);
    double t = 1.0;
    if (!(st->f_cur + gd + 0.5 * dAd <= fmaxh + 1e-4 * gd) && dAd > 0.0) t = fmin(1.0, -gd / dAd);
    st->f_cur += t * gd + 0.5 * t * t * dAd;
    st->fhist[(k + 1) % RELCP_GLL_M] = st->f_cur;
    st->fix = t < 1.0;
    st->t_ls = t;
    st->n_ls += t < 1.0;
    // BB steps are invariant under the scaling s, y -> t s, t y
    double al = (acc[1] <= 0.0 || acc[2] == 0.0) ? 1.0 / st->L : ((k % 2 == 0) ? acc[0] / acc[1] : acc[1] / acc[2]);
    const double lo = 1e-10 / st->L, hi = 1e10 / st->L;
    st->alpha = fmin(hi, fmax(lo, al));
    if (k + 1 >= st->max_iter) st->done = 1;
}

// One BB projected-gradient update (the gather half of iteration k), with a
// nonmonotone (GLL) line search that makes plain BB globally convergent
// (spectral projected gradient, reading R1):
//   d = P(x - alpha g) - x,  f(x + t d) = f + t g.d + t^2/2 d.A d  (f quadratic,
//   f(x) = 1/2 x^T A x + q^T x; the LCP is its KKT system), so
//   the line search is closed form: t = 1 when
//   f + g.d + 1/2 s.y <= max(last M f) + gamma g.d, else t = -g.d / s.y (the
//   exact minimiser along d, which satisfies the Armijo test for gamma < 1/2).
// The iterate lives in two slots (x_k, g_k) and (x+, g+ = A x+ + q): the pass
// reads the current slot and writes the other one, and the parity bit flips.
// A shortened step (t < 1) is not written back: the next K6 / K7 read both
// slots and form x_k + t (x+ - x_k), g_k + t (g+ - g_k) on the fly (A is
// linear), so the common t = 1 iteration moves exactly the bytes of plain BB.
template <bool CR>
__global__ void __launch_bounds__(K7_NT(CR), CR ? ITER_MINB_CR : ITER_MINB) k_lcp_iter(int64_t nc, int64_t cap, const int32_t *__restrict__ ia,
                                                       const int32_t *__restrict__ ib, const double *__restrict__ n,
                                                       const double *__restrict__ ta, const double *__restrict__ tb,
                                                       int64_t rs, const double *__restrict__ rc,
                                                       const double *__restrict__ U, double s,
                                                       const double *__restrict__ q, double *xA, double *gA,
                                                       double *xB, double *gB, double *part, unsigned *counter,
                                                       LcpState *st, double *acc_out) {
    __shared__ double sh[6 * 32];
    pdl_wait();
    pdl_open();
    if (st->done) return;
    const double alpha = st->alpha;
    const bool fix = st->fix != 0;
    const double tl = st->t_ls;
    const double *xc = st->par ? xB : xA, *gc = st->par ? gB : gA;
    double *xw = st->par ? xA : xB, *gw = st->par ? gA : gB;  // the other slot: read (fix) then written
    double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t a_first = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const K7Rows r{nc, cap, rs, ia, ib, n, ta, tb, rc, q, s};
    // ILP constraints per thread per trip: independent loads in flight.  The
    // rare blended pass (fix) runs one row per trip to keep the register
    // budget of the common pass.
    if (fix)
        k7_rows<CR, 1, true>(a_first, stride, r, U, alpha, tl, xc, gc, xw, gw, acc);
    else
        k7_rows<CR, CR ? ITER_ILP_CR : ITER_ILP, false>(a_first, stride, r, U, alpha, tl, xc, gc, xw, gw, acc);
    const int ops[6] = {0, 0, 0, 1, 1, 0};
    if (grid_reduce_last<6>(acc, ops, part, counter, sh) && threadIdx.x == 0) {
        if (acc_out) {
            for (int k = 0; k < 6; ++k) acc_out[k] = acc[k];
            return;
        }
        bb_iter_finalize(st, acc);
    }
}

__device__ void bb_finish_finalize(LcpState *st, const double *acc) {
    st->resid = acc[0];
    st->fix = 0;
    st->conv = acc[0] <= st->tol;
}

// After a BB solve that ended on a shortened step (fix): the iterate is the
// blend of the two slots; write it into (x, g) and recompute the residual.
__global__ void __launch_bounds__(RELCP_NT) k_bb_finish(int64_t nc, double *x, double *g, const double *xo,
                                                        const double *go, double *part, unsigned *counter,
                                                        LcpState *st, double *acc_out) {
    __shared__ double sh[32];
    const double tl = st->t_ls;
    double acc[1] = {0.0};
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nc; a += (int64_t)gridDim.x * blockDim.x) {
        const double xv = fma(tl, x[a] - xo[a], xo[a]), gv = fma(tl, g[a] - go[a], go[a]);
        x[a] = xv;
        g[a] = gv;
        acc[0] = fmax(acc[0], fabs(fmin(xv, gv)));
    }
    const int ops[1] = {1};
    if (grid_reduce_last<1>(acc, ops, part, counter, sh) && threadIdx.x == 0) {
        if (acc_out) {
            acc_out[0] = acc[0];
            return;
        }
        bb_finish_finalize(st, acc);
    }
}

// APGD (NEXT rank 2): Nesterov-accelerated projected gradient with
// gradient-based adaptive restart, in lagged form so that each iteration is
// still one K6 + one K7 pass:
//   y = x + beta (x - x'),  g_y = g + beta (g - g')        (linearity of A)
//   x+ = max(0, y - t g_y),  g+ = A x+ + q                 (t = 1/(1.1 L))
//   restart (theta = 1, beta = 0) if g_y . (x+ - x) > 0, else
//   theta+ = (theta sqrt(theta^2 + 4) - theta^2) / 2,
//   beta+  = theta (1 - theta) / (theta^2 + theta+).
// The new iterate overwrites the previous one's slot; the parity bit flips.
template <bool CR>
__global__ void __launch_bounds__(RELCP_NT, CR ? APGD_MINB_CR : ITER_MINB) k_apgd_iter(
    int64_t nc, int64_t cap, const int32_t *__restrict__ ia, const int32_t *__restrict__ ib,
    const double *__restrict__ n, const double *__restrict__ ta, const double *__restrict__ tb, int64_t rs,
    const double *__restrict__ rc, const double *__restrict__ U, double s, const double *__restrict__ q, double *xA, double *gA, double *xB,
    double *gB, double *part, unsigned *counter, LcpState *st) {
    __shared__ double sh[3 * 32];
    pdl_wait();
    pdl_open();
    if (st->done) return;
    const double t = st->alpha, beta = st->beta;
    double *xc = xA, *gc = gA, *xp = xB, *gp = gB;
    if (st->par) {
        xc = xB; gc = gB; xp = xA; gp = gA;
    }
    double acc[3] = {0.0, 0.0, 0.0};
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nc; a += (int64_t)gridDim.x * blockDim.x) {
        const double x0 = xc[a], g0 = gc[a];
        const double y = x0 + beta * (x0 - xp[a]), gy = g0 + beta * (g0 - gp[a]);
        const double xn = fmax(0.0, y - t * gy);
        const double gn = fma(s, ROW_DOT(a), q[a]);
        xp[a] = xn;
        gp[a] = gn;
        acc[0] = fma(gy, xn - x0, acc[0]);
        acc[1] = fmax(acc[1], fabs(fmin(xn, gn)));
        acc[2] = fmax(acc[2], isfinite(gn) ? 0.0 : 1.0);
    }
    const int ops[3] = {0, 1, 1};
    if (grid_reduce_last<3>(acc, ops, part, counter, sh) && threadIdx.x == 0) {
        const long long k = st->iter;
        st->iter = k + 1;
        st->par ^= 1;  // the new iterate is current
        st->resid = acc[1];
        if (acc[2] > 0.0 || !isfinite(acc[0])) {
            st->nan = 1;
            st->done = 1;
            return;
        }
        if (acc[1] <= st->tol) {
            st->conv = 1;
            st->done = 1;
            return;
        }
        const double th = st->theta;
        if (acc[0] > 0.0) {  // adaptive restart
            st->theta = 1.0;
            st->beta = 0.0;
        } else {
            const double th1 = 0.5 * (th * sqrt(th * th + 4.0) - th * th);
            st->beta = th * (1.0 - th) / (th * th + th1);
            st->theta = th1;
        }
        if (k + 1 >= st->max_iter) st->done = 1;
    }
}

__global__ void k_apgd_setup(LcpState *st) {
    st->alpha = 1.0 / (1.1 * st->L);  // power iteration underestimates ||A|| slightly
    st->theta = 1.0;
    st->beta = 0.0;
    st->par = 0;
}

// obj = x^T (g - q) = x^T A x
__global__ void __launch_bounds__(RELCP_NT) k_objective(int64_t nc, const double *__restrict__ x,
                                                        const double *__restrict__ g, const double *__restrict__ q,
                                                        double *part, unsigned *counter, LcpState *st,
                                                        double *acc_out) {
    __shared__ double sh[32];
    double acc[1] = {0.0};
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nc; a += (int64_t)gridDim.x * blockDim.x)
        acc[0] = fma(x[a], g[a] - q[a], acc[0]);
    const int ops[1] = {0};
    if (grid_reduce_last<1>(acc, ops, part, counter, sh) && threadIdx.x == 0) {
        if (acc_out)
            acc_out[0] = acc[0];
        else
            st->obj = acc[0];
    }
}

__global__ void k_set_L(LcpState *st, double L) { st->L = L; }

static double op_scale(const relcp_ctx *ctx) {
    const double dt = ctx->p.dt;
    return ctx->p.dynamics == RELCP_INERTIAL ? dt * dt : dt;  // P:L553 vs P:L512
}

// ------------------------------------------------------------ small stores: one cluster runs the BB loop
// Small stores are latency-bound: two kernels of dependent load chains plus a
// grid-wide reduction, ~12 us per iteration at cfg1 against < 1 us of
// traffic.  Here ONE thread-block
// cluster of CL_CTAS CTAs (one per SM, non-portable size 16) runs `iters`
// whole BB iterations per launch: K6 (k6_group) on the cluster's warps ->
// cluster barrier -> K7 (k7_rows) -> each CTA's block partials into its own
// shared memory -> cluster barrier -> every CTA combines the CTAs' partials
// in rank order over distributed shared memory and runs the same finalize
// (bb_iter_finalize) on its own copy of the LCP state, so all CTAs take
// identical, deterministic steps with no third barrier (the next partials are
// written only after the next K6 barrier).  Hardware cluster barriers replace
// kernel boundaries and the grid's last-block reduction; U, x and g stay in
// L2 (the store is a few MB).
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#ifndef CL_CTAS
#define CL_CTAS 16
#endif
#ifndef CL_NT
#define CL_NT 512
#endif
#define CL_WARPS (CL_NT / 32)
// eligibility: at most one 32-body group per warp of the cluster and a store
// of <= 16k rows (cfg1: 11.8 -> 7.8 us per iteration; cfg2, 20k bodies / 31k
// rows: 15.1 -> 19.3 us, because 16 SMs then run 2-3 dependent K6 chains per
// warp where 148 SMs run one: the per-pass kernels stay above this size)
#ifndef RELCP_CLUSTER_MAX_ROWS
#define RELCP_CLUSTER_MAX_ROWS 16384
#endif
#define RELCP_CLUSTER_MAX_BODIES (CL_CTAS * CL_WARPS * 32)
#ifndef CL_FENCE
#define CL_FENCE 0  // extra gpu-scope fences before the cluster barriers (A/B)
#endif
#ifndef CL_ITERS
#define CL_ITERS 128  // BB iterations per cluster launch (host convergence read between launches)
#endif

template <bool SORTED, bool CR>
__global__ void __launch_bounds__(CL_NT, 1) k_bb_cluster(int iters, K6Op o, K7Rows r, double *xA, double *gA,
                                                         double *xB, double *gB, double *U, LcpState *gst) {
    extern __shared__ double2 cl_dyn[];  // CL_WARPS x K6_SMEM_D2: K6 staging
    __shared__ LcpState st;
    __shared__ double part[6];
    __shared__ double sh[6 * 32];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank(), ncta = cl.num_blocks();
    if (threadIdx.x == 0) st = *gst;
    __syncthreads();
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    auto c6 = reinterpret_cast<double2(*)[SCATTER_TILE + 1]>(cl_dyn + wl * K6_SMEM_D2);
    const int64_t nwarp = (o.nb + 31) >> 5;
    const int ops[6] = {0, 0, 0, 1, 1, 0};
    for (int it = 0; it < iters && !st.done; ++it) {
        // K6: U = W D max(0, x - alpha g) (the current slot, or the blend after a shortened step)
        const XEff xe = xeff_setup<1>(&st, xA, gA, xB, gB, nullptr);
        for (int64_t w = rank * CL_WARPS + wl; w < nwarp; w += (int64_t)ncta * CL_WARPS)
            k6_group<1, SORTED>(w, o, xe, c6, lane, U, nullptr, nullptr);
        if (CL_FENCE) __threadfence();
        cl.sync();  // barrier.cluster arrive (release) / wait (acquire): U visible to the cluster
        // K7: x+, g+ into the other slot, partials
        const bool par = st.par != 0;
        const double *xc = par ? xB : xA, *gc = par ? gB : gA;
        double *xw = par ? xA : xB, *gw = par ? gA : gB;
        double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        const int64_t first = (int64_t)rank * CL_NT + threadIdx.x, stride = (int64_t)ncta * CL_NT;
        if (st.fix)
            k7_rows<CR, 1, true>(first, stride, r, U, st.alpha, st.t_ls, xc, gc, xw, gw, acc);
        else
            k7_rows<CR, 2, false>(first, stride, r, U, st.alpha, st.t_ls, xc, gc, xw, gw, acc);
        block_reduce<6>(acc, ops, sh);
        if (threadIdx.x == 0)
#pragma unroll
            for (int k = 0; k < 6; ++k) part[k] = acc[k];
        if (CL_FENCE) __threadfence();
        cl.sync();
        if (threadIdx.x < 32) {
            // lane q reads CTA q's partials (one DSMEM round trip), then a
            // fixed shuffle tree: the same association in every CTA
            const unsigned q = threadIdx.x;
            double tot[6];
            const double *pq = cl.map_shared_rank(part, q < ncta ? q : 0);
#pragma unroll
            for (int k = 0; k < 6; ++k) tot[k] = q < ncta ? pq[k] : (ops[k] == 0 ? 0.0 : -INFINITY);
#pragma unroll
            for (int k = 0; k < 6; ++k) tot[k] = ops[k] == 0 ? warp_sum(tot[k]) : warp_max(tot[k]);
            if (threadIdx.x == 0) bb_iter_finalize(&st, tot);
        }
        __syncthreads();
    }
    if (rank == 0 && threadIdx.x == 0) *gst = st;
    cl.sync();  // no CTA leaves while another may still read its partials
}

// 1 when the cluster launch of k_bb_cluster is possible on this device (probed once)
static int cluster_probe(relcp_ctx *ctx) {
    if (ctx->cl_ok >= 0) return ctx->cl_ok;
    ctx->cl_ok = 0;
    const size_t dyn = sizeof(double2) * CL_WARPS * K6_SMEM_D2;
    void (*ks[4])(int, K6Op, K7Rows, double *, double *, double *, double *, double *, LcpState *) = {
        k_bb_cluster<true, true>, k_bb_cluster<true, false>, k_bb_cluster<false, true>, k_bb_cluster<false, false>};
    for (auto k : ks) {
        if (cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL_CTAS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(CL_CTAS);
    cfg.blockDim = dim3(CL_NT);
    cfg.dynamicSmemBytes = dyn;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, (void *)k_bb_cluster<true, true>, &cfg) != cudaSuccess || ncl < 1) {
        cudaGetLastError();
        return 0;
    }
    ctx->cl_ok = 1;
    return 1;
}

static int cluster_launch(relcp_ctx *ctx, int iters, bool sorted, bool cr, const K6Op &o, const K7Rows &r,
                          double *xA, double *gA, double *xB, double *gB) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL_CTAS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(CL_CTAS);
    cfg.blockDim = dim3(CL_NT);
    cfg.dynamicSmemBytes = sizeof(double2) * CL_WARPS * K6_SMEM_D2;
    cfg.stream = ctx->stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    double *U = ctx->U.p;
    LcpState *gst = ctx->st.p;
    if (sorted && cr) CK(cudaLaunchKernelEx(&cfg, k_bb_cluster<true, true>, iters, o, r, xA, gA, xB, gB, U, gst));
    else if (sorted) CK(cudaLaunchKernelEx(&cfg, k_bb_cluster<true, false>, iters, o, r, xA, gA, xB, gB, U, gst));
    else if (cr) CK(cudaLaunchKernelEx(&cfg, k_bb_cluster<false, true>, iters, o, r, xA, gA, xB, gB, U, gst));
    else CK(cudaLaunchKernelEx(&cfg, k_bb_cluster<false, false>, iters, o, r, xA, gA, xB, gB, U, gst));
    ++ctx->launches;
    return RELCP_OK;
}

// JDS layout: the solve's private slot-order view in / out
__global__ void k_jds_in(int64_t nc, const int *__restrict__ perm, const double *__restrict__ lam,
                         const double *__restrict__ q, double *__restrict__ x, double *__restrict__ qs) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nc; a += (int64_t)gridDim.x * blockDim.x) {
        const int r = perm[a];
        x[a] = lam[r];
        qs[a] = q[r];
    }
}
__global__ void k_jds_out(int64_t nc, const int *__restrict__ perm, const double *__restrict__ x,
                          const double *__restrict__ g, double *__restrict__ lam, double *__restrict__ gout) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nc; a += (int64_t)gridDim.x * blockDim.x) {
        const int r = perm[a];
        lam[r] = x[a];
        gout[r] = g[a];
    }
}

static int lcp_solve_view(relcp_ctx *ctx, const relcp_bodies *b, relcp_constraints *cs, relcp_solve_report *rep);

int lcp_solve(relcp_ctx *ctx, const relcp_bodies *b, relcp_constraints *cs, relcp_solve_report *rep) {
    const int64_t nc = cs->count, nb = b->n;
    if (!cs->q || !cs->lambda || !cs->g) return set_err(ctx, RELCP_E_ARG, "solve: q, lambda and g are required");
    if (ctx->op_nc != nc || ctx->op_nb != nb || ctx->op_key_ia != cs->ia) CKS(op_prepare(ctx, b, cs));
    if (ctx->op_jds && ctx->p.solver == RELCP_SOLVER_APGD_FUSED) {  // the fused row pass needs the CSR layout
        ctx->op_nc = -1;
        CKS(op_prepare(ctx, b, cs));
    }
    PHASE(ctx, "solve.prepare");
    if (!ctx->op_jds || nc == 0) return lcp_solve_view(ctx, b, cs, rep);
    // JDS: solve on the slot-order view (ids, q, lambda, g; compact rows in ctx->rc), then
    // write lambda and g back in the caller's row order
    CK(ctx->jq.grow(nc));
    CK(ctx->jx.grow(nc));
    CK(ctx->jg.grow(nc));
    k_jds_in<<<grid_for(nc), RELCP_NT, 0, ctx->stream>>>(nc, ctx->jperm.p, cs->lambda, cs->q, ctx->jx.p, ctx->jq.p);
    CKL();
    relcp_constraints v = *cs;
    v.ia = ctx->jia.p;
    v.ib = ctx->jib.p;
    v.q = ctx->jq.p;
    v.lambda = ctx->jx.p;
    v.g = ctx->jg.p;
    ++ctx->jds_solves;
    const int rc = lcp_solve_view(ctx, b, &v, rep);
    if (rc < 0 && rc != RELCP_E_NAN) return rc;
    k_jds_out<<<grid_for(nc), RELCP_NT, 0, ctx->stream>>>(nc, ctx->jperm.p, ctx->jx.p, ctx->jg.p, cs->lambda, cs->g);
    CKL();
    CK(cudaStreamSynchronize(ctx->stream));
    return rc;
}

// the solve proper on cs: the caller's store, or the JDS slot-order view (op_scatter slots)
static int lcp_solve_view(relcp_ctx *ctx, const relcp_bodies *b, relcp_constraints *cs, relcp_solve_report *rep) {
    const int64_t nc = cs->count, nb = b->n;
    const int sl = ctx->op_jds;  // x / g / q arrays of cs are in slot order
    CK(ctx->vtmp.grow(nc > 0 ? nc : 1));
    const double s = op_scale(ctx);
    cudaStream_t st = ctx->stream;
    k_state_init<<<1, 1, 0, st>>>(ctx->st.p, nc, ctx->p.lcp_tol, (long long)ctx->p.lcp_max_iter);
    CKL();
    if (nc == 0) {
        if (rep) memset(rep, 0, sizeof(*rep));
        if (rep) rep->converged = 1;
        CK(cudaMemsetAsync(ctx->U.p, 0, sizeof(double) * 6 * nb, st));
        CK(cudaStreamSynchronize(st));
        return RELCP_OK;
    }
    const int gridc = grid_for(nc, RELCP_NT, ITER_MINB);  // one wave of resident blocks
    k_project<<<gridc, RELCP_NT, 0, st>>>(nc, cs->lambda);
    CKL();
    // power iteration for L = ||A|| (alpha_0 = 1/L, R1).  A BB solve after an
    // augmentation of <= 1 % of the rows in the same step reuses the previous
    // L: the augmented A holds the previous one as a principal submatrix, so
    // ||A|| can only grow, by little; BB's first step is then at most slightly
    // long and the GLL line search guards it (R1).  APGD (step 1/(1.1 L))
    // always recomputes.
    const bool reuse_L = ctx->p.solver == RELCP_SOLVER_BB && ctx->L_reuse > 0.0 && isfinite(ctx->L_reuse) &&
                         nc >= ctx->L_reuse_nc && (double)nc <= 1.01 * (double)ctx->L_reuse_nc;
    if (reuse_L) {
        k_set_L<<<1, 1, 0, st>>>(ctx->st.p, ctx->L_reuse);
        CKL();
    }
    if (!reuse_L) {
        k_fill<<<gridc, RELCP_NT, 0, st>>>(nc, ctx->vtmp.p, 1.0);
        CKL();
    }
    for (int it = 0; it < (reuse_L ? 0 : ctx->p.power_iters); ++it) {
        CKS(op_scatter(ctx, nb, ctx->vtmp.p, nullptr, 0, &ctx->st.p->pnorm, ctx->U.p, nullptr, nullptr, nullptr, sl));
        CKS(op_gather_apply(ctx, cs, ctx->U.p, ctx->vtmp.p, s, 1));
    }
    PHASE(ctx, "solve.power");
    // g_0 = A x_0 + q
    CKS(op_scatter(ctx, nb, cs->lambda, nullptr, 0, nullptr, ctx->U.p, nullptr, nullptr, nullptr, sl));
    const bool cr = ctx->op_compact != 0;
    const int gridi = cr ? grid_for(nc, RELCP_NT, APGD_MINB_CR) : gridc;  // k_apgd_iter: one wave
    const int grid7 = cr ? grid_for(nc, ITER_NT_CR, ITER_MINB_CR) : gridc;  // K7 (k_lcp_iter)
#define ROWS_ARGS nc, cs->capacity, cs->ia, cs->ib, cs->n, cs->ta, cs->tb, ctx->op_rs, ctx->rc.p
    if (cr)
        k_lcp_init<true><<<gridc, RELCP_NT, 0, st>>>(ROWS_ARGS, ctx->U.p, s, cs->q, cs->lambda, cs->g, ctx->partials.p,
                                                     ctx->counter.p, ctx->st.p, nullptr);
    else
        k_lcp_init<false><<<gridc, RELCP_NT, 0, st>>>(ROWS_ARGS, ctx->U.p, s, cs->q, cs->lambda, cs->g,
                                                      ctx->partials.p, ctx->counter.p, ctx->st.p, nullptr);
    CKL();
    const bool apgd = ctx->p.solver == RELCP_SOLVER_APGD || (ctx->p.solver == RELCP_SOLVER_APGD_FUSED && !ctx->op_sorted);
    // fused APGD needs the sorted store (a-side rows contiguous); else plain APGD
    const bool fused = ctx->p.solver == RELCP_SOLVER_APGD_FUSED && ctx->op_sorted;
    double *xB = nullptr, *gB = nullptr;
    if (fused) {
        // second iterate slot x_{-1} = x_0 (beta_0 = 0 makes it irrelevant but
        // finite); theta = 1, beta = 0, t = 1/(1.1 L); U = W D x_0 is current
        CK(ctx->apgd_buf.grow(nc));
        xB = ctx->apgd_buf.p;
        CK(cudaMemcpyAsync(xB, cs->lambda, sizeof(double) * nc, cudaMemcpyDeviceToDevice, st));
        k_apgd_setup<<<1, 1, 0, st>>>(ctx->st.p);
        CKL();
    }
    const bool bb = !apgd && !fused;
    if (bb) {
        // second slot for (x+, g+) (k_lcp_iter); nothing to initialise: the
        // first pass reads slot A = (lambda, g) and writes it
        CK(ctx->apgd_buf.grow(2 * nc));
        xB = ctx->apgd_buf.p;
        gB = ctx->apgd_buf.p + nc;
    }
    if (apgd) {
        // second iterate buffer (x', g') = (x_0, g_0); theta = 1, beta = 0, t = 1/(1.1 L)
        CK(ctx->apgd_buf.grow(2 * nc));
        xB = ctx->apgd_buf.p;
        gB = ctx->apgd_buf.p + nc;
        CK(cudaMemcpyAsync(xB, cs->lambda, sizeof(double) * nc, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(gB, cs->g, sizeof(double) * nc, cudaMemcpyDeviceToDevice, st));
        k_apgd_setup<<<1, 1, 0, st>>>(ctx->st.p);
        CKL();
    }
    PHASE(ctx, "solve.init");
    int batch = ctx->p.check_every > 0 ? ctx->p.check_every : 32;
    if (ctx->timing) {
        if (batch > 64) batch = 64;
        if (!ctx->ev_ready) {
            for (int k = 0; k < 3 * 64 + 2; ++k) CK(cudaEventCreate(&ctx->ev[k]));
            ctx->ev_ready = 1;
        }
    }
    // small stores: the whole BB loop in one thread-block cluster (k_bb_cluster)
    const bool use_cl = bb && !ctx->op_jds && nc <= RELCP_CLUSTER_MAX_ROWS && nb <= RELCP_CLUSTER_MAX_BODIES &&
                        ctx->p.cluster != 0 && cluster_probe(ctx);
    bool cl_timed = false;
    K6Op k6o{};
    K7Rows k7r{};
    if (use_cl) {
        k6o = op_k6(ctx);
        k7r = K7Rows{nc, cs->capacity, ctx->op_rs, cs->ia, cs->ib, cs->n, cs->ta, cs->tb, ctx->rc.p, cs->q, s};
        ++ctx->cluster_solves;
    }
    long long it_before = 0;
    int pending = 0, batches = 0;
    bool capturing = false, graph_timed = false;
    cudaGraphExec_t gexec = nullptr;
    struct GraphGuard {  // destroys the replayed batch graph on every exit path
        cudaGraphExec_t &g;
        ~GraphGuard() {
            if (g) cudaGraphExecDestroy(g);
        }
    } graph_guard{gexec};
    // `batch` BB iterations: K6 (scatter + projection) then K7 (gather + update)
#ifndef RELCP_PDL
#define RELCP_PDL 1
#endif
    auto enqueue_batch = [&]() -> int {
        ctx->pdl = RELCP_PDL;  // K6 / K7 of the batch: programmatic dependent launches
        struct PdlOff {
            relcp_ctx *c;
            ~PdlOff() { c->pdl = 0; }
        } pdl_off{ctx};
        for (int j = 0; j < batch; ++j) {
            // per-kernel events only for direct (uncaptured) batches in timing mode
            const bool ev_on = ctx->timing && !capturing;
            if (fused) {
                // row pass (g_{k+1}, x_{k+2}, a-side sums) then the b-side scatter + W
                if (ev_on) CK(cudaEventRecord(ctx->ev[3 * j], st));
                CKS(op_fused_rows(ctx, cs, nb, s, cs->lambda, xB));
                if (ev_on) CK(cudaEventRecord(ctx->ev[3 * j + 1], st));
                CKS(op_scatter(ctx, nb, cs->lambda, nullptr, 3, nullptr, ctx->U.p, nullptr, xB, nullptr));
                if (ev_on) CK(cudaEventRecord(ctx->ev[3 * j + 2], st));
                continue;
            }
            if (ev_on) CK(cudaEventRecord(ctx->ev[3 * j], st));
            CKS(op_scatter(ctx, nb, cs->lambda, cs->g, apgd ? 2 : 1, nullptr, ctx->U.p, nullptr, xB, gB, sl));
            if (ev_on) CK(cudaEventRecord(ctx->ev[3 * j + 1], st));
            if (apgd && cr)
                CK(launch_k(ctx->pdl, k_apgd_iter<true>, gridi, RELCP_NT, 0, st, ROWS_ARGS, ctx->U.p, s, cs->q,
                            cs->lambda, cs->g, xB, gB, ctx->partials.p, ctx->counter.p, ctx->st.p));
            else if (apgd)
                CK(launch_k(ctx->pdl, k_apgd_iter<false>, gridi, RELCP_NT, 0, st, ROWS_ARGS, ctx->U.p, s, cs->q,
                            cs->lambda, cs->g, xB, gB, ctx->partials.p, ctx->counter.p, ctx->st.p));
            else if (cr)
                CK(launch_k(ctx->pdl, k_lcp_iter<true>, grid7, ITER_NT_CR, 0, st, ROWS_ARGS, ctx->U.p, s, cs->q,
                            cs->lambda, cs->g, xB, gB, ctx->partials.p, ctx->counter.p, ctx->st.p, (double *)nullptr));
            else
                CK(launch_k(ctx->pdl, k_lcp_iter<false>, gridi, RELCP_NT, 0, st, ROWS_ARGS, ctx->U.p, s, cs->q,
                            cs->lambda, cs->g, xB, gB, ctx->partials.p, ctx->counter.p, ctx->st.p, (double *)nullptr));
            CKL();
            if (ev_on) CK(cudaEventRecord(ctx->ev[3 * j + 2], st));
        }
        return RELCP_OK;
    };
    for (;;) {
        CK(cudaMemcpyAsync(ctx->st_host, ctx->st.p, sizeof(LcpState), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const long long executed = ctx->st_host->iter - it_before;
        ctx->lcp_iterations += executed;
        if (ctx->timing && pending > 0 && cl_timed) {
            // a cluster launch stops at convergence: its time covers exactly the executed iterations
            float a = 0.f;
            CK(cudaEventElapsedTime(&a, ctx->ev[3 * 64], ctx->ev[3 * 64 + 1]));
            if (executed > 0) {
                ctx->iter_ms += a;
                ctx->iter_timed += executed;
            }
        } else if (ctx->timing && pending > 0 && graph_timed) {
            // a graph batch counts only when every one of its iterations ran
            // (iterations after convergence exit at once and would dilute it)
            if (executed == pending) {
                float a = 0.f;
                CK(cudaEventElapsedTime(&a, ctx->ev[3 * 64], ctx->ev[3 * 64 + 1]));
                ctx->iter_ms += a;
                ctx->iter_timed += pending;
            }
        } else if (ctx->timing && pending > 0) {
            for (long long j = 0; j < executed && j < pending; ++j) {
                float a = 0.f, b2 = 0.f;
                CK(cudaEventElapsedTime(&a, ctx->ev[3 * j], ctx->ev[3 * j + 1]));
                CK(cudaEventElapsedTime(&b2, ctx->ev[3 * j + 1], ctx->ev[3 * j + 2]));
                ctx->scatter_ms += a;
                ctx->gather_ms += b2;
                ctx->iter_ms += a + b2;
                ++ctx->iter_timed;
                ++ctx->split_timed;
            }
        }
        it_before = ctx->st_host->iter;
        if (ctx->st_host->done) break;
        if (use_cl) {
            if (ctx->timing) CK(cudaEventRecord(ctx->ev[3 * 64], st));
            CKS(cluster_launch(ctx, CL_ITERS, ctx->op_sorted != 0, cr, k6o, k7r, cs->lambda, cs->g, xB, gB));
            if (ctx->timing) CK(cudaEventRecord(ctx->ev[3 * 64 + 1], st));
            cl_timed = true;
            ++batches;
            pending = CL_ITERS;
            continue;
        }
        if (!gexec && batches >= 1) {
            // the solve runs long: capture one batch as a CUDA graph, replay it
            cudaGraph_t graph = nullptr;
            CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            capturing = true;
            const int rc = enqueue_batch();
            capturing = false;
            cudaError_t ec = cudaStreamEndCapture(st, &graph);
            ctx->launches -= 2 * batch;  // captured, not executed
            if (rc < 0) return rc;
            CK(ec);
            ec = cudaGraphInstantiate(&gexec, graph, 0);
            cudaGraphDestroy(graph);
            CK(ec);
        }
        if (gexec) {
            if (ctx->timing) CK(cudaEventRecord(ctx->ev[3 * 64], st));
            CK(cudaGraphLaunch(gexec, st));
            if (ctx->timing) CK(cudaEventRecord(ctx->ev[3 * 64 + 1], st));
            graph_timed = true;
            ctx->launches += 2 * batch;
        } else {
            CKS(enqueue_batch());
        }
        ++batches;
        pending = batch;
    }
    PHASE(ctx, "solve.loop");
    if (gexec) {
        const cudaError_t e = cudaGraphExecDestroy(gexec);
        gexec = nullptr;
        CK(e);
    }
    if (bb && ctx->st_host->fix) {
        // ended on a shortened step: the iterate is x_k + t (x+ - x_k), x+ in the
        // current slot, x_k in the other one
        const bool pb = ctx->st_host->par != 0;
        k_bb_finish<<<gridc, RELCP_NT, 0, st>>>(nc, pb ? xB : cs->lambda, pb ? gB : cs->g, pb ? cs->lambda : xB,
                                                pb ? cs->g : gB, ctx->partials.p, ctx->counter.p, ctx->st.p, nullptr);
        CKL();
    }
    if (bb && ctx->st_host->par) {  // the current BB iterate lives in the second slot
        CK(cudaMemcpyAsync(cs->lambda, xB, sizeof(double) * nc, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(cs->g, gB, sizeof(double) * nc, cudaMemcpyDeviceToDevice, st));
    }
    if (apgd && ctx->st_host->par) {  // the current APGD iterate lives in the second buffer
        CK(cudaMemcpyAsync(cs->lambda, xB, sizeof(double) * nc, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(cs->g, gB, sizeof(double) * nc, cudaMemcpyDeviceToDevice, st));
    }
    if (fused && ctx->st_host->par)  // the current fused-BB iterate lives in the second slot
        CK(cudaMemcpyAsync(cs->lambda, xB, sizeof(double) * nc, cudaMemcpyDeviceToDevice, st));
    k_objective<<<gridc, RELCP_NT, 0, st>>>(nc, cs->lambda, cs->g, cs->q, ctx->partials.p, ctx->counter.p, ctx->st.p,
                                            nullptr);
    CKL();
    CK(cudaMemcpyAsync(ctx->st_host, ctx->st.p, sizeof(LcpState), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const LcpState &h = *ctx->st_host;
    if (rep) {
        rep->iterations = h.iter;
        rep->residual = h.resid;
        rep->converged = h.conv;
        rep->objective = -0.5 * h.obj;
        rep->L = h.L;
    }
    if (h.nan) return set_err(ctx, RELCP_E_NAN, "solve: non-finite iterate after %lld iterations", h.iter);
    if (!h.conv) return RELCP_W_MAX_ITER;
    return RELCP_OK;
}


// ------------------------------------------------------------ split reductions (dd.cu)
static const int kDDops[5][6] = {{0}, {1, 1, 0}, {0, 0, 0, 1, 1, 0}, {1}, {0}};
static const int kDDn[5] = {1, 3, 6, 1, 1};
int lcp_dd_nvals(int kind) { return kDDn[kind]; }
const int *lcp_dd_ops(int kind) { return kDDops[kind]; }
double lcp_scale(const relcp_ctx *ctx) { return op_scale(ctx); }

__global__ void k_dd_finalize(LcpState *st, int kind, const double *__restrict__ acc) {
    double a[6];
    for (int k = 0; k < 6; ++k) a[k] = k < 6 ? acc[k] : 0.0;
    if (kind == DD_POWER) power_finalize(st, a);
    else if (kind == DD_INIT) lcp_init_finalize(st, a);
    else if (kind == DD_ITER) {
        if (!st->done) bb_iter_finalize(st, a);
    } else if (kind == DD_FINISH) bb_finish_finalize(st, a);
    else st->obj = a[0];
}

int lcp_dd_state_init(relcp_ctx *ctx, int64_t nc_global) {
    k_state_init<<<1, 1, 0, ctx->stream>>>(ctx->st.p, nc_global, ctx->p.lcp_tol, (long long)ctx->p.lcp_max_iter);
    CKL();
    return RELCP_OK;
}

int lcp_dd_project_fill(relcp_ctx *ctx, int64_t nc, double *lambda, double *v, double val) {
    if (nc <= 0) return RELCP_OK;
    k_project<<<grid_for(nc, RELCP_NT, ITER_MINB), RELCP_NT, 0, ctx->stream>>>(nc, lambda);
    CKL();
    k_fill<<<grid_for(nc, RELCP_NT, ITER_MINB), RELCP_NT, 0, ctx->stream>>>(nc, v, val);
    CKL();
    return RELCP_OK;
}

int lcp_dd_init(relcp_ctx *ctx, const relcp_constraints *cs, double s, double *acc_out) {
    const int64_t nc = cs->count;
    const int gridc = grid_for(nc, RELCP_NT, ITER_MINB);
#define DD_ROWS nc, cs->capacity, cs->ia, cs->ib, cs->n, cs->ta, cs->tb, ctx->op_rs, ctx->rc.p
    if (ctx->op_compact)
        k_lcp_init<true><<<gridc, RELCP_NT, 0, ctx->stream>>>(DD_ROWS, ctx->U.p, s, cs->q, cs->lambda, cs->g,
                                                              ctx->partials.p, ctx->counter.p, ctx->st.p, acc_out);
    else
        k_lcp_init<false><<<gridc, RELCP_NT, 0, ctx->stream>>>(DD_ROWS, ctx->U.p, s, cs->q, cs->lambda, cs->g,
                                                               ctx->partials.p, ctx->counter.p, ctx->st.p, acc_out);
    CKL();
    return RELCP_OK;
}

int lcp_dd_iter(relcp_ctx *ctx, const relcp_constraints *cs, double s, double *xB, double *gB, double *acc_out) {
    const int64_t nc = cs->count;
    if (ctx->op_compact)
        k_lcp_iter<true><<<grid_for(nc, ITER_NT_CR, ITER_MINB_CR), ITER_NT_CR, 0, ctx->stream>>>(
            DD_ROWS, ctx->U.p, s, cs->q, cs->lambda, cs->g, xB, gB, ctx->partials.p, ctx->counter.p, ctx->st.p,
            acc_out);
    else
        k_lcp_iter<false><<<grid_for(nc, RELCP_NT, ITER_MINB), RELCP_NT, 0, ctx->stream>>>(
            DD_ROWS, ctx->U.p, s, cs->q, cs->lambda, cs->g, xB, gB, ctx->partials.p, ctx->counter.p, ctx->st.p,
            acc_out);
#undef DD_ROWS
    CKL();
    return RELCP_OK;
}

int lcp_dd_finish(relcp_ctx *ctx, int64_t nc, double *x, double *g, const double *xo, const double *go,
                  double *acc_out) {
    k_bb_finish<<<grid_for(nc, RELCP_NT, ITER_MINB), RELCP_NT, 0, ctx->stream>>>(nc, x, g, xo, go, ctx->partials.p,
                                                                                ctx->counter.p, ctx->st.p, acc_out);
    CKL();
    return RELCP_OK;
}

int lcp_dd_objective(relcp_ctx *ctx, int64_t nc, const double *x, const double *g, const double *q,
                     double *acc_out) {
    k_objective<<<grid_for(nc, RELCP_NT, ITER_MINB), RELCP_NT, 0, ctx->stream>>>(nc, x, g, q, ctx->partials.p,
                                                                                ctx->counter.p, ctx->st.p, acc_out);
    CKL();
    return RELCP_OK;
}

int lcp_dd_finalize(relcp_ctx *ctx, int kind, const double *acc_dev) {
    k_dd_finalize<<<1, 1, 0, ctx->stream>>>(ctx->st.p, kind, acc_dev);
    CKL();
    return RELCP_OK;
}
