// K6 with TMA bulk staging (CSR layout, store sorted by ia; DESIGN.md §5 "K6
// pipeline").  The per-warp kernel (k6_group) is bound by each 32-body group's
// chain of dependent loads.  Here a persistent CTA owns a ring of K6P_STAGES
// shared-memory stages; one thread streams whole groups into them with
// cp.async.bulk (the group's a-side rows [pa[b0], pa[b0 + 32]) of the n, t_a,
// x, g planes, its b-side CSR range [row_ptr[b0], row_ptr[b0 + 32]) of ids and
// payload, its W planes and both bound arrays: every range is contiguous),
// completion on one mbarrier per stage, K6P_STAGES - 1 groups ahead of the
// group being summed; the bounds of the group after that are loaded one
// iteration earlier still.  All threads then form each entry's contribution
// (lane per entry, gathers of x / g at the b-side ids), the segment sums per
// body run in the same order as k6_group (a-side rows, then b-side entries,
// one accumulator), so U is bitwise the per-warp kernel's.  Groups larger
// than a stage fall back to k6_group on warp 0.
//
// Measured (profiles/README.md): 0.75 ms vs 0.17 ms for the per-warp kernel
// at cfg5 A_0.  A 32-body group's data is ~26 separate ranges of 0.1-1 KB
// (SoA planes), and the bulk copies are paid per request: the stages arrive
// ~3x slower than the consumers drain them (ncu: 66 % of the warp samples
// waiting at the stage barrier).  Kept as an option (params.k6_pipe = 1) and
// parity-tested bitwise; not the default.
#pragma once
#include "k6k7.cuh"

#ifndef K6P_CAP
#define K6P_CAP 224  // entries per side and stage
#endif
#ifndef K6P_STAGES
#define K6P_STAGES 3
#endif
#ifndef K6P_NT
#define K6P_NT 256
#endif
#ifndef K6P_MINB
#define K6P_MINB 2
#endif

namespace k6p {
constexpr int PD = K6P_CAP + 2;                   // doubles per staged plane (16-byte alignment pad)
constexpr int A_PLANES = 10;                      // n (3), t_a (3), x_c, g_c, x_p, g_p
constexpr int B_PLANES = 6;                       // signed [n; t_b]
constexpr int OFF_A = 0;                          // bytes
constexpr int OFF_B = OFF_A + A_PLANES * PD * 8;  // payload planes
constexpr int OFF_ID = OFF_B + B_PLANES * PD * 8; // ids (K6P_CAP + 4 ints)
constexpr int OFF_W = OFF_ID + ((K6P_CAP + 4) * 4 + 15) / 16 * 16;
constexpr int WPD = 34;                           // doubles per staged W plane
constexpr int OFF_PA = OFF_W + 7 * WPD * 8;       // pa[b0 .. b0 + 32] (+ pad)
constexpr int OFF_RP = OFF_PA + 48 * 4;           // row_ptr[b0 .. b0 + 32]
constexpr int STAGE = OFF_RP + 48 * 4;
constexpr int SMEM = K6P_STAGES * STAGE;
}  // namespace k6p

struct K6PHdr {
    int a0, a1, b0, b1;  // entry ranges of the group
    int ovf;             // the group does not fit a stage: k6_group fallback
    int pad[K6P_STAGES > 0 ? 27 : 27];  // per-copy element offsets (alignment), see k6p_issue
};

__device__ __forceinline__ uint32_t k6p_smem(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// one bulk copy of n elements of esz bytes at src[i0..] into dst (16-B aligned
// stage region); returns the element offset of src[i0] inside dst
__device__ __forceinline__ int k6p_copy(void *dst, const void *src, int64_t i0, int64_t n, int esz, uint64_t *bar,
                                        uint32_t &bytes) {
    if (n <= 0) return 0;
    const uintptr_t s0 = (uintptr_t)src + (uintptr_t)(i0 * esz);
    const uintptr_t a0 = s0 & ~(uintptr_t)15;
    const uint32_t sz = (uint32_t)(((s0 - a0) + (uintptr_t)n * esz + 15) & ~(uintptr_t)15);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     k6p_smem(dst)),
                 "l"(a0), "r"(sz), "r"(k6p_smem(bar))
                 : "memory");
    bytes += sz;
    return (int)((s0 - a0) / esz);
}

template <int MODE>
__global__ void __launch_bounds__(K6P_NT, K6P_MINB) k_scatter_pipe(
    K6Op o, const double *__restrict__ x, const double *__restrict__ g, const double *__restrict__ xb,
    const double *__restrict__ gb, const LcpState *__restrict__ st, const double *__restrict__ xscale,
    double *__restrict__ U, double *__restrict__ Fout) {
    extern __shared__ __align__(128) unsigned char k6p_dyn[];
    __shared__ __align__(8) uint64_t bar[K6P_STAGES];
    __shared__ K6PHdr hdr[K6P_STAGES];
    __shared__ double Fs[6][33];
    if (MODE != 0 && st->done) return;
    const XEff xe = xeff_setup<MODE>(st, x, g, xb, gb, xscale);
    const bool need_p = (MODE == 1 && xe.fix) || MODE == 2;  // the other slot is read
    const bool need_g = MODE != 0;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t nb = o.nb, nwarp = (nb + 31) >> 5;
    const int64_t G = gridDim.x;
    // group index of this CTA's i-th group (K6_REVERSE order, like k_scatter)
    auto grp = [&](int64_t i) -> int64_t {
        const int64_t q = blockIdx.x + i * G;
        return q < nwarp ? nwarp - 1 - q : -1;
    };
    if (tid == 0) {
        for (int s = 0; s < K6P_STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(k6p_smem(&bar[s])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // producer state (warp 0, the same in every lane): bounds of the next group to issue
    int nx_a0 = 0, nx_a1 = 0, nx_b0 = 0, nx_b1 = 0;
    auto load_bounds = [&](int64_t w) {
        if (w < 0) return;
        const int64_t c0 = w << 5, c1 = c0 + 32 < nb ? c0 + 32 : nb;
        nx_a0 = o.pa[c0]; nx_a1 = o.pa[c1]; nx_b0 = o.row_ptr[c0]; nx_b1 = o.row_ptr[c1];
    };
    // group i into stage i % S: warp 0, one bulk copy per lane (bounds in nx_*,
    // identical in every lane of warp 0), the byte count summed over the warp
    auto issue = [&](int64_t i) {
        const int64_t w = grp(i);
        if (w < 0) return;
        const int s = (int)(i % K6P_STAGES);
        unsigned char *sb = k6p_dyn + (size_t)s * k6p::STAGE;
        K6PHdr &h = hdr[s];
        const int na = nx_a1 - nx_a0, nbe = nx_b1 - nx_b0;
        const int ovf = na > K6P_CAP || nbe > K6P_CAP;
        if (lane == 0) {
            h.a0 = nx_a0; h.a1 = nx_a1; h.b0 = nx_b0; h.b1 = nx_b1;
            h.ovf = ovf;
        }
        uint32_t bytes = 0;
        uint64_t *bb = &bar[s];
        const int64_t c0 = w << 5, nbody = c0 + 32 < nb ? 32 : nb - c0;
        double *A = (double *)(sb + k6p::OFF_A), *B = (double *)(sb + k6p::OFF_B);
        double *Wd = (double *)(sb + k6p::OFF_W);
        const int l = lane;
        int pd = -1;
        if (!ovf && l < 3) pd = k6p_copy(A + l * k6p::PD, o.cn + l * o.cap, nx_a0, na, 8, bb, bytes);
        else if (!ovf && l < 6) pd = k6p_copy(A + l * k6p::PD, o.cta + (l - 3) * o.cap, nx_a0, na, 8, bb, bytes);
        else if (!ovf && l == 6) pd = k6p_copy(A + 6 * k6p::PD, xe.xc, nx_a0, na, 8, bb, bytes);
        else if (!ovf && l == 7 && need_g) pd = k6p_copy(A + 7 * k6p::PD, xe.gc, nx_a0, na, 8, bb, bytes);
        else if (!ovf && l == 8 && need_p) pd = k6p_copy(A + 8 * k6p::PD, xe.xp, nx_a0, na, 8, bb, bytes);
        else if (!ovf && l == 9 && need_p) pd = k6p_copy(A + 9 * k6p::PD, xe.gp, nx_a0, na, 8, bb, bytes);
        else if (!ovf && l >= 10 && l < 16)
            pd = k6p_copy(B + (l - 10) * k6p::PD, o.ew + (l - 10) * o.E, nx_b0, nbe, 8, bb, bytes);
        else if (!ovf && l == 16) pd = k6p_copy(sb + k6p::OFF_ID, o.ecid, nx_b0, nbe, 4, bb, bytes);
        else if (l >= 17 && l < 24) pd = k6p_copy(Wd + (l - 17) * k6p::WPD, o.W + (l - 17) * nb, c0, nbody, 8, bb, bytes);
        else if (l == 24) pd = k6p_copy(sb + k6p::OFF_PA, o.pa, c0, nbody + 1, 4, bb, bytes);
        else if (l == 25) pd = k6p_copy(sb + k6p::OFF_RP, o.row_ptr, c0, nbody + 1, 4, bb, bytes);
        if (pd >= 0 && l < 27) h.pad[l] = pd;
        #pragma unroll
        for (int d = 16; d > 0; d >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, d);
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(k6p_smem(bb)), "r"(bytes)
                         : "memory");
    };
    // prologue: groups 0 .. S-2 issued, bounds of group S-1 loaded (warp 0)
    if (wid == 0) {
        for (int64_t i = 0; i < K6P_STAGES - 1; ++i) {
            load_bounds(grp(i));
            issue(i);
        }
        load_bounds(grp(K6P_STAGES - 1));
    }
    for (int64_t i = 0;; ++i) {
        const int64_t w = grp(i);
        if (w < 0) break;
        const int s = (int)(i % K6P_STAGES);
        if (wid == 0) {
            // refill the stage released at the end of the previous group (generic-proxy
            // accesses ordered before the async-proxy writes), then fetch the bounds of
            // the group after it
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(i + K6P_STAGES - 1);
            load_bounds(grp(i + K6P_STAGES));
        }
        {
            const uint32_t ph = (uint32_t)((i / K6P_STAGES) & 1);
            asm volatile(
                "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                "@!P1 bra WAIT_%=;\n\t}" ::"r"(k6p_smem(&bar[s])),
                "r"(ph)
                : "memory");
        }
        unsigned char *sb = k6p_dyn + (size_t)s * k6p::STAGE;
        const K6PHdr &h = hdr[s];
        const int64_t b0 = w << 5;
        const int nbody = b0 + 32 < nb ? 32 : (int)(nb - b0);
        if (h.ovf) {  // rare: the whole group on warp 0 from global memory (stage memory as staging)
            if (wid == 0) k6_group<MODE, true>(w, o, xe, reinterpret_cast<double2(*)[SCATTER_TILE + 1]>(sb), lane, U,
                                               Fout, nullptr);
            __syncthreads();
            continue;
        }
        const int na = h.a1 - h.a0, nbe = h.b1 - h.b0;
        double *A = (double *)(sb + k6p::OFF_A), *B = (double *)(sb + k6p::OFF_B);
        const int *ids = (const int *)(sb + k6p::OFF_ID) + h.pad[16];
        // phase 1: each entry's contribution, in place of its inputs
        for (int e = tid; e < na; e += K6P_NT) {
            double xv;
            {
                double x0 = A[6 * k6p::PD + h.pad[6] + e];
                if (MODE == 0) {
                    xv = x0;
                } else if (MODE == 1) {
                    double g0 = A[7 * k6p::PD + h.pad[7] + e];
                    if (xe.fix) {
                        const double xq = A[8 * k6p::PD + h.pad[8] + e], gq = A[9 * k6p::PD + h.pad[9] + e];
                        x0 = fma(xe.tl, x0 - xq, xq);
                        g0 = fma(xe.tl, g0 - gq, gq);
                    }
                    xv = fmax(0.0, x0 - xe.alpha * g0);
                } else {
                    const double g0 = A[7 * k6p::PD + h.pad[7] + e];
                    const double y = x0 + xe.beta * (x0 - A[8 * k6p::PD + h.pad[8] + e]);
                    const double gy = g0 + xe.beta * (g0 - A[9 * k6p::PD + h.pad[9] + e]);
                    xv = fmax(0.0, y - xe.alpha * gy);
                }
                xv *= xe.sc;
            }
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                double &c = A[k * k6p::PD + h.pad[k] + e];
                c = -c * xv;
            }
        }
        for (int e = tid; e < nbe; e += K6P_NT) {
            const double xv = xeff_at<MODE>(xe, ids[e]);
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                double &c = B[k * k6p::PD + h.pad[10 + k] + e];
                c = c * xv;
            }
        }
        __syncthreads();
        // phase 2: warp k < 6 sums component k of its 32 bodies (a-side rows,
        // then b-side entries: k6_group's order)
        if (wid < 6) {
            const int k = wid;
            double f = 0.0;
            if (lane < nbody) {
                const int *pa_s = (const int *)(sb + k6p::OFF_PA) + h.pad[24];
                const int *rp_s = (const int *)(sb + k6p::OFF_RP) + h.pad[25];
                const double *ca = A + k * k6p::PD + h.pad[k] - h.a0;
                for (int j = pa_s[lane]; j < pa_s[lane + 1]; ++j) f += ca[j];
                const double *cb = B + k * k6p::PD + h.pad[10 + k] - h.b0;
                for (int j = rp_s[lane]; j < rp_s[lane + 1]; ++j) f += cb[j];
            }
            Fs[k][lane] = f;
        }
        __syncthreads();
        // phase 3: U_b = W_b F_b, coalesced AoS stores through the F staging
        if (tid < 32) {
            double u[6] = {0, 0, 0, 0, 0, 0}, f[6];
#pragma unroll
            for (int k = 0; k < 6; ++k) f[k] = Fs[k][lane];
            if (lane < nbody) {
                const double *Wd = (const double *)(sb + k6p::OFF_W);
                auto Wk = [&](int k) { return Wd[k * k6p::WPD + h.pad[17 + k] + lane]; };
                const double w0 = Wk(0), s00 = Wk(1), s01 = Wk(2), s02 = Wk(3), s11 = Wk(4), s12 = Wk(5),
                             s22 = Wk(6);
                u[0] = w0 * f[0];
                u[1] = w0 * f[1];
                u[2] = w0 * f[2];
                u[3] = s00 * f[3] + s01 * f[4] + s02 * f[5];
                u[4] = s01 * f[3] + s11 * f[4] + s12 * f[5];
                u[5] = s02 * f[3] + s12 * f[4] + s22 * f[5];
            }
            __syncwarp();
            double *flat = &Fs[0][0];  // 198 doubles: U staged after F was read
#pragma unroll
            for (int k = 0; k < 6; ++k) flat[6 * lane + k] = u[k];
            __syncwarp();
            const int nvals = 6 * nbody;
#pragma unroll
            for (int t = 0; t < 6; ++t) {
                const int m = lane + 32 * t;
                if (m < nvals) U[6 * b0 + m] = flat[m];
            }
            if (Fout) {
                __syncwarp();
#pragma unroll
                for (int k = 0; k < 6; ++k) flat[6 * lane + k] = f[k];
                __syncwarp();
#pragma unroll
                for (int t = 0; t < 6; ++t) {
                    const int m = lane + 32 * t;
                    if (m < nvals) Fout[6 * b0 + m] = flat[m];
                }
            }
        }
        __syncthreads();  // the stage is free for the producer
    }
}
