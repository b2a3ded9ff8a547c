// K6 with TMA bulk staging of per-group records (CSR layout, store sorted by
// ia; DESIGN.md §5 "K6 pipeline", params.k6_pipe).
//
// op_prepare packs, for every 32-body group, ONE contiguous record (k6r::*):
// the group's entry counts, the per-body bounds of its a-side rows and b-side
// entries, the W planes of its bodies, its a-side rows [n; t_a] (AoS, 48 B)
// and its b-side entries (ids, then the signed payload [n; t_b], AoS).  A
// persistent CTA owns a ring of K6P_STAGES shared-memory stages; warp 0
// streams each group's record plus the a-side ranges of x / g (the iterate,
// which changes every iteration) with cp.async.bulk into a stage, completion
// on one mbarrier per stage, K6P_STAGES - 1 groups ahead of the group being
// summed.  All threads then form each entry's contribution (lane per entry;
// the b-side x / g gathered at the entries' ids), and six warps sum one
// component each per body in k6_group's order (a-side rows, then b-side
// entries, one accumulator), so U is bitwise the per-warp kernel's.  Groups
// whose record exceeds a stage fall back to k6_group on warp 0.
//
// Measured (profiles/README.md): 0.53 ms vs 0.17 ms for the per-warp kernel at
// cfg5 A_0: two CTAs per SM sum ~2 groups at a time through a serial chain of
// shared-memory phases, where the per-warp kernel keeps 32 groups in flight.
// Kept as an option (params.k6_pipe = 1), bitwise equal; not the default.
#pragma once
#include "k6k7.cuh"

#ifndef K6P_REC_CAP
#define K6P_REC_CAP 20480  // record bytes per stage
#endif
#ifndef K6P_CAPG
#define K6P_CAPG 288       // b-side entries per stage with prefetched x / g gathers
#endif
#ifndef K6P_CAPA
#define K6P_CAPA 256       // a-side rows per stage (x / g planes)
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

namespace k6r {  // record layout (bytes)
constexpr int OFF_APOS = 64;                 // int[33]: a-side bounds relative to the group's first row
constexpr int OFF_BPOS = OFF_APOS + 144;     // int[33]: b-side bounds relative to the group's first entry
constexpr int OFF_W = OFF_BPOS + 144;        // 7 planes x 32 doubles
constexpr int OFF_A = OFF_W + 7 * 32 * 8;    // a-side rows, 6 doubles each
__host__ __device__ constexpr int64_t off_ids(int64_t na) { return OFF_A + 48 * na; }
__host__ __device__ constexpr int64_t off_b(int64_t na, int64_t nbe) { return off_ids(na) + ((4 * nbe + 15) & ~15ll); }
__host__ __device__ constexpr int64_t size(int64_t na, int64_t nbe) { return off_b(na, nbe) + 48 * nbe; }
// header ints: [0] na, [1] nbe, [2] bodies in the group, [3] first a-side row, [4] first b-side entry
}  // namespace k6r

namespace k6p {
constexpr int PD = K6P_CAPA + 2;                // doubles per staged x / g plane
constexpr int OFF_X = K6P_REC_CAP;              // 4 planes: x_c, g_c, x_p, g_p
constexpr int OFF_G = OFF_X + 4 * PD * 8;       // gathered x_c, g_c at the b-side ids (2 x K6P_CAPG)
constexpr int STAGE = OFF_G + 2 * K6P_CAPG * 8;
constexpr int SMEM = K6P_STAGES * STAGE;
}  // namespace k6p

struct K6PHdr {
    int ovf;
    int pad[4];  // element offsets of the x_c, g_c, x_p, g_p copies (16-B alignment)
};

__device__ __forceinline__ uint32_t k6p_smem(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// one bulk copy of n elements of esz bytes at src[i0..] into dst (16-B aligned);
// returns the element offset of src[i0] inside dst
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

// record sizes (bytes) per group
__global__ void k_k6r_size(int64_t nb, const int *__restrict__ pa, const int *__restrict__ row_ptr,
                           long long *__restrict__ sz) {
    const int64_t nw = (nb + 31) >> 5;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c0 = w << 5, c1 = c0 + 32 < nb ? c0 + 32 : nb;
        sz[w] = k6r::size(pa[c1] - pa[c0], row_ptr[c1] - row_ptr[c0]);
    }
}

// pack the records (one warp per group)
__global__ void k_k6r_fill(int64_t nb, const int *__restrict__ pa, const int *__restrict__ row_ptr,
                           const long long *__restrict__ off, const double *__restrict__ cn,
                           const double *__restrict__ cta, int64_t cap, const int *__restrict__ ecid,
                           const double *__restrict__ ew, int64_t E, const double *__restrict__ W,
                           unsigned char *__restrict__ rec) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (nb + 31) >> 5;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nw;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        unsigned char *r = rec + off[w];
        const int64_t c0 = w << 5, c1 = c0 + 32 < nb ? c0 + 32 : nb;
        const int nbody = (int)(c1 - c0);
        const int a0 = pa[c0], na = pa[c1] - a0, e0 = row_ptr[c0], nbe = row_ptr[c1] - e0;
        int *h = (int *)r;
        if (lane == 0) {
            h[0] = na; h[1] = nbe; h[2] = nbody; h[3] = a0; h[4] = e0;
        }
        int *apos = (int *)(r + k6r::OFF_APOS), *bpos = (int *)(r + k6r::OFF_BPOS);
        for (int l = lane; l <= 32; l += 32) {
            const int64_t b = c0 + (l < nbody ? l : nbody);
            apos[l] = pa[b] - a0;
            bpos[l] = row_ptr[b] - e0;
        }
        double *Wr = (double *)(r + k6r::OFF_W);
        for (int k = 0; k < 7; ++k) Wr[k * 32 + lane] = lane < nbody ? W[k * nb + c0 + lane] : 0.0;
        double *A = (double *)(r + k6r::OFF_A);
        for (int e = lane; e < na; e += 32)
            for (int k = 0; k < 3; ++k) {
                A[6 * e + k] = cn[k * cap + a0 + e];
                A[6 * e + 3 + k] = cta[k * cap + a0 + e];
            }
        int *ids = (int *)(r + k6r::off_ids(na));
        double *B = (double *)(r + k6r::off_b(na, nbe));
        for (int e = lane; e < nbe; e += 32) {
            ids[e] = ecid[e0 + e];
            for (int k = 0; k < 6; ++k) B[6 * e + k] = ew[k * E + e0 + e];
        }
    }
}

__device__ __forceinline__ void k6p_wait(uint64_t *bar, uint32_t ph) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(k6p_smem(bar)),
        "r"(ph)
        : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(K6P_NT, K6P_MINB) k_scatter_pipe(
    K6Op o, const unsigned char *__restrict__ rec, const long long *__restrict__ roff, const double *__restrict__ x,
    const double *__restrict__ g, const double *__restrict__ xb, const double *__restrict__ gb,
    const LcpState *__restrict__ st, const double *__restrict__ xscale, double *__restrict__ U,
    double *__restrict__ Fout) {
    extern __shared__ __align__(128) unsigned char k6p_dyn[];
    __shared__ __align__(8) uint64_t bar[K6P_STAGES];
    __shared__ K6PHdr hdr[K6P_STAGES];
    __shared__ double Fs[6][33];
    if (MODE != 0 && st->done) return;
    const XEff xe = xeff_setup<MODE>(st, x, g, xb, gb, xscale);
    const bool need_p = (MODE == 1 && xe.fix) || MODE == 2;  // the other slot is read
    const bool need_g = MODE != 0;
    // gathers prefetched for the plain apply and the unblended BB step (APGD and
    // the blended BB step read two slots: direct loads)
    const bool gpre = MODE == 0 || (MODE == 1 && !xe.fix);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t nb = o.nb, nwarp = (nb + 31) >> 5;
    const int64_t G = gridDim.x;
    auto grp = [&](int64_t i) -> int64_t {  // this CTA's i-th group (K6_REVERSE order)
        const int64_t q = blockIdx.x + i * G;
        return q < nwarp ? nwarp - 1 - q : -1;
    };
    if (tid == 0) {
        for (int s = 0; s < K6P_STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(k6p_smem(&bar[s])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // producer (warp 0, the same in every lane): record offsets / size and the
    // a-side row range of the next group, loaded one iteration ahead
    long long n_r0 = 0, n_r1 = 0;
    int n_a0 = 0, n_na = 0;
    auto load_next = [&](int64_t w) {
        if (w < 0) return;
        n_r0 = roff[w];
        n_r1 = roff[w + 1];
        const int64_t c0 = w << 5, c1 = c0 + 32 < nb ? c0 + 32 : nb;
        n_a0 = o.pa[c0];
        n_na = o.pa[c1] - n_a0;
    };
    auto issue = [&](int64_t i) {
        const int64_t w = grp(i);
        if (w < 0) return;
        const int s = (int)(i % K6P_STAGES);
        unsigned char *sb = k6p_dyn + (size_t)s * k6p::STAGE;
        K6PHdr &h = hdr[s];
        const int64_t rs = n_r1 - n_r0;
        const int ovf = rs > K6P_REC_CAP || n_na > K6P_CAPA;
        uint32_t bytes = 0;
        uint64_t *bb = &bar[s];
        double *X = (double *)(sb + k6p::OFF_X);
        int pd = -1;
        if (!ovf) {
            if (lane == 0) pd = k6p_copy(sb, rec, n_r0, rs, 1, bb, bytes);
            else if (lane == 1) pd = k6p_copy(X, xe.xc, n_a0, n_na, 8, bb, bytes);
            else if (lane == 2 && need_g) pd = k6p_copy(X + k6p::PD, xe.gc, n_a0, n_na, 8, bb, bytes);
            else if (lane == 3 && need_p) pd = k6p_copy(X + 2 * k6p::PD, xe.xp, n_a0, n_na, 8, bb, bytes);
            else if (lane == 4 && need_p) pd = k6p_copy(X + 3 * k6p::PD, xe.gp, n_a0, n_na, 8, bb, bytes);
            if (lane >= 1 && lane <= 4 && pd >= 0) h.pad[lane - 1] = pd;
        }
        if (lane == 0) h.ovf = ovf;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, d);
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(k6p_smem(bb)), "r"(bytes)
                         : "memory");
    };
    if (wid == 0) {
        for (int64_t i = 0; i < K6P_STAGES - 1; ++i) {
            load_next(grp(i));
            issue(i);
        }
        load_next(grp(K6P_STAGES - 1));
    }
    if (gpre && grp(0) >= 0) {  // group 0's gathers (the loop prefetches i + 1 from there on)
        k6p_wait(&bar[0], 0u);
        if (!hdr[0].ovf) {
            const int na0 = ((const int *)k6p_dyn)[0], nbe0 = ((const int *)k6p_dyn)[1];
            const int *ids0 = (const int *)(k6p_dyn + k6r::off_ids(na0));
            double *G0 = (double *)(k6p_dyn + k6p::OFF_G);
            for (int e = tid; e < nbe0 && e < K6P_CAPG; e += K6P_NT) {
                const int c = ids0[e];
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(k6p_smem(G0 + e)), "l"(xe.xc + c)
                             : "memory");
                if (MODE == 1)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(k6p_smem(G0 + K6P_CAPG + e)),
                                 "l"(xe.gc + c)
                                 : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int64_t i = 0;; ++i) {
        const int64_t w = grp(i);
        if (w < 0) break;
        const int s = (int)(i % K6P_STAGES);
        if (wid == 0) {
            // refill the stage released at the end of the previous group (generic-proxy
            // accesses ordered before the async-proxy writes); fetch the next bounds
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(i + K6P_STAGES - 1);
            load_next(grp(i + K6P_STAGES));
        }
        k6p_wait(&bar[s], (uint32_t)((i / K6P_STAGES) & 1));
        // prefetch the next group's b-side x / g gathers (cp.async, 8 B each) into its
        // stage: they land while this group is summed.  Thread t gathers the entries it
        // will consume (e = t, t + K6P_NT, ...), so its own cp.async.wait_group suffices.
        if (gpre) {
            const int64_t w1 = grp(i + 1);
            if (w1 >= 0) {
                const int s1 = (int)((i + 1) % K6P_STAGES);
                k6p_wait(&bar[s1], (uint32_t)(((i + 1) / K6P_STAGES) & 1));
                if (!hdr[s1].ovf) {
                    unsigned char *sb1 = k6p_dyn + (size_t)s1 * k6p::STAGE;
                    const int na1 = ((const int *)sb1)[0], nbe1 = ((const int *)sb1)[1];
                    const int *ids1 = (const int *)(sb1 + k6r::off_ids(na1));
                    double *G1 = (double *)(sb1 + k6p::OFF_G);
                    for (int e = tid; e < nbe1 && e < K6P_CAPG; e += K6P_NT) {
                        const int c = ids1[e];
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(k6p_smem(G1 + e)),
                                     "l"(xe.xc + c)
                                     : "memory");
                        if (MODE == 1)
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(k6p_smem(G1 + K6P_CAPG + e)),
                                         "l"(xe.gc + c)
                                         : "memory");
                    }
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group 1;" ::: "memory");  // this group's gathers (committed last round)
        }
        unsigned char *sb = k6p_dyn + (size_t)s * k6p::STAGE;
        const K6PHdr &h = hdr[s];
        const int64_t b0 = w << 5;
        if (h.ovf) {  // rare: the whole group on warp 0 from global memory (stage memory as staging)
            if (wid == 0) k6_group<MODE, true>(w, o, xe, reinterpret_cast<double2(*)[SCATTER_TILE + 1]>(sb), lane, U,
                                               Fout, nullptr);
            __syncthreads();
            continue;
        }
        const int *rh = (const int *)sb;
        const int na = rh[0], nbe = rh[1], nbody = rh[2];
        double *A = (double *)(sb + k6r::OFF_A);
        const int *ids = (const int *)(sb + k6r::off_ids(na));
        double *B = (double *)(sb + k6r::off_b(na, nbe));
        const double *X = (const double *)(sb + k6p::OFF_X);
        // phase 1: each entry's contribution, in place of its inputs
        for (int e = tid; e < na; e += K6P_NT) {
            double xv;
            {
                double x0 = X[h.pad[0] + e];
                if (MODE == 0) {
                    xv = x0;
                } else if (MODE == 1) {
                    double g0 = X[k6p::PD + h.pad[1] + e];
                    if (xe.fix) {
                        const double xq = X[2 * k6p::PD + h.pad[2] + e], gq = X[3 * k6p::PD + h.pad[3] + e];
                        x0 = fma(xe.tl, x0 - xq, xq);
                        g0 = fma(xe.tl, g0 - gq, gq);
                    }
                    xv = fmax(0.0, x0 - xe.alpha * g0);
                } else {
                    const double g0 = X[k6p::PD + h.pad[1] + e];
                    const double y = x0 + xe.beta * (x0 - X[2 * k6p::PD + h.pad[2] + e]);
                    const double gy = g0 + xe.beta * (g0 - X[3 * k6p::PD + h.pad[3] + e]);
                    xv = fmax(0.0, y - xe.alpha * gy);
                }
                xv *= xe.sc;
            }
            double2 *c = reinterpret_cast<double2 *>(A + 6 * e);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double2 v = c[k];
                c[k] = make_double2(-v.x * xv, -v.y * xv);
            }
        }
        const double *Gs = (const double *)(sb + k6p::OFF_G);
        for (int e = tid; e < nbe; e += K6P_NT) {
            double xv;
            if (gpre && e < K6P_CAPG) {
                const double x0 = Gs[e];
                xv = MODE == 0 ? x0 : fmax(0.0, x0 - xe.alpha * Gs[K6P_CAPG + e]);
                xv *= xe.sc;
            } else {
                xv = xeff_at<MODE>(xe, ids[e]);
            }
            double2 *c = reinterpret_cast<double2 *>(B + 6 * e);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double2 v = c[k];
                c[k] = make_double2(v.x * xv, v.y * xv);
            }
        }
        __syncthreads();
        // phase 2: warp k < 6 sums component k of its 32 bodies (k6_group's order)
        if (wid < 6) {
            const int k = wid;
            double f = 0.0;
            if (lane < nbody) {
                const int *apos = (const int *)(sb + k6r::OFF_APOS), *bpos = (const int *)(sb + k6r::OFF_BPOS);
                for (int j = apos[lane]; j < apos[lane + 1]; ++j) f += A[6 * j + k];
                for (int j = bpos[lane]; j < bpos[lane + 1]; ++j) f += B[6 * j + k];
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
                const double *Wd = (const double *)(sb + k6r::OFF_W);
                const double w0 = Wd[lane], s00 = Wd[32 + lane], s01 = Wd[64 + lane], s02 = Wd[96 + lane],
                             s11 = Wd[128 + lane], s12 = Wd[160 + lane], s22 = Wd[192 + lane];
                u[0] = w0 * f[0];
                u[1] = w0 * f[1];
                u[2] = w0 * f[2];
                u[3] = s00 * f[3] + s01 * f[4] + s02 * f[5];
                u[4] = s01 * f[3] + s11 * f[4] + s12 * f[5];
                u[5] = s02 * f[3] + s12 * f[4] + s22 * f[5];
            }
            __syncwarp();
            double *flat = &Fs[0][0];  // 198 doubles
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
