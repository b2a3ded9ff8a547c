// Deterministic exclusive prefix sums (integer; used for the CSR row
// pointers, pair offsets and order-preserving stream compaction).
// Tile = 1024 threads x 4 items; levels recurse on the tile totals.
#include "common.cuh"

#define SCAN_NT 1024
#define SCAN_IPT 4
#define SCAN_TILE (SCAN_NT * SCAN_IPT)

template <class T>
__device__ __forceinline__ T block_excl_scan(T v, T *sh, T *total) {
    // warp inclusive scan
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (wid == 0) {
        T s = lane < (blockDim.x >> 5) ? sh[lane] : (T)0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        sh[lane] = s;  // inclusive warp totals
    }
    __syncthreads();
    T wofs = wid > 0 ? sh[wid - 1] : (T)0;
    if (total) *total = sh[(blockDim.x >> 5) - 1];
    T r = wofs + x - v;
    __syncthreads();
    return r;
}

template <class T>
__global__ void k_tile_sums(const T *__restrict__ in, int64_t n, T *__restrict__ sums) {
    __shared__ T sh[32];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
    T s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k)
        if (base + k < n) s += in[base + k];
    T tot;
    block_excl_scan<T>(s, sh, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

template <class T>
__global__ void k_tile_scan(const T *__restrict__ in, int64_t n, const T *__restrict__ offs, T *__restrict__ out,
                            T *__restrict__ total_out) {
    __shared__ T sh[32];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
    T v[SCAN_IPT];
    T s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
        v[k] = base + k < n ? in[base + k] : (T)0;
        s += v[k];
    }
    T tot;
    T ex = block_excl_scan<T>(s, sh, &tot);
    T o = (offs ? offs[blockIdx.x] : (T)0) + ex;
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
        if (base + k < n) out[base + k] = o;
        o += v[k];
    }
    if (total_out && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *total_out = (offs ? offs[blockIdx.x] : (T)0) + tot;
}

// out[i] = sum_{j<i} in[i]; *dev_total = sum (device).  scratch >= levels.
template <class T>
static cudaError_t scan_rec(cudaStream_t st, const T *in, T *out, int64_t n, T *dev_total, T *scratch) {
    int64_t nt = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (nt <= 1) {
        k_tile_scan<T><<<1, SCAN_NT, 0, st>>>(in, n, nullptr, out, dev_total);
        return cudaGetLastError();
    }
    T *sums = scratch, *offs = scratch + nt;
    k_tile_sums<T><<<(unsigned)nt, SCAN_NT, 0, st>>>(in, n, sums);
    cudaError_t e = scan_rec<T>(st, sums, offs, nt, nullptr, scratch + 2 * nt);
    if (e != cudaSuccess) return e;
    k_tile_scan<T><<<(unsigned)nt, SCAN_NT, 0, st>>>(in, n, offs, out, dev_total);
    return cudaGetLastError();
}

static int64_t scratch_need(int64_t n) {
    int64_t need = 1;
    while (n > SCAN_TILE) {
        n = (n + SCAN_TILE - 1) / SCAN_TILE;
        need += 2 * n;
    }
    return need + 8;
}

int scan_exclusive_ll(relcp_ctx *ctx, const long long *in, long long *out, int64_t n, long long *total_host) {
    if (n <= 0) {
        if (total_host) *total_host = 0;
        return RELCP_OK;
    }
    CK(ctx->scan_tmp.grow(scratch_need(n) + 1));
    long long *dtot = ctx->scan_tmp.p;
    CK(scan_rec<long long>(ctx->stream, in, out, n, dtot, ctx->scan_tmp.p + 1));
    if (total_host) {
        CK(cudaMemcpyAsync(ctx->red_host, dtot, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        memcpy(total_host, ctx->red_host, sizeof(long long));
    }
    return RELCP_OK;
}

int scan_exclusive_int(relcp_ctx *ctx, const int *in, int *out, int64_t n, int *total_host) {
    if (n <= 0) {
        if (total_host) *total_host = 0;
        return RELCP_OK;
    }
    // int scratch lives in the long-long scratch buffer (reinterpreted)
    CK(ctx->scan_tmp.grow(scratch_need(n) + 1));
    int *scr = (int *)ctx->scan_tmp.p;
    int *dtot = scr;
    CK(scan_rec<int>(ctx->stream, in, out, n, dtot, scr + 2));
    if (total_host) {
        CK(cudaMemcpyAsync(ctx->red_host, dtot, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        memcpy(total_host, ctx->red_host, sizeof(int));
    }
    return RELCP_OK;
}
