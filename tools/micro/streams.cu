// Micro-benchmark: does HBM throughput depend on the number of concurrent SoA
// streams a row pass reads?  P planes of fp64 (stride n) against the same data
// blocked per 32 rows (one contiguous 32 * P * 8 byte chunk per warp load set).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o streams streams.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int P, bool BLOCKED, int ILP>
__global__ void __launch_bounds__(256) k(long n, const double *__restrict__ in, double *__restrict__ o1,
                                         double *__restrict__ o2) {
    const long stride = (long)gridDim.x * blockDim.x;
    for (long a0 = blockIdx.x * (long)blockDim.x + threadIdx.x; a0 < n; a0 += ILP * stride) {
        double v[ILP][P];
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            long a = a0 + u * stride;
            if (a >= n) a = a0;
#pragma unroll
            for (int p = 0; p < P; ++p)
                v[u][p] = BLOCKED ? in[(a >> 5) * (32 * P) + p * 32 + (a & 31)] : in[(long)p * n + a];
        }
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            const long a = a0 + u * stride;
            if (a >= n) continue;
            double s = 0, t = 1;
#pragma unroll
            for (int p = 0; p < P; ++p) {
                s += v[u][p];
                t = fma(t, 0.5, v[u][p]);
            }
            o1[a] = s;
            o2[a] = t;
        }
    }
}
template <int P, bool B, int ILP>
void run(long n, const double *in, double *o1, double *o2, int bps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = 148 * bps;
    for (int i = 0; i < 3; ++i) k<P, B, ILP><<<grid, 256>>>(n, in, o1, o2);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) k<P, B, ILP><<<grid, 256>>>(n, in, o1, o2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 20;
    printf("P=%2d %s ILP=%d blocks/SM=%d : %.1f us  %.0f GB/s\n", P, B ? "blocked" : "planes ", ILP, bps, 1e3 * ms,
           (P * 8.0 + 16.0) * n / ms / 1e6);
}
int main() {
    const long n = 8L << 20;
    double *in, *o1, *o2;
    cudaMalloc(&in, 16 * 8 * n);
    cudaMalloc(&o1, 8 * n);
    cudaMalloc(&o2, 8 * n);
    cudaMemset(in, 0, 16 * 8 * n);
    run<4, false, 2>(n, in, o1, o2, 8);
    run<12, false, 1>(n, in, o1, o2, 8);
    run<12, true, 1>(n, in, o1, o2, 8);
    run<12, false, 2>(n, in, o1, o2, 4);
    run<12, true, 2>(n, in, o1, o2, 4);
    run<12, false, 3>(n, in, o1, o2, 2);
    run<12, true, 3>(n, in, o1, o2, 2);
    run<12, false, 2>(n, in, o1, o2, 8);
    run<12, true, 2>(n, in, o1, o2, 8);
    if (cudaDeviceSynchronize() != cudaSuccess) return 1;
    return 0;
}
