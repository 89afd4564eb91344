// gather_lab.cu -- ceiling of the random-banded (C5) SpMM's x gathers on B200.
//
// C5 (BASELINE.json): n = 8M rows, 16-32 nonzeros per row, columns uniform in
// a band of +-65536.  Every nonzero gathers one x row (m*8 bytes) at a random
// position of a ~131K-row window: no reuse inside an SM, all reuse in L2.
// This lab times, with the SpMM's lane layout (m/2 lanes per row, 16-byte
// loads, 4 gathers in flight per lane):
//   gather   : 24 gathers per row, column indices hashed in registers (no
//              matrix stream) -- the L2 gather ceiling
//   stream   : the matrix stream alone (12 B per nonzero + x/y once)
//   both     : gathers with indices/values streamed from HBM (the SpMM's work
//              without the ordered-sum constraint)
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/gather_lab.cu -o build/gather_lab
// ./build/gather_lab [m=8]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e = (x);                                                         \
        if (e != cudaSuccess) {                                                      \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                 \
        }                                                                            \
    } while (0)

constexpr int64_t N = 8000000;
constexpr int K = 24;          // nonzeros per row (C5 average)
constexpr int BAND = 65536;

__device__ __forceinline__ uint32_t hash32(uint32_t a) {
    a ^= a >> 16;
    a *= 0x7feb352dU;
    a ^= a >> 15;
    a *= 0x846ca68bU;
    a ^= a >> 16;
    return a;
}

__device__ __forceinline__ int col_of(int64_t row, int k) {
    const uint32_t h = hash32(static_cast<uint32_t>(row) * 40503u + static_cast<uint32_t>(k) * 2654435761u);
    int64_t c = row - BAND + static_cast<int64_t>(h % (2 * BAND + 1));
    if (c < 0) c = -c;
    if (c >= N) c = 2 * (N - 1) - c;
    return static_cast<int>(c);
}

template <int M, int MODE>   // MODE 0 gather (hashed cols), 1 stream only, 2 gather + stream
__global__ void __launch_bounds__(256) lab_kernel(const double* __restrict__ x, double* __restrict__ y,
                                                  const int32_t* __restrict__ col, const double* __restrict__ val) {
    constexpr int LPR = M / 2, RPB = 256 / LPR;
    const int cp = (threadIdx.x % LPR) * 2;
    for (int64_t row = static_cast<int64_t>(blockIdx.x) * RPB + threadIdx.x / LPR; row < N;
         row += static_cast<int64_t>(gridDim.x) * RPB) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int k = 0; k < K; k += 4) {
            int j[4];
            double v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (MODE == 0) {
                    j[q] = col_of(row, k + q);
                    v[q] = 1.0;
                } else {
                    j[q] = __ldg(col + row * K + k + q);
                    v[q] = __ldg(val + row * K + k + q);
                }
            }
            if (MODE == 1) {
#pragma unroll
                for (int q = 0; q < 4; ++q) a0 += v[q] * j[q];
            } else {
                double2 xs[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) xs[q] = __ldg(reinterpret_cast<const double2*>(x + static_cast<int64_t>(j[q]) * M + cp));
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    a0 += v[q] * xs[q].x;
                    a1 += v[q] * xs[q].y;
                }
            }
        }
        *reinterpret_cast<double2*>(y + row * M + cp) = make_double2(a0, a1);
    }
}

__global__ void fill_cols(int32_t* col, double* val) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < N * K;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        col[e] = col_of(e / K, static_cast<int>(e % K));
        val[e] = 1.0;
    }
}

template <int M, int MODE>
float run(const double* x, double* y, const int32_t* col, const double* val, int grid) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int i = 0; i < 3; ++i) lab_kernel<M, MODE><<<grid, 256>>>(x, y, col, val);
    CK(cudaEventRecord(a));
    const int reps = 10;
    for (int i = 0; i < reps; ++i) lab_kernel<M, MODE><<<grid, 256>>>(x, y, col, val);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms / reps;
}

template <int M>
void lab() {
    double *x, *y, *val;
    int32_t* col;
    CK(cudaMalloc(&x, N * M * 8));
    CK(cudaMalloc(&y, N * M * 8));
    CK(cudaMalloc(&col, N * K * 4));
    CK(cudaMalloc(&val, N * K * 8));
    CK(cudaMemset(x, 0, N * M * 8));
    fill_cols<<<148 * 8, 256>>>(col, val);
    CK(cudaDeviceSynchronize());
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int grid = sms * 8;
    const double gath = static_cast<double>(N) * K * M * 8;   // bytes gathered (L2 -> SM)
    const double comp = 16.0 * N * M + 12.0 * N * K;          // compulsory DRAM bytes
    const float t0 = run<M, 0>(x, y, col, val, grid);
    const float t1 = run<M, 1>(x, y, col, val, grid);
    const float t2 = run<M, 2>(x, y, col, val, grid);
    printf("m=%d gather-only %.3f ms (%.1f TB/s gathered)  stream-only %.3f ms  gather+stream %.3f ms "
           "(%.1f TB/s gathered, %.2f TB/s compulsory)\n",
           M, t0, gath / t0 / 1e9, t1, t2, gath / t2 / 1e9, comp / t2 / 1e9);
    CK(cudaFree(x));
    CK(cudaFree(y));
    CK(cudaFree(col));
    CK(cudaFree(val));
}

int main(int argc, char** argv) {
    const int m = argc > 1 ? atoi(argv[1]) : 8;
    if (m == 8) lab<8>();
    else if (m == 16) lab<16>();
    else lab<32>();
    return 0;
}
