// lsu_tex_lab.cu -- does feeding the CSR SpMM's column / value reads through the
// texture pipe take them off the load/store data pipe that bounds the m = 8
// kernel (profiles/r02y_ncu_c5_spmm.md)?
//
// Every warp repeats the m = 8 kernel's memory pattern: per "batch" 4 gathers of
// 8 random 64-byte x rows (4 lanes x 16 bytes per row, L2-resident window) and
// the batch's 4 columns + 4 values (48 bytes per row, the same for a row's 4 lanes):
//   none    gathers only (the floor: one 64-byte wavefront per nonzero)
//   shared  three 16-byte shared-memory loads per lane (what the kernel does)
//   tex     three 16-byte tex1Dfetch<int4> from a linear texture (quad-uniform)
//   ldg     three 16-byte ld.global.nc loads (quad-uniform)
// Reported: ns per batch per SM and the gather rate in TB/s.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/lsu_tex_lab tools/lsu_tex_lab.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                               \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess) {                                                            \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                                   \
        }                                                                                   \
    } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t h) {
    h ^= h >> 16;
    h *= 0x7feb352dU;
    h ^= h >> 15;
    h *= 0x846ca68bU;
    h ^= h >> 16;
    return h;
}

template <int MODE>
__global__ void __launch_bounds__(256, 4) k(const double2* __restrict__ x, uint32_t nrows, const int4* __restrict__ mat,
                                            cudaTextureObject_t tex, uint32_t nmat, int iters, double* sink) {
    extern __shared__ int4 sm[];
    const int lane = threadIdx.x & 31, grp = lane >> 2, part = lane & 3;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (MODE == 1)
        for (int i = threadIdx.x; i < 3072; i += 256) sm[i] = make_int4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    double acc = 0.0;
    uint32_t mrow = (gw * 8u + grp) * 97u;   // this row's stream of (cols, vals) chunks
    for (int it = 0; it < iters; ++it) {
        int4 c = make_int4(0, 0, 0, 0), v0 = c, v1 = c;
        if (MODE == 1) {
            const int b = ((threadIdx.x >> 2) * 13 + it * 3) % 3069;
            c = sm[b];
            v0 = sm[b + 1];
            v1 = sm[b + 2];
        } else if (MODE == 2) {
            const int b = static_cast<int>((mrow + it * 3u) % (nmat - 3));
            c = tex1Dfetch<int4>(tex, b);
            v0 = tex1Dfetch<int4>(tex, b + 1);
            v1 = tex1Dfetch<int4>(tex, b + 2);
        } else if (MODE == 3) {
            const uint32_t b = (mrow + it * 3u) % (nmat - 3);
            c = __ldg(mat + b);
            v0 = __ldg(mat + b + 1);
            v1 = __ldg(mat + b + 2);
        }
        const uint32_t salt = c.x + v0.y + v1.z;   // a data dependence, as the gathers depend on the columns
        double2 g[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t r = mix(gw * 0x9E3779B9u + static_cast<uint32_t>(it) * 131u + grp * 7u + q * 977u + (salt & 1u)) % nrows;
            g[q] = __ldg(x + static_cast<int64_t>(r) * 4 + part);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) acc += g[q].x * __int_as_float(v0.x) + g[q].y;
    }
    if (acc == 1.2345) sink[0] = acc;
}

// The same nonzeros with 32 bytes of x per lane (ld.global.nc.v4.f64, LDG.E.256):
// 2 lanes per row, 16 rows per warp, the batch's columns / values from shared
// memory as in mode "shared" (one 16-byte chunk triple per row).
__global__ void __launch_bounds__(256, 3) k256(const double* __restrict__ x, uint32_t nrows, int iters, double* sink) {
    extern __shared__ int4 sm[];
    const int lane = threadIdx.x & 31, grp = lane >> 1, part = lane & 1;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int i = threadIdx.x; i < 3072; i += 256) sm[i] = make_int4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        const int b = ((threadIdx.x >> 1) * 3 + it * 3) % 3069;
        const int4 c = sm[b], v0 = sm[b + 1], v1 = sm[b + 2];
        const uint32_t salt = c.x + v0.y + v1.z;
        double g[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t r = mix(gw * 0x9E3779B9u + static_cast<uint32_t>(it) * 131u + grp * 7u + q * 977u + (salt & 1u)) % nrows;
            const double* p = x + static_cast<int64_t>(r) * 8 + part * 4;
            asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                         : "=d"(g[q][0]), "=d"(g[q][1]), "=d"(g[q][2]), "=d"(g[q][3]) : "l"(p));
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) acc += g[q][0] * __int_as_float(v0.x) + g[q][1] + g[q][2] + g[q][3];
    }
    if (acc == 1.2345) sink[0] = acc;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t xbytes = size_t(8) << 20;            // 8 MB window of 64-byte rows (the C5 band at m = 8)
    const uint32_t nrows = static_cast<uint32_t>(xbytes / 64);
    const uint32_t nmat = 4u << 20;                   // 64 MB of 16-byte chunks (L2-resident after warm-up)
    double2* x;
    int4* mat;
    double* sink;
    CK(cudaMalloc(&x, xbytes));
    CK(cudaMalloc(&mat, size_t(nmat) * 16));
    CK(cudaMalloc(&sink, 8));
    CK(cudaMemset(x, 0, xbytes));
    CK(cudaMemset(mat, 0, size_t(nmat) * 16));
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = mat;
    rd.res.linear.desc = cudaCreateChannelDesc<int4>();
    rd.res.linear.sizeInBytes = size_t(nmat) * 16;
    cudaTextureDesc td{};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex;
    CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const int grid = sms * 4, iters = 2048;
    const char* names[4] = {"none", "shared", "tex", "ldg"};
    std::printf("{\"sms\": %d, \"warps_per_sm\": 32, \"modes\": {", sms);
    for (int mode = 0; mode < 4; ++mode) {
        auto launch = [&](int its) {
            switch (mode) {
                case 0: k<0><<<grid, 256, 49152>>>(x, nrows, mat, tex, nmat, its, sink); break;
                case 1: k<1><<<grid, 256, 49152>>>(x, nrows, mat, tex, nmat, its, sink); break;
                case 2: k<2><<<grid, 256, 49152>>>(x, nrows, mat, tex, nmat, its, sink); break;
                default: k<3><<<grid, 256, 49152>>>(x, nrows, mat, tex, nmat, its, sink); break;
            }
        };
        if (mode == 0) {
            CK(cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152));
        }
        launch(64);
        CK(cudaEventRecord(a));
        launch(iters);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        const double nnz = double(grid) * 8 /*warps*/ * 8 /*rows*/ * 4 * iters;
        std::printf("%s\"%s\": {\"ms\": %.3f, \"gather_TBps\": %.2f, \"ns_per_nnz_per_sm\": %.4f}", mode ? ", " : "",
                    names[mode], ms, nnz * 64.0 / (ms * 1e-3) / 1e12, ms * 1e6 / (nnz / sms));
    }
    {
        // 3 blocks of 256 threads per SM (the register budget of 4 x 32-byte gathers per lane)
        const int grid3 = sms * 3;
        CK(cudaFuncSetAttribute(k256, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
        k256<<<grid3, 256, 65536>>>(reinterpret_cast<const double*>(x), nrows, 64, sink);
        CK(cudaEventRecord(a));
        k256<<<grid3, 256, 65536>>>(reinterpret_cast<const double*>(x), nrows, iters, sink);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        const double nnz = double(grid3) * 8 * 16 * 4 * iters;
        std::printf(", \"ldg256_shared\": {\"ms\": %.3f, \"gather_TBps\": %.2f, \"ns_per_nnz_per_sm\": %.4f}", ms,
                    nnz * 64.0 / (ms * 1e-3) / 1e12, ms * 1e6 / (nnz / sms));
    }
    std::printf("}}\n");
    return 0;
}
