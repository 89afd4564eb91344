// l2_lab.cu -- measured L2 -> SM ceilings on this B200 (VERDICT r1 "no measured
// L2 -> SM gather ceiling"): the roofline the gather-bound C5 CSR SpMM is
// reported against besides HBM.
//
//   stream  every SM streams a window that stays L2-resident (coalesced 16-byte
//           loads, grid-stride, many passes): the L2 read bandwidth
//   gather  each warp instruction gathers 32/L segments of G = 16*L bytes at
//           pseudo-random G-aligned offsets inside an L2-resident window W (the
//           C5 SpMM's x gathers: G = 8*m bytes per nonzero, W = the band window);
//           offsets come from a register hash, so no index traffic competes
//
// All reads go through ld.global.nc (L1 allocate, as in the SpMM) with a
// per-launch offset so L1 cannot serve repeats across passes; timing with CUDA
// events after a warm-up pass; bytes = useful bytes delivered to the SMs.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_lab tools/l2_lab.cu
// run:   tools/l2_lab > gpurun_out/l2_lab.json
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstdio>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
            return 1;                                                                           \
        }                                                                                       \
    } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t h) {
    h ^= h >> 16;
    h *= 0x7feb352dU;
    h ^= h >> 15;
    h *= 0x846ca68bU;
    h ^= h >> 16;
    return h;
}

__global__ void stream_kernel(const double2* __restrict__ buf, int64_t n16, int passes, double* sink) {
    double acc = 0.0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int p = 0; p < passes; ++p) {
        // rotate the start per pass so a block never re-reads its own previous lines from L1
        const int64_t rot = (static_cast<int64_t>(p) * 7919 * blockDim.x) % n16;
        for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride) {
            int64_t j = i + rot;
            if (j >= n16) j -= n16;
            const double2 v = __ldg(buf + j);
            acc += v.x + v.y;
        }
    }
    if (acc == 1.2345) sink[0] = acc;
}

template <int L>   // lanes per segment: segment = 16 * L bytes
__global__ void gather_kernel(const double2* __restrict__ buf, uint32_t nseg, int iters, uint32_t salt, double* sink) {
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int sub = lane / L, part = lane % L;
    double acc = 0.0;
#pragma unroll 4
    for (int it = 0; it < iters; ++it) {
        const uint32_t seg = mix(gw * 0x9E3779B9u + static_cast<uint32_t>(it) * 131u + sub * 7u + salt) % nseg;
        const double2 v = __ldg(buf + static_cast<int64_t>(seg) * L + part);
        acc += v.x + v.y;
    }
    if (acc == 1.2345) sink[0] = acc;
}

int main() {
    int sms = 0, dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int l2 = 0;
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    const size_t maxw = size_t(64) << 20;
    double2* buf;
    double* sink;
    CK(cudaMalloc(&buf, maxw));
    CK(cudaMalloc(&sink, 8));
    CK(cudaMemset(buf, 0, maxw));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    std::printf("{\"sms\": %d, \"l2_bytes\": %d, \"stream\": [", sms, l2);
    bool first = true;
    for (size_t w : {size_t(4) << 20, size_t(16) << 20, size_t(32) << 20, size_t(48) << 20}) {
        const int64_t n16 = static_cast<int64_t>(w / 16);
        const int passes = static_cast<int>(std::max<size_t>(8, (size_t(4) << 30) / w));
        const int grid = sms * 8, block = 256;
        stream_kernel<<<grid, block>>>(buf, n16, 2, sink);
        CK(cudaEventRecord(a));
        stream_kernel<<<grid, block>>>(buf, n16, passes, sink);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        std::printf("%s{\"window_MB\": %zu, \"GBps\": %.1f}", first ? "" : ", ", w >> 20,
                    static_cast<double>(w) * passes / (ms * 1e-3) / 1e9);
        first = false;
    }
    // HBM: a 4 GiB read-only stream (once) and a 2 x 2 GiB copy, for the read
    // mix of read-dominated kernels next to the copy peak of MEASURED_PEAKS.json
    {
        const size_t big = size_t(4) << 30;
        double2* h;
        CK(cudaMalloc(&h, big));
        CK(cudaMemset(h, 0, big));
        const int64_t n16 = static_cast<int64_t>(big / 16);
        stream_kernel<<<sms * 8, 256>>>(h, n16, 1, sink);
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            CK(cudaEventRecord(a));
            stream_kernel<<<sms * 8, 256>>>(h, n16, 1, sink);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, a, b));
            best = std::min(best, ms);
        }
        float bestc = 1e30f;
        for (int r = 0; r < 5; ++r) {
            CK(cudaEventRecord(a));
            CK(cudaMemcpyAsync(reinterpret_cast<char*>(h) + big / 2, h, big / 2, cudaMemcpyDeviceToDevice));
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, a, b));
            bestc = std::min(bestc, ms);
        }
        std::printf("], \"hbm_read_GBps\": %.1f, \"hbm_copy_GBps\": %.1f", static_cast<double>(big) / (best * 1e-3) / 1e9,
                    static_cast<double>(big) / (bestc * 1e-3) / 1e9);
        CK(cudaFree(h));
    }
    std::printf(", \"gather\": [");
    first = true;
    for (size_t w : {size_t(1) << 20, size_t(8) << 20, size_t(32) << 20}) {
        for (int L : {1, 2, 4, 8, 16}) {
            const uint32_t nseg = static_cast<uint32_t>(w / (16u * L));
            const int grid = sms * 8, block = 256, iters = 4096;
            auto launch = [&](int its, uint32_t salt) {
                switch (L) {
                    case 1: gather_kernel<1><<<grid, block>>>(buf, nseg, its, salt, sink); break;
                    case 2: gather_kernel<2><<<grid, block>>>(buf, nseg, its, salt, sink); break;
                    case 4: gather_kernel<4><<<grid, block>>>(buf, nseg, its, salt, sink); break;
                    case 8: gather_kernel<8><<<grid, block>>>(buf, nseg, its, salt, sink); break;
                    default: gather_kernel<16><<<grid, block>>>(buf, nseg, its, salt, sink); break;
                }
            };
            launch(64, 1u);
            CK(cudaEventRecord(a));
            launch(iters, 7u);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, a, b));
            const double bytes = static_cast<double>(grid) * block * 16.0 * iters;
            std::printf("%s{\"window_MB\": %zu, \"segment_B\": %d, \"GBps\": %.1f}", first ? "" : ", ", w >> 20,
                        16 * L, bytes / (ms * 1e-3) / 1e9);
            first = false;
        }
    }
    std::printf("]}\n");
    return 0;
}
