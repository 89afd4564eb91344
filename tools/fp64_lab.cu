// fp64_lab.cu -- DADD throughput and latency on this GPU (sizes the exact-dot budget).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/fp64_lab.cu -o build/fp64_lab
#include <cuda_runtime.h>
#include <cstdio>

template <int CH>
__global__ void k_dadd(double* out, int iters, double d) {
    double a[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) a[c] = __dadd_rn(a[c], d);
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += a[c];
    if (s == 1.2345) out[0] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 1 << 14;
    auto run = [&](const char* name, auto kern, int chains, int blocks, int threads) {
        kern<<<blocks, threads>>>(out, iters, 1e-300);
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(out, iters, 1e-300);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = double(blocks) * threads * chains * iters;
        printf("%-34s %8.3f ms  %8.2f Gop/s  %6.2f op/clk/SM@1.9GHz\n", name, ms, ops / ms / 1e6,
               ops / (ms * 1e-3) / sms / 1.9e9);
    };
    run("throughput 8 chains x 1024 thr x 4/SM", k_dadd<8>, 8, sms * 4, 256);
    run("throughput 4 chains x 2048 thr/SM", k_dadd<4>, 4, sms * 8, 256);
    run("latency 1 chain x 1 warp/SM", k_dadd<1>, 1, sms, 32);
    run("1 chain x 4 warps/SM (1/SMSP)", k_dadd<1>, 1, sms, 128);
    run("1 chain x 16 warps/SM", k_dadd<1>, 1, sms, 512);
    run("2 chains x 16 warps/SM", k_dadd<2>, 2, sms, 512);
    run("4 chains x 8 warps/SM", k_dadd<4>, 4, sms, 256);
    return 0;
}
