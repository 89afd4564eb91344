// dot_lab.cu -- what does a read-only 2-vector pass cost on B200, with plain,
// Kahan-free naive and exact (TwoSum expansion) accumulation?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 tools/dot_lab.cu -o build/dot_lab
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            printf("CUDA %s %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                            \
        }                                                                       \
    } while (0)

// naive per-thread sum, block tree, atomic double add (no exactness)
template <int UNR, int MINB>
__global__ void __launch_bounds__(256, MINB) k_naive(const double2* a, const double2* b, long n, double* out) {
    double s0 = 0, s1 = 0;
    const long stride = (long)gridDim.x * blockDim.x;
    for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += UNR * stride) {
        double2 x[UNR], y[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (q + u * stride < n) { x[u] = a[q + u * stride]; y[u] = b[q + u * stride]; }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (q + u * stride < n) { s0 += x[u].x * y[u].x; s1 += x[u].y * y[u].y; }
    }
    for (int o = 16; o; o >>= 1) { s0 += __shfl_down_sync(~0u, s0, o); s1 += __shfl_down_sync(~0u, s1, o); }
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s0 + s1);
}

__device__ __forceinline__ void two(double& a0, double& a1, double x) {
    const double s0 = __dadd_rn(a0, x);
    const double b0 = __dsub_rn(s0, a0);
    const double e0 = __dadd_rn(__dsub_rn(a0, __dsub_rn(s0, b0)), __dsub_rn(x, b0));
    a0 = s0;
    a1 = __dadd_rn(a1, e0);
}

// one TwoSum level + plain second term (cost model of the exact path)
template <int UNR, int MINB>
__global__ void __launch_bounds__(256, MINB) k_twosum(const double2* a, const double2* b, long n, double* out) {
    double s0 = 0, s1 = 0, t0 = 0, t1 = 0;
    const long stride = (long)gridDim.x * blockDim.x;
    for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += UNR * stride) {
        double2 x[UNR], y[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (q + u * stride < n) { x[u] = a[q + u * stride]; y[u] = b[q + u * stride]; }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (q + u * stride < n) {
                two(s0, t0, __dmul_rn(x[u].x, y[u].x));
                two(s1, t1, __dmul_rn(x[u].y, y[u].y));
            }
    }
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s0 + s1 + t0 + t1);
}

__device__ __forceinline__ void grow3(double (&a)[3], double x, unsigned long long* slot) {
    const double s0 = __dadd_rn(a[0], x);
    if (!isfinite(s0)) { atomicAdd(slot, 1ull); return; }
    const double b0 = __dsub_rn(s0, a[0]);
    const double e0 = __dadd_rn(__dsub_rn(a[0], __dsub_rn(s0, b0)), __dsub_rn(x, b0));
    const double s1 = __dadd_rn(a[1], e0);
    const double b1 = __dsub_rn(s1, a[1]);
    const double e1 = __dadd_rn(__dsub_rn(a[1], __dsub_rn(s1, b1)), __dsub_rn(e0, b1));
    a[0] = s0;
    a[1] = s1;
    if (e1 != 0.0) {
        const double s2 = __dadd_rn(a[2], e1);
        const double b2 = __dsub_rn(s2, a[2]);
        const double e2 = __dadd_rn(__dsub_rn(a[2], __dsub_rn(s2, b2)), __dsub_rn(e1, b2));
        a[2] = s2;
        if (e2 != 0.0) atomicAdd(slot + 1, 1ull);
    }
}

template <int UNR, int MINB, int ND>
__global__ void __launch_bounds__(256, MINB) k_exact(const double2* a, const double2* b, long n, unsigned long long* slot,
                                                     double* out) {
    double acc[ND][2][3] = {};
    const long stride = (long)gridDim.x * blockDim.x;
    for (long q = (long)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += UNR * stride) {
        double2 x[UNR], y[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (q + u * stride < n) { x[u] = a[q + u * stride]; y[u] = b[q + u * stride]; }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (q + u * stride < n) {
                grow3(acc[0][0], __dmul_rn(x[u].x, y[u].x), slot);
                grow3(acc[0][1], __dmul_rn(x[u].y, y[u].y), slot);
                if (ND > 1) {
                    grow3(acc[ND - 1][0], __dmul_rn(x[u].x, x[u].x), slot);
                    grow3(acc[ND - 1][1], __dmul_rn(x[u].y, x[u].y), slot);
                }
            }
    }
    double t = 0;
#pragma unroll
    for (int d = 0; d < ND; ++d) t += acc[d][0][0] + acc[d][1][0] + acc[d][0][1] + acc[d][1][1] + acc[d][0][2];
    if ((threadIdx.x & 31) == 0) atomicAdd(out, t);
}

template <class F>
void bench(const char* name, F f, double bytes) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) f();
    cudaEventRecord(a);
    for (int i = 0; i < 20; ++i) f();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-32s %8.1f us  %7.1f GB/s\n", name, 1000 * ms / 20, bytes / (ms / 20 / 1e3) / 1e9);
}

int main() {
    const long n = 1l << 23;  // double2 packets per vector: 134 MB
    double2 *a, *b, *c;
    double* out;
    CK(cudaMalloc(&a, n * 16));
    CK(cudaMalloc(&b, n * 16));
    CK(cudaMalloc(&c, n * 16));
    CK(cudaMalloc(&out, 8));
    {
        double* h = (double*)malloc(n * 16);
        for (long i = 0; i < 2 * n; ++i) h[i] = ((i * 2654435761ul) % 1000003) / 1000003.0 - 0.5;
        CK(cudaMemcpy(a, h, n * 16, cudaMemcpyHostToDevice));
        for (long i = 0; i < 2 * n; ++i) h[i] = ((i * 40503ul + 7) % 999983) / 999983.0 - 0.3;
        CK(cudaMemcpy(b, h, n * 16, cudaMemcpyHostToDevice));
        free(h);
    }
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double bytes = 2.0 * n * 16;
    bench("memcpy (read+write 134MB)", [&] { cudaMemcpyAsync(c, a, n * 16, cudaMemcpyDeviceToDevice); }, bytes);
    for (int bl : {2, 4, 8}) {
        char nm[64];
        snprintf(nm, 64, "naive u2 grid=%dx", bl);
        bench(nm, [&] { k_naive<2, 2><<<sms * bl, 256>>>(a, b, n, out); }, bytes);
        snprintf(nm, 64, "naive u4 grid=%dx", bl);
        bench(nm, [&] { k_naive<4, 2><<<sms * bl, 256>>>(a, b, n, out); }, bytes);
        snprintf(nm, 64, "twosum u2 grid=%dx", bl);
        bench(nm, [&] { k_twosum<2, 2><<<sms * bl, 256>>>(a, b, n, out); }, bytes);
        snprintf(nm, 64, "twosum u4 grid=%dx", bl);
        bench(nm, [&] { k_twosum<4, 2><<<sms * bl, 256>>>(a, b, n, out); }, bytes);
    }
    unsigned long long* slot;
    CK(cudaMalloc(&slot, 64));
    for (int bl : {2, 3, 4, 6}) {
        char nm[64];
        snprintf(nm, 64, "exact1 u2 grid=%dx", bl);
        bench(nm, [&] { k_exact<2, 2, 1><<<sms * bl, 256>>>(a, b, n, slot, out); }, bytes);
        snprintf(nm, 64, "exact1 u4 grid=%dx", bl);
        bench(nm, [&] { k_exact<4, 2, 1><<<sms * bl, 256>>>(a, b, n, slot, out); }, bytes);
        snprintf(nm, 64, "exact2 u2 grid=%dx", bl);
        bench(nm, [&] { k_exact<2, 2, 2><<<sms * bl, 256>>>(a, b, n, slot, out); }, bytes);
        snprintf(nm, 64, "exact2 u4 grid=%dx", bl);
        bench(nm, [&] { k_exact<4, 2, 2><<<sms * bl, 256>>>(a, b, n, slot, out); }, bytes);
    }
    bench("naive u8 grid=8x", [&] { k_naive<8, 1><<<sms * 8, 256>>>(a, b, n, out); }, bytes);
    bench("naive u8 grid=4x", [&] { k_naive<8, 1><<<sms * 4, 256>>>(a, b, n, out); }, bytes);
    return 0;
}
