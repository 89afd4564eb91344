// h2d_lab.cu -- host<->device copy rates on the GPU box: pageable cudaMemcpy,
// pinned DMA, multi-threaded host memcpy into pinned memory, cudaHostRegister.
// nvcc -O3 -std=c++17 tools/h2d_lab.cu -o build/h2d_lab -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
    const size_t B = 256ull << 20;
    std::vector<char> host(B, 1);
    char *pinned, *dev;
    cudaMallocHost(&pinned, B);
    cudaMalloc(&dev, B);
    std::memset(pinned, 2, B);
    auto rate = [&](const char* name, auto f) {
        f();
        cudaDeviceSynchronize();
        double t = now();
        for (int i = 0; i < 5; ++i) f();
        cudaDeviceSynchronize();
        t = (now() - t) / 5;
        printf("%-40s %7.2f ms  %6.1f GB/s\n", name, t * 1e3, B / t / 1e9);
    };
    rate("pageable cudaMemcpy H2D", [&] { cudaMemcpy(dev, host.data(), B, cudaMemcpyHostToDevice); });
    rate("pageable cudaMemcpy D2H", [&] { cudaMemcpy(host.data(), dev, B, cudaMemcpyDeviceToHost); });
    rate("pinned DMA H2D", [&] { cudaMemcpy(dev, pinned, B, cudaMemcpyHostToDevice); });
    rate("pinned DMA D2H", [&] { cudaMemcpy(pinned, dev, B, cudaMemcpyDeviceToHost); });
    for (int nt : {1, 4, 8, 16, 32}) {
        char nm[64];
        snprintf(nm, 64, "host memcpy -> pinned, %d threads", nt);
        rate(nm, [&] {
            std::vector<std::thread> th;
            for (int t = 0; t < nt; ++t)
                th.emplace_back([&, t] {
                    size_t b = B * t / nt, e = B * (t + 1) / nt;
                    std::memcpy(pinned + b, host.data() + b, e - b);
                });
            for (auto& x : th) x.join();
        });
    }
    double t = now();
    cudaHostRegister(host.data(), B, cudaHostRegisterDefault);
    printf("cudaHostRegister 256 MB: %.2f ms\n", (now() - t) * 1e3);
    rate("registered DMA H2D", [&] { cudaMemcpy(dev, host.data(), B, cudaMemcpyHostToDevice); });
    rate("registered DMA D2H", [&] { cudaMemcpy(host.data(), dev, B, cudaMemcpyDeviceToHost); });
    t = now();
    cudaHostUnregister(host.data());
    printf("cudaHostUnregister: %.2f ms\n", (now() - t) * 1e3);
    printf("hardware threads: %u\n", std::thread::hardware_concurrency());
    // pipelined staging like api.cu upload_host: 2 x CH pinned halves, 8-thread memcpy, async DMA
    for (size_t CH : {16ull << 20, 64ull << 20}) {
        cudaStream_t st;
        cudaStreamCreate(&st);
        cudaEvent_t done[2];
        for (auto& e : done) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        double tm = 0, tw = 0;
        auto pipe = [&] {
            size_t k = 0;
            for (size_t o = 0; o < B; o += CH, ++k) {
                const size_t n = std::min(CH, B - o);
                char* half = pinned + (k & 1) * CH;
                double a = now();
                if (k >= 2) cudaEventSynchronize(done[k & 1]);
                double b = now();
                std::vector<std::thread> th;
                for (int t = 0; t < 8; ++t)
                    th.emplace_back([&, t] { size_t bb = n * t / 8, ee = n * (t + 1) / 8;
                                             std::memcpy(half + bb, host.data() + o + bb, ee - bb); });
                for (auto& x : th) x.join();
                double c = now();
                tw += b - a;
                tm += c - b;
                cudaMemcpyAsync(dev + o, half, n, cudaMemcpyHostToDevice, st);
                cudaEventRecord(done[k & 1], st);
            }
            cudaStreamSynchronize(st);
        };
        char nm[64];
        snprintf(nm, 64, "pipelined staging H2D chunk %zu MB", CH >> 20);
        tm = tw = 0;
        rate(nm, pipe);
        printf("   (per call: memcpy %.2f ms, waits %.2f ms)\n", tm / 6 * 1e3, tw / 6 * 1e3);
    }
    return 0;
}
