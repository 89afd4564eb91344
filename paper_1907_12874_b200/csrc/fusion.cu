// fusion.cu -- the paper's vector-fusion micro-benchmark (SURVEY.md 8(f)
// rank 4; Fig. 2 / Table 1) on B200:
//   run #1  three passes  y = a x + b y ; z = b x + a z ; z = b y + c z   (9N transfers)
//   run #2  one pass      y = a x + b y , z = b x + a z                  (5N transfers)
//   run #3  one pass      all three updates, y and z kept in registers   (5N transfers)
// The passes are the solver's own group programs (group.cuh), timed with CUDA
// events on the context stream; the claim under test is that time follows the
// transferred bytes, not the flops.
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"

namespace mbg {

// Fig. 2 run #2: y = a*x + b*y ; z = b*x + a*z
struct PFusion2 {
    static constexpr const char* NAME = "fusion_run2";
    static constexpr int NIN = 3, NOUT = 2, NCO = 3, NDOT = 0;   // in: x y z ; co: a b c
    __device__ static void run(const double* in, double* out, double*, const double* co) {
        out[0] = fmadd_rn(fmadd_rn(0.0, co[0], in[0]), co[1], in[1]);
        out[1] = fmadd_rn(fmadd_rn(0.0, co[1], in[0]), co[0], in[2]);
    }
};
// Fig. 2 run #3: ... ; z = b*y + c*z with the y and z just computed
struct PFusion3 {
    static constexpr const char* NAME = "fusion_run3";
    static constexpr int NIN = 3, NOUT = 2, NCO = 3, NDOT = 0;
    __device__ static void run(const double* in, double* out, double*, const double* co) {
        const double y = fmadd_rn(fmadd_rn(0.0, co[0], in[0]), co[1], in[1]);
        const double z = fmadd_rn(fmadd_rn(0.0, co[1], in[0]), co[0], in[2]);
        out[0] = y;
        out[1] = fmadd_rn(fmadd_rn(0.0, co[1], y), co[2], z);
    }
};

__global__ void fusion_init_kernel(double* v, int64_t n, uint64_t salt) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint64_t z = (static_cast<uint64_t>(i) + salt) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        v[i] = static_cast<double>(z >> 11) * (1.0 / 9007199254740992.0) - 0.5;
    }
}

}  // namespace mbg

using namespace mbg;

extern "C" int mbg_fusion_bench(mbg_ctx* ctx, int64_t n, int reps, double* ms_per_run, double* gbs_per_run,
                                int* identical) {
    try {
        if (!ctx || n < 1 || reps < 1 || !ms_per_run) throw Invalid("fusion_bench: bad arguments");
        MBG_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t st = ctx->stream;
        DevBuf<double> x(n), y(n), z(n), y0(n), z0(n), yk(n), zk(n), co(3);
        const double abc[3] = {0.5, 0.25, 0.125};
        MBG_CUDA(cudaMemcpyAsync(co.p, abc, sizeof abc, cudaMemcpyHostToDevice, st));
        fusion_init_kernel<<<1184, 256, 0, st>>>(x.p, n, 1);
        fusion_init_kernel<<<1184, 256, 0, st>>>(y0.p, n, 2);
        fusion_init_kernel<<<1184, 256, 0, st>>>(z0.p, n, 3);
        MBG_CUDA(cudaGetLastError());
        auto args = [&](std::initializer_list<const double*> in, std::initializer_list<double*> out,
                        std::initializer_list<int> c) {
            GroupArgs g{};
            g.len = n;
            g.m = 1;
            int i = 0;
            for (auto p : in) g.in[i++] = p;
            i = 0;
            for (auto p : out) g.out[i++] = p;
            i = 0;
            for (int k : c) g.coef[i++] = co.p + k;
            return g;
        };
        auto run = [&](int which) {
            if (which == 1) {
                launch_group<PUpd2>(st, args({x.p, y.p}, {y.p}, {0, 1}), ctx->num_sms);
                launch_group<PUpd2>(st, args({x.p, z.p}, {z.p}, {1, 0}), ctx->num_sms);
                launch_group<PUpd2>(st, args({y.p, z.p}, {z.p}, {1, 2}), ctx->num_sms);
            } else if (which == 2) {
                launch_group<PFusion2>(st, args({x.p, y.p, z.p}, {y.p, z.p}, {0, 1, 2}), ctx->num_sms);
            } else {
                launch_group<PFusion3>(st, args({x.p, y.p, z.p}, {y.p, z.p}, {0, 1, 2}), ctx->num_sms);
            }
            MBG_CUDA(cudaGetLastError());
        };
        cudaEvent_t e0, e1;
        MBG_CUDA(cudaEventCreate(&e0));
        MBG_CUDA(cudaEventCreate(&e1));
        const double transfers[4] = {0, 9, 5, 5};
        int same = 1;
        for (int which = 1; which <= 3; ++which) {
            MBG_CUDA(cudaMemcpyAsync(y.p, y0.p, n * 8, cudaMemcpyDeviceToDevice, st));
            MBG_CUDA(cudaMemcpyAsync(z.p, z0.p, n * 8, cudaMemcpyDeviceToDevice, st));
            run(which);   // warm-up (also the value checked below)
            if (which != 2) {
                if (which == 1) {
                    MBG_CUDA(cudaMemcpyAsync(yk.p, y.p, n * 8, cudaMemcpyDeviceToDevice, st));
                    MBG_CUDA(cudaMemcpyAsync(zk.p, z.p, n * 8, cudaMemcpyDeviceToDevice, st));
                } else {
                    // run #3 must reproduce run #1 bit for bit (same statements, same order)
                    std::vector<double> a(static_cast<size_t>(n)), b(static_cast<size_t>(n));
                    MBG_CUDA(cudaStreamSynchronize(st));
                    for (auto [p, q] : {std::pair<double*, double*>{y.p, yk.p}, {z.p, zk.p}}) {
                        MBG_CUDA(cudaMemcpy(a.data(), p, n * 8, cudaMemcpyDeviceToHost));
                        MBG_CUDA(cudaMemcpy(b.data(), q, n * 8, cudaMemcpyDeviceToHost));
                        if (std::memcmp(a.data(), b.data(), static_cast<size_t>(n) * 8) != 0) same = 0;
                    }
                }
            }
            MBG_CUDA(cudaEventRecord(e0, st));
            for (int r = 0; r < reps; ++r) run(which);
            MBG_CUDA(cudaEventRecord(e1, st));
            MBG_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            MBG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            ms_per_run[which - 1] = ms / reps;
            if (gbs_per_run)
                gbs_per_run[which - 1] = transfers[which] * 8.0 * static_cast<double>(n) / (ms / reps * 1e-3) / 1e9;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (identical) *identical = same;
        return MBG_OK;
    } catch (const Invalid& e) {
        set_error(e.what());
        return MBG_ERR_INVALID;
    } catch (const std::exception& e) {
        set_error(e.what());
        return MBG_ERR_RUNTIME;
    }
}
