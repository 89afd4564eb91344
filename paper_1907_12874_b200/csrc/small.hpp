// small.hpp -- one-launch classical BiCGStab loop for small systems (small.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace mbg {

struct SmallArgs {
    int64_t n;
    int m;
    const int32_t* off;
    const int32_t* col;
    const double* val;
    double *x, *r, *r0, *p, *v, *s, *t;
    double* sc;          // scalar bank (NSCAL * m)
    int* ctl;            // control words
    double* hist;        // (maxit + 1) * m
    int64_t* slots;      // long accumulators, slot d at slots + d * m * NSLOT
    int fused, fixed, maxit;
    double tol2;
};

// Systems up to this many elements (n * m) take the one-launch path.
constexpr int64_t SMALL_MAX_LEN = int64_t(1) << 20;
bool small_path_enabled();   // MBG_SMALL=0 turns it off
int launch_small_classical(cudaStream_t st, const SmallArgs& a, int num_sms);

}  // namespace mbg
