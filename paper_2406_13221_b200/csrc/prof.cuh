// prof.cuh — optional per-launch CUDA-event timing by kernel category, used
// by bench.py to attribute device time live (roofline of the dominant kernel).
// Disabled by default: a disabled scope costs one branch.
#pragma once
#include <cuda_runtime.h>

enum ProfCat {
    PROF_NTT = 0,      // forward/inverse NTT (both passes), any caller
    PROF_MODUP = 1,    // ModUp basis conversion
    PROF_INNER = 2,    // key inner product
    PROF_MODDOWN = 3,  // ModDown conversion + combine
    PROF_TENSOR = 4,   // ct x ct tensor
    PROF_RESCALE = 5,  // rescale conversion + combine
    PROF_ELEM = 6,     // add / const / plaintext / linear combinations
    PROF_OTHER = 7,    // keygen, encryption, decryption, refresh
    PROF_NCAT = 8
};

bool prof_enabled();
void prof_begin(int cat, double bytes, cudaStream_t s);
void prof_end(cudaStream_t s);

struct ProfScope {
    bool on;
    cudaStream_t s;
    ProfScope(int cat, double bytes, cudaStream_t st) : on(prof_enabled()), s(st) {
        if (on) prof_begin(cat, bytes, s);
    }
    ~ProfScope() {
        if (on) prof_end(s);
    }
};
