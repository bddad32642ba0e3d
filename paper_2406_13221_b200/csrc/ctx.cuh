// ctx.cuh — device context: ring tables and key-switching workspace.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "modarith.cuh"

#define HELR_MAXP 64
#define HELR_MAXLIMBS 128  // entries of one LimbMap (one batched NTT launch)

// Per-prime scalar tables, passed by value to kernels (all device pointers).
struct Tables {
    const u64* q;        // [LK]
    const u64* br1;      // floor(2^128/q) high word
    const u64* br0;      // low word
    const u64* tw;       // [LK][N][2]  (psi^brv(k), Shoup quotient)
    const u64* itw;      // [LK][N][2]  (psi^-brv(k), Shoup quotient)
    const u64* ninv;     // [LK]  N^-1
    const u64* ninv_sh;
    const u64* itw1n;    // [LK]  psi^-brv(1) * N^-1  (last inverse stage)
    const u64* itw1n_sh;
    int log_n, n, L, K, alpha, beta;
    // fp64 NTT path for primes < 2^41 (ntt.cuh): the same twiddles as exact doubles
    const double* twd;    // [LK][N]  psi^brv(k)
    const double* itwd;   // [LK][N]  psi^-brv(k)
    const double* qd;     // [LK]  q
    const double* qinvd;  // [LK]  fl(1 / q)
    const double* nid;    // [LK]  N^-1
    const double* i1d;    // [LK]  psi^-brv(1) N^-1
};

// Limb selection for batched kernels: limb i of item z lives at
// base + z*item_stride + off[i]*N and uses prime prime[i].
struct LimbMap {
    int count;
    unsigned char off[HELR_MAXLIMBS];
    unsigned char prime[HELR_MAXLIMBS];
};

struct helr_ctx {
    int log_n, n, L, K, LK, dnum, alpha, beta, eta, max_batch;
    std::vector<u64> primes, psi;
    Tables t;
    // raw device allocations of the tables
    u64* d_tab = nullptr;
    size_t tab_words = 0;
    // rescale: qlinv[l*L + i] = q_l^-1 mod q_i (+ shoup), l >= 1, i < l
    const u64* qlinv = nullptr;
    const u64* qlinv_sh = nullptr;
    // ModUp: per (level l, digit j): offset into modup table
    std::vector<size_t> modup_off;  // [L * beta]
    const u64* modup = nullptr;     // packed, see ctx.cu
    size_t* d_modup_offs = nullptr; // device copy of modup_off
    std::vector<size_t> mr_off;      // merged ModDown+rescale tables per level (see ctx.cu)
    // ModDown (level-independent)
    const u64* md_phinv = nullptr;     // [K]   (P/p_k)^-1 mod p_k
    const u64* md_phinv_sh = nullptr;
    const u64* md_phmod = nullptr;     // [K][L] (P/p_k) mod q_i
    const u64* md_phmod_sh = nullptr;
    const u64* md_pinv = nullptr;      // [L] P^-1 mod q_i
    const u64* md_pinv_sh = nullptr;
    const u64* pmod = nullptr;         // [L] P mod q_i
    const u64* pmod_sh = nullptr;
    const u64* md_pinv_dbl = nullptr;  // [K] bits of (double)1/p_k
    const u64* imul_f = nullptr;       // [L][N] NTT of X^(N/2)
    const u64* one_sh = nullptr;       // [LK] floor(2^64 / q)
    const u64* t128 = nullptr;         // [LK] 2^128 mod q
    const u64* t128_sh = nullptr;
    // key-switching workspace
    u64* ws = nullptr;
    size_t ws_words = 0;
    // fused-iteration driver workspace (nag.cu), allocated on first use
    u64* nag_ws = nullptr;
    size_t nag_words = 0;
    int nag_graphs = 0;  // live captured graphs pointing into nag_ws
    // device encoder tables (encode.cu), built on first use
    void* enc_tw = nullptr;   // double2[N/2]
    int* enc_tpos = nullptr;  // [N/2]
    int* enc_tneg = nullptr;  // [N/2]
};

// ---- programmatic dependent launch (PDL) -----------------------------------
// Every kernel of the iteration starts with pdl_begin(): wait until the
// previous kernel in the stream has completed and its writes are visible.
// Launched through launch_pdl (cudaLaunchAttributeProgrammaticStreamSerialization)
// the next kernel's launch is processed while its predecessor runs (the
// trigger fires implicitly at the predecessor's completion; an explicit early
// trigger, which lets waiting CTAs occupy SMs during the last wave, measured
// 1 % slower); inside a captured graph the edges become programmatic.
// Measured: 190.7 -> 192.9 it/s.  HELR_PDL=0 turns the attribute off.
#ifndef HELR_PDL_TRIGGER
#define HELR_PDL_TRIGGER 0  // early trigger measured slower (dependents idle on SMs)
#endif
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (HELR_PDL_TRIGGER) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
bool pdl_enabled();
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                     Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

void set_error(const std::string& msg);
bool cuda_ok(cudaError_t e, const char* what);
void clear_stale_error(const char* where);

// helpers shared by the .cu files
inline LimbMap limb_range(int first_prime, int count, int first_off = 0) {
    LimbMap m;
    m.count = count;
    for (int i = 0; i < count; i++) {
        m.off[i] = (unsigned char)(first_off + i);
        m.prime[i] = (unsigned char)(first_prime + i);
    }
    return m;
}
