// hoist.cu — key inner product for hoisted rotate-and-sums (and any batched
// key switch): one thread per (coefficient, extended limb) carrying NB
// ciphertexts, cp.async step prefetch, fp64 or 128-bit integer
// multiply-accumulate.  Split from ops.cu so the two
// translation units compile in parallel.
#include <cstdlib>
#include <type_traits>

#include "async.cuh"
#include "ks.cuh"

// Per-thread asynchronous prefetch: every thread copies the key words and
// permuted ext words of rotation step t + S - 1 into its own shared-memory
// slots (cp.async, 8 bytes each) while it multiplies step t, so the gathers'
// latency overlaps the arithmetic without holding them in registers.  Each
// slot is written and read by the same thread, so cp.async.wait_group alone
// orders them (no block barrier).
__device__ __forceinline__ void cp_async8(u64* dst, const u64* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

#ifndef HELR_HOIST_EXP
#define HELR_HOIST_EXP 0  // timing experiments only (wrong results): 1 keys from a cache-resident window, 2 digits likewise
#endif
constexpr int HOIST_T = 128;     // threads per block (coefficients per tile)
#ifndef HELR_HOIST_STAGES
#define HELR_HOIST_STAGES 3
#endif
constexpr int HOIST_STAGES = HELR_HOIST_STAGES;  // steps in flight per thread
#ifndef HELR_HOIST_KEYREG
#define HELR_HOIST_KEYREG 0  // 1: key words bypass shared memory (ld.global.nc into registers one step ahead)
#endif
constexpr bool HOIST_KEYREG = HELR_HOIST_KEYREG;


// grid: x = coefficient tile * chunks + chunk (chunks of NB ciphertexts share
// the tile's key words through L2 at the same time), y = extended limb e.
// Kernel arguments of the key inner product (hoisted or single key).
struct HoistArgs {
    const u64* ext;
    long long ext_item_stride, ext_digit_stride;
    u64* acc;
    long long acc_item_stride;
    int n, log_n, nl, K, L, LK, B, nchunks, fold;
    const u64* one_sh;
    const u64* dadd;  // optional [B][3][L][N] tensor: Q limbs also get (P mod q) * (d0, d1)
    long long dadd_is;
    const u64* pm;
    const u64* pm_sh;
};

// FULL: the chunk holds all NB ciphertexts (uniform per CTA), so the step
// loop has no per-ciphertext branches: one basic block in which the prefetch
// of step t + S - 1 is written piecewise between the multiply-accumulate
// groups of step t.
template <int ND, int NB, bool DBL, bool FULL>
__device__ __forceinline__ void hoist_body(const HoistKeys& hk, const HoistArgs& A, const Tables& tb) {
    const u64* __restrict__ ext = A.ext;
    const long long ext_item_stride = A.ext_item_stride, ext_digit_stride = A.ext_digit_stride;
    u64* acc = A.acc;
    const long long acc_item_stride = A.acc_item_stride;
    const int n = A.n, log_n = A.log_n, nl = A.nl, K = A.K, L = A.L, LK = A.LK, B = A.B, nchunks = A.nchunks,
              fold = A.fold;
    const u64* one_sh = A.one_sh;
    constexpr int KW = HOIST_KEYREG ? 0 : 2 * ND;  // key words staged in shared memory
    constexpr int W = KW + NB * ND;                 // words per thread per stage
    constexpr int S = HOIST_STAGES;
    extern __shared__ u64 hsm[];
    const int tid = threadIdx.x;
    const int e = blockIdx.y;
    const int tile = blockIdx.x / nchunks, chunk = blockIdx.x - tile * nchunks;
    const int i = tile * HOIST_T + tid;
    const int b0 = chunk * NB;
    if (i >= n) return;
    const int p = e < nl ? e : L + (e - nl);
    const u64 q = tb.q[p], r1 = tb.br1[p], r0 = tb.br0[p], osh = one_sh[p];
    const int nb = B - b0 < NB ? B - b0 : NB;
    const u64* xb = ext + (size_t)b0 * ext_item_stride + (size_t)e * n;
    const size_t k0off = ((size_t)p) * n + i;
    const size_t k1off = ((size_t)LK + p) * n + i;
    const size_t kds = (size_t)2 * LK * n;
    auto slot = [&](int stage, int w) -> u64* { return hsm + ((size_t)(stage * W + w) * HOIST_T + tid); };
    const unsigned ei = 2u * (unsigned)brv_dev(i, log_n) + 1u;  // Galois index of this coefficient
    // prefetch of step t in NB pieces: piece b copies ciphertext b's permuted
    // digit words and a share of the 2 ND key words; the last piece commits
    auto issue_piece = [&](int t, int b, int& src) {
        // past the last step the prefetch re-reads the last step's words into
        // a stage that was already consumed (harmless, L2 hits): no branch,
        // so the whole step stays one basic block
        const int stage = t % S;
        const int tc = t < hk.nsteps ? t : hk.nsteps - 1;
        if (b == 0) src = galois_perm_e(ei, (u64)hk.gal[tc], log_n);
        const u64* kt = hk.key[tc];
#pragma unroll
        for (int w = b; w < KW; w += NB) {
            const int j = w < ND ? w : w - ND;
#if HELR_HOIST_EXP & 1
            cp_async8(slot(stage, w), hk.key[0] + tid + 128 * w);
#else
            cp_async8(slot(stage, w), kt + (size_t)j * kds + (w < ND ? k0off : k1off));
#endif
        }
        if (FULL || b < nb) {
#pragma unroll
            for (int j = 0; j < ND; j++)
#if HELR_HOIST_EXP & 2
                cp_async8(slot(stage, KW + b * ND + j), ext + (src & 1023) + 1024 * (b * ND + j));
#else
                cp_async8(slot(stage, KW + b * ND + j),
                          xb + (size_t)b * ext_item_stride + (size_t)j * ext_digit_stride + src);
#endif
        }
        if (b == NB - 1) cp_async_commit();
    };
    auto issue = [&](int t) {
        int src = 0;
#pragma unroll
        for (int b = 0; b < NB; b++) issue_piece(t, b, src);
    };
    using Acc = typename std::conditional<DBL, dacc, macc>::type;
    Acc a0[NB], a1[NB];
#pragma unroll
    for (int b = 0; b < NB; b++) {
        if constexpr (DBL) a0[b] = a1[b] = dacc{0.0, 0.0, 0.0};
        else a0[b] = a1[b] = macc{0, 0, 0, 0};
    }
#pragma unroll
    for (int t = 0; t < S - 1; t++) issue(t);
    int run = 0;
    static_assert(S >= 2, "the prefetch needs at least two stages");
    // HOIST_KEYREG: this step's key words were loaded into registers during the
    // previous step (coalesced ld.global.nc), the next step's are requested
    // before this step's arithmetic starts
    u64 kn[2 * ND], kn2[2 * ND];  // key words of steps t + 1 and t + 2
    auto load_keys = [&](int t, u64 (&dst)[2 * ND]) {
        const int tc = t < hk.nsteps ? t : hk.nsteps - 1;
        const u64* kt = hk.key[tc];
#pragma unroll
        for (int w = 0; w < 2 * ND; w++) {
            const int j = w < ND ? w : w - ND;
            dst[w] = __ldg(kt + (size_t)j * kds + (w < ND ? k0off : k1off));
        }
    };
    if constexpr (HOIST_KEYREG) { load_keys(0, kn); load_keys(1, kn2); }
    for (int t = 0; t < hk.nsteps; t++) {
        // step t's words have landed (step t + 1 may still be in flight); they
        // are read into registers first and step t + S - 1 is issued AFTER
        // that, so its address arithmetic and cp.async instructions sit
        // between this step's fp64 multiply-accumulates in the instruction
        // stream (the fp64 pipe takes one instruction every other cycle; the
        // integer work fills the gaps) instead of forming a separate phase
        cp_async_wait<S - 2>();
        const int stage = t % S;
        u64 kw[2 * ND], dw[NB * ND];
        if constexpr (HOIST_KEYREG) {
#pragma unroll
            for (int j = 0; j < 2 * ND; j++) { kw[j] = kn[j]; kn[j] = kn2[j]; }
            load_keys(t + 2, kn2);
        } else {
#pragma unroll
            for (int j = 0; j < 2 * ND; j++) kw[j] = *slot(stage, j);
        }
#pragma unroll
        for (int b = 0; b < NB; b++) {
#pragma unroll
            for (int j = 0; j < ND; j++) dw[b * ND + j] = (FULL || b < nb) ? *slot(stage, KW + b * ND + j) : 0;
        }
        int nsrc = 0;
        if constexpr (DBL) {
            double k0h[ND], k0l[ND], k1h[ND], k1l[ND];
#pragma unroll
            for (int j = 0; j < ND; j++) {
                split21(kw[j], k0h[j], k0l[j]);
                split21(kw[ND + j], k1h[j], k1l[j]);
            }
#pragma unroll
            for (int b = 0; b < NB; b++) {
                issue_piece(t + S - 1, b, nsrc);
                if (FULL || b < nb) {
#pragma unroll
                    for (int j = 0; j < ND; j++) {
                        double uh, ul;
                        split21_d(__longlong_as_double((long long)dw[b * ND + j]), uh, ul);
                        mac_d(a0[b], uh, ul, k0h[j], k0l[j]);
                        mac_d(a1[b], uh, ul, k1h[j], k1l[j]);
                    }
                }
            }
        } else {
            if (run == fold) {  // fold into a residue before the 128-bit sum can overflow
#pragma unroll
                for (int b = 0; b < NB; b++) {
                    a0[b] = macc{reduce128(resolve(a0[b]), q, r1, r0, osh), 0, 0, 0};
                    a1[b] = macc{reduce128(resolve(a1[b]), q, r1, r0, osh), 0, 0, 0};
                }
                run = 0;
            }
            run++;
#pragma unroll
            for (int b = 0; b < NB; b++) {
                issue_piece(t + S - 1, b, nsrc);
                if (FULL || b < nb) {
#pragma unroll
                    for (int j = 0; j < ND; j++) {
                        const u64 u = dw[b * ND + j];
                        mac_split(a0[b], u, kw[j]);
                        mac_split(a1[b], u, kw[ND + j]);
                    }
                }
            }
        }
    }
    cp_async_wait<0>();
    if constexpr (DBL) {
        // fold on the fp64 pipe (see k_ks_inner): hh 2^42 + mid 2^21 + ll
        const DblC dc{tb.qd[p], tb.qinvd[p]};
        const double t42 = reduce_d(4398046511104.0, dc);
        auto fold = [&](const dacc& c) -> double {
            return __dadd_rn(__dadd_rn(mulmod_d(reduce_d(c.hh, dc), t42, dc), mulmod_d(reduce_d(c.mid, dc), 2097152.0, dc)),
                             reduce_d(c.ll, dc));
        };
#pragma unroll
        for (int b = 0; b < NB; b++) {
            if (b < nb) {
                u64* ap = acc + (size_t)(b0 + b) * acc_item_stride;
                double f0 = fold(a0[b]), f1 = fold(a1[b]);
                if (A.dadd && e < nl) {  // merged ModDown + rescale: + (P mod q) * (d0, d1)
                    const u64* db = A.dadd + (size_t)(b0 + b) * A.dadd_is + (size_t)e * n + i;
                    const double w = u2d(A.pm[e]);
                    f0 = __dadd_rn(f0, mulmod_d(u2d(db[0]), w, dc));
                    f1 = __dadd_rn(f1, mulmod_d(u2d(db[(size_t)L * n]), w, dc));
                }
                ap[(size_t)e * n + i] = d2u_canon(f0, dc);
                ap[((size_t)(nl + K) + e) * n + i] = d2u_canon(f1, dc);
            }
        }
        return;
    }
#pragma unroll
    for (int b = 0; b < NB; b++) {
        if (b < nb) {
            u64* ap = acc + (size_t)(b0 + b) * acc_item_stride;
            u64 o0, o1;
            if constexpr (DBL) {
                o0 = reduce128(dresolve_s(a0[b]), q, r1, r0, osh);
                o1 = reduce128(dresolve_s(a1[b]), q, r1, r0, osh);
            } else {
                o0 = reduce128(resolve(a0[b]), q, r1, r0, osh);
                o1 = reduce128(resolve(a1[b]), q, r1, r0, osh);
            }
            if (A.dadd && e < nl) {  // merged ModDown + rescale: + (P mod q) * (d0, d1)
                const u64* db = A.dadd + (size_t)(b0 + b) * A.dadd_is + (size_t)e * n + i;
                const u64 w = A.pm[e], ws = A.pm_sh[e];
                o0 = add_mod(o0, shoup(db[0], w, ws, q), q);
                o1 = add_mod(o1, shoup(db[(size_t)L * n], w, ws, q), q);
            }
            ap[(size_t)e * n + i] = o0;
            ap[((size_t)(nl + K) + e) * n + i] = o1;
        }
    }
}

template <int ND, int NB>
#ifndef HELR_HOIST_MINB
#define HELR_HOIST_MINB 4  // 128 registers, 4 CTAs per SM (3 -> 4 after the interleaved prefetch: 1.42 -> 1.37 ms per step)
#endif
__global__ void __launch_bounds__(HOIST_T, HELR_HOIST_MINB) k_ks_inner_hoisted(HoistKeys hk, HoistArgs A, Tables tb) {
    pdl_begin();
    const int e = blockIdx.y;
    const int p = e < A.nl ? e : A.L + (e - A.nl);
    const int chunk = blockIdx.x % A.nchunks;
    const bool full = A.B - chunk * NB >= NB;
    if (tb.q[p] < NTT_DBL_BOUND) {  // uniform per CTA (one limb per CTA)
        if (full) hoist_body<ND, NB, true, true>(hk, A, tb);
        else hoist_body<ND, NB, true, false>(hk, A, tb);
    } else {
        if (full) hoist_body<ND, NB, false, true>(hk, A, tb);
        else hoist_body<ND, NB, false, false>(hk, A, tb);
    }
}

// ---- bulk-copy pipeline variant ---------------------------------------------
// One producer warp streams each rotation step's operands into a ring of
// shared-memory stages with cp.async.bulk (completion on per-stage
// mbarriers): the 2 * ND contiguous 1 KB key rows of the CTA's 128
// coefficients, and for every (ciphertext, digit) the four 256-byte runs the
// Galois permutation sends the CTA's four 32-coefficient warps to (a
// permutation maps every 32-aligned run of NTT slots onto one 32-aligned
// run).  The four consumer warps read their permuted digit words and key
// words from shared memory and run the same multiply-accumulate and fold as
// hoist_body; after each step every warp releases the stage on an "empty"
// mbarrier.  Replaces 12 per-thread 8-byte cp.async per step with ~36 bulk
// copies per CTA (HELR_HOIST_PIPE=0 keeps the per-thread kernel).
#ifndef HELR_HOIST_PSTAGES
#define HELR_HOIST_PSTAGES 4
#endif
constexpr int HP_S = HELR_HOIST_PSTAGES;
constexpr int HP_C = 128;       // consumer threads = coefficients per CTA tile
constexpr int HP_THREADS = HP_C + 32;

__device__ __forceinline__ void mbar_arrive(u64* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int ND, int NB, bool DBL>
__device__ __forceinline__ void hoist_pipe_body(const HoistKeys& hk, const HoistArgs& A, const Tables& tb, u64* sm,
                                                u64* full, u64* empty) {
    constexpr int KW = 2 * ND * HP_C;     // key words per stage
    constexpr int DW = NB * ND * HP_C;    // digit words per stage
    constexpr int SW = KW + DW;
    const int n = A.n, log_n = A.log_n, nl = A.nl, K = A.K, L = A.L, LK = A.LK, B = A.B, nchunks = A.nchunks;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int e = blockIdx.y;
    const int tile = blockIdx.x / nchunks, chunk = blockIdx.x - tile * nchunks;
    const int i0 = tile * HP_C;
    const int b0 = chunk * NB;
    const int nb = B - b0 < NB ? B - b0 : NB;
    const int p = e < nl ? e : L + (e - nl);
    const size_t kds = (size_t)2 * LK * n;
    const int nsteps = hk.nsteps;

    if (warp == HP_C / 32) {
        // ---------------- producer warp
        const u64* xb = A.ext + (size_t)b0 * A.ext_item_stride + (size_t)e * n;
        const unsigned bytes = (unsigned)(KW + nb * ND * HP_C) * 8u;
        for (int t = 0; t < nsteps; t++) {
            const int st = t % HP_S;
            if (t >= HP_S) mbar_wait(&empty[st], (unsigned)((t / HP_S - 1) & 1));
            if (lane == 0) mbar_expect_tx(&full[st], bytes);
            __syncwarp();
            u64* sb = sm + (size_t)st * SW;
            const u64* kt = hk.key[t];
            // copy c: c < 2 ND -> key row (poly, j); else digit run (b, j, w)
            const int ncopies = 2 * ND + nb * ND * 4;
            for (int c = lane; c < ncopies; c += 32) {
                if (c < 2 * ND) {
                    const int poly = c / ND, j = c % ND;
                    bulk_g2s(sb + c * HP_C, kt + (size_t)j * kds + ((size_t)poly * LK + p) * n + i0, HP_C * 8, &full[st]);
                } else {
                    const int d = c - 2 * ND;
                    const int w = d & 3, bj = d >> 2;       // bj = b * ND + j
                    const int b = bj / ND, j = bj % ND;
                    const int run = galois_perm(i0 + 32 * w, (u64)hk.gal[t], log_n) >> 5;
                    bulk_g2s(sb + KW + (size_t)d * 32,
                             xb + (size_t)b * A.ext_item_stride + (size_t)j * A.ext_digit_stride + (size_t)run * 32, 256,
                             &full[st]);
                }
            }
        }
        return;
    }
    // ---------------- consumer warps: one coefficient per thread
    const int i = i0 + tid;
    const u64 q = tb.q[p], r1 = tb.br1[p], r0 = tb.br0[p], osh = A.one_sh[p];
    const unsigned ei = 2u * (unsigned)brv_dev(i, log_n) + 1u;
    using Acc = typename std::conditional<DBL, dacc, macc>::type;
    Acc a0[NB], a1[NB];
#pragma unroll
    for (int b = 0; b < NB; b++) {
        if constexpr (DBL) a0[b] = a1[b] = dacc{0.0, 0.0, 0.0};
        else a0[b] = a1[b] = macc{0, 0, 0, 0};
    }
    int run = 0;
    for (int t = 0; t < nsteps; t++) {
        const int st = t % HP_S;
        const int off = galois_perm_e(ei, (u64)hk.gal[t], log_n) & 31;
        mbar_wait(&full[st], (unsigned)((t / HP_S) & 1));
        const u64* sb = sm + (size_t)st * SW;
        const u64* db = sb + KW + warp * 32 + off;   // + (b * ND + j) * 128
        if constexpr (DBL) {
            double k0h[ND], k0l[ND], k1h[ND], k1l[ND];
#pragma unroll
            for (int j = 0; j < ND; j++) {
                split21(sb[j * HP_C + tid], k0h[j], k0l[j]);
                split21(sb[(ND + j) * HP_C + tid], k1h[j], k1l[j]);
            }
#pragma unroll
            for (int b = 0; b < NB; b++) {
                if (b < nb) {
#pragma unroll
                    for (int j = 0; j < ND; j++) {
                        double uh, ul;
                        split21_d(__longlong_as_double((long long)db[(b * ND + j) * HP_C]), uh, ul);
                        mac_d(a0[b], uh, ul, k0h[j], k0l[j]);
                        mac_d(a1[b], uh, ul, k1h[j], k1l[j]);
                    }
                }
            }
        } else {
            if (run == A.fold) {
#pragma unroll
                for (int b = 0; b < NB; b++) {
                    a0[b] = macc{reduce128(resolve(a0[b]), q, r1, r0, osh), 0, 0, 0};
                    a1[b] = macc{reduce128(resolve(a1[b]), q, r1, r0, osh), 0, 0, 0};
                }
                run = 0;
            }
            run++;
            u64 k0[ND], k1[ND];
#pragma unroll
            for (int j = 0; j < ND; j++) {
                k0[j] = sb[j * HP_C + tid];
                k1[j] = sb[(ND + j) * HP_C + tid];
            }
#pragma unroll
            for (int b = 0; b < NB; b++) {
                if (b < nb) {
#pragma unroll
                    for (int j = 0; j < ND; j++) {
                        const u64 u = db[(b * ND + j) * HP_C];
                        mac_split(a0[b], u, k0[j]);
                        mac_split(a1[b], u, k1[j]);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
    u64* acc = A.acc;
    if (i >= n) return;
    if constexpr (DBL) {
        const DblC dc{tb.qd[p], tb.qinvd[p]};
        const double t42 = reduce_d(4398046511104.0, dc);
        auto fold = [&](const dacc& c) -> double {
            return __dadd_rn(__dadd_rn(mulmod_d(reduce_d(c.hh, dc), t42, dc), mulmod_d(reduce_d(c.mid, dc), 2097152.0, dc)),
                             reduce_d(c.ll, dc));
        };
#pragma unroll
        for (int b = 0; b < NB; b++) {
            if (b < nb) {
                u64* ap = acc + (size_t)(b0 + b) * A.acc_item_stride;
                double f0 = fold(a0[b]), f1 = fold(a1[b]);
                if (A.dadd && e < nl) {
                    const u64* dd = A.dadd + (size_t)(b0 + b) * A.dadd_is + (size_t)e * n + i;
                    const double w = u2d(A.pm[e]);
                    f0 = __dadd_rn(f0, mulmod_d(u2d(dd[0]), w, dc));
                    f1 = __dadd_rn(f1, mulmod_d(u2d(dd[(size_t)L * n]), w, dc));
                }
                ap[(size_t)e * n + i] = d2u_canon(f0, dc);
                ap[((size_t)(nl + K) + e) * n + i] = d2u_canon(f1, dc);
            }
        }
    } else {
#pragma unroll
        for (int b = 0; b < NB; b++) {
            if (b < nb) {
                u64* ap = acc + (size_t)(b0 + b) * A.acc_item_stride;
                u64 o0 = reduce128(resolve(a0[b]), q, r1, r0, osh);
                u64 o1 = reduce128(resolve(a1[b]), q, r1, r0, osh);
                if (A.dadd && e < nl) {
                    const u64* dd = A.dadd + (size_t)(b0 + b) * A.dadd_is + (size_t)e * n + i;
                    const u64 w = A.pm[e], ws = A.pm_sh[e];
                    o0 = add_mod(o0, shoup(dd[0], w, ws, q), q);
                    o1 = add_mod(o1, shoup(dd[(size_t)L * n], w, ws, q), q);
                }
                ap[(size_t)e * n + i] = o0;
                ap[((size_t)(nl + K) + e) * n + i] = o1;
            }
        }
    }
}

#ifndef HELR_HOIST_PMINB
#define HELR_HOIST_PMINB 4
#endif
template <int ND, int NB>
__global__ void __launch_bounds__(HP_THREADS, HELR_HOIST_PMINB) k_ks_inner_pipe(HoistKeys hk, HoistArgs A, Tables tb) {
    extern __shared__ __align__(128) u64 hp_sm[];
    __shared__ __align__(8) u64 bars[2 * HP_S];
    pdl_begin();
    if (threadIdx.x == 0) {
        for (int s = 0; s < HP_S; s++) {
            mbar_init(&bars[s], 1);                 // full: the producer's expect_tx arrival
            mbar_init(&bars[HP_S + s], HP_C / 32);  // empty: one arrival per consumer warp
        }
    }
    __syncthreads();
    const int e = blockIdx.y;
    const int p = e < A.nl ? e : A.L + (e - A.nl);
    if (tb.q[p] < NTT_DBL_BOUND)  // uniform per CTA
        hoist_pipe_body<ND, NB, true>(hk, A, tb, hp_sm, bars, bars + HP_S);
    else
        hoist_pipe_body<ND, NB, false>(hk, A, tb, hp_sm, bars, bars + HP_S);
}

static bool hoist_pipe_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* v = getenv("HELR_HOIST_PIPE");
        on = v ? (atoi(v) != 0) : 0;  // measured slower: per-lane bulk copies serialise
    }
    return on != 0;
}

template <int ND, int NB>
static void launch_pipe_nb(dim3 g, cudaStream_t s, const HoistKeys& hk, HoistArgs A, const Tables& tb) {
    A.nchunks = (A.B + NB - 1) / NB;
    const size_t smem = sizeof(u64) * (size_t)HP_S * (2 * ND + NB * ND) * HP_C;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_ks_inner_pipe<ND, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    g.x = (unsigned)(((A.n + HP_C - 1) / HP_C) * A.nchunks);
    launch_pdl(k_ks_inner_pipe<ND, NB>, g, dim3(HP_THREADS), smem, s, hk, A, tb);
}

// Steps per 128-bit accumulation run: a run adds fold*nd products (each <
// 2^(2 bits)) to a residue (< 2^bits) and must stay below 2^128.
static int hoist_fold(const helr_ctx* c, int nd) {
    int bits = 0;
    for (u64 q : c->primes) {
        int b = 64 - __builtin_clzll(q);
        if (b > bits) bits = b;
    }
    const int room = 128 - 2 * bits;  // 2^room products fit, less one for the residue
    const long long terms = room >= 20 ? (1ll << 20) : (1ll << room) - 1;
    const long long f = terms / nd;
    return f < 1 ? 1 : (f > (1 << 20) ? (1 << 20) : (int)f);
}

template <int ND, int NB>
static void launch_hoisted_nb(dim3 g, cudaStream_t s, const HoistKeys& hk, HoistArgs A, const Tables& tb) {
    A.nchunks = (A.B + NB - 1) / NB;
    const size_t smem = sizeof(u64) * (size_t)HOIST_STAGES * ((HOIST_KEYREG ? 0 : 2) + NB) * ND * HOIST_T;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_ks_inner_hoisted<ND, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    g.x *= A.nchunks;
    launch_pdl(k_ks_inner_hoisted<ND, NB>, g, dim3(HOIST_T), smem, s, hk, A, tb);
}
// ciphertexts per thread: HELR_HOIST_NB (1, 2, 4 or 8; default 4) caps it
static int hoist_nb_cap() {
    static int cap = -1;
    if (cap < 0) {
        const char* v = getenv("HELR_HOIST_NB");
        cap = v ? atoi(v) : 4;
        if (cap != 1 && cap != 2 && cap != 8) cap = 4;
    }
    return cap;
}
template <int ND>
static void launch_hoisted(dim3 g, cudaStream_t s, const HoistKeys& hk, const HoistArgs& A, const Tables& tb) {
    const int nb = A.B;
    const int cap = hoist_nb_cap();
    const int want = nb <= 1 ? 1 : nb <= 2 ? 2 : nb <= 4 ? 4 : 8;
    const int NBs = want < cap ? want : cap;
    if (hoist_pipe_enabled() && A.n % HP_C == 0 && A.n >= 1024) {
        if constexpr (ND <= 4) {
            if (NBs == 1) { launch_pipe_nb<ND, 1>(g, s, hk, A, tb); return; }
            if (NBs == 2) { launch_pipe_nb<ND, 2>(g, s, hk, A, tb); return; }
            launch_pipe_nb<ND, 4>(g, s, hk, A, tb);
            return;
        }
    }
    if (NBs == 1) launch_hoisted_nb<ND, 1>(g, s, hk, A, tb);
    else if (NBs == 2) launch_hoisted_nb<ND, 2>(g, s, hk, A, tb);
    else if (NBs == 4) launch_hoisted_nb<ND, 4>(g, s, hk, A, tb);
    else if constexpr (ND <= 3) launch_hoisted_nb<ND, 8>(g, s, hk, A, tb);
    else launch_hoisted_nb<ND, 4>(g, s, hk, A, tb);
}

// Key inner product of the ModUp'd digits in w.ext with hk's keys (summed over
// hk.nsteps Galois steps) into w.acc; dadd (optional) adds (P mod q)(d0, d1).
int key_inner(helr_ctx* c, const KsWs& w, const HoistKeys& hk, int nb, int level, const u64* dadd,
                     long long dadd_is, cudaStream_t s) {
    const int n = c->n, nl = level + 1, K = c->K, ne = nl + K;
    const int nd = (nl + c->alpha - 1) / c->alpha;
    dim3 g(blocks_for(n, HOIST_T), ne, 1);
    HoistArgs A{w.ext, w.ext_s, w.ext_ds, w.acc, w.acc_s, n, c->log_n, nl, K, c->L, c->LK, nb, 1, hoist_fold(c, nd),
                c->one_sh, dadd, dadd_is, c->pmod, c->pmod_sh};
    // algorithmic bytes: every operand once — the ModUp'd
    // digits once (the per-step Galois gathers re-read them from L2), every
    // step's key, the two output polynomials
    ProfScope ps(PROF_INNER, 8.0 * n * ((double)nb * nd * ne + 2.0 * nd * ne * hk.nsteps + 2.0 * nb * ne +
                                        (dadd ? 2.0 * nb * nl : 0.0)), s);
    switch (nd) {
        case 1: launch_hoisted<1>(g, s, hk, A, c->t); break;
        case 2: launch_hoisted<2>(g, s, hk, A, c->t); break;
        case 3: launch_hoisted<3>(g, s, hk, A, c->t); break;
        case 4: launch_hoisted<4>(g, s, hk, A, c->t); break;
        case 5: launch_hoisted<5>(g, s, hk, A, c->t); break;
        case 6: launch_hoisted<6>(g, s, hk, A, c->t); break;
        case 7: launch_hoisted<7>(g, s, hk, A, c->t); break;
        case 8: launch_hoisted<8>(g, s, hk, A, c->t); break;
        default: set_error("key switching: more than 8 digits"); return HELR_EINVAL;
    }
    CHECK_KERNEL("key inner product");
    return HELR_OK;
}

