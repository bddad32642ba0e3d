// ntt.cuh — negacyclic NTT passes for sm_100a.
//
// Forward: Cooley-Tukey over bit-reversed powers of psi with Harvey lazy
// butterflies; output slot i = a(psi^(2 brv(i) + 1)).  Inverse:
// Gentleman-Sande with psi^-1, N^-1 folded into the last stage.  Twiddle
// products use Shoup with an approximate quotient (shoup_lazy4, result in
// [0, 4q)), so lazy values live in [0, 8q) forward and [0, 4q) inverse —
// 8q < 2^64 because every prime is below 2^61 (checked at context
// creation).  Outputs are reduced to [0, q), so both transforms equal,
// residue for residue, the oracle's loops.
//
// Decomposition.  log N = s1 + s2.  The first s1 forward stages only mix
// elements with equal index mod 2^s2 ("columns", stride 2^s2); the last s2
// stages only mix within contiguous blocks of 2^s2 ("rows").  Each pass is
// one kernel holding T = 2^LOG_T elements per sub-transform in registers
// (R = 2^LOG_R per thread, radix-R register stages) and exchanging through
// shared memory between register groups, so a limb is read and written
// once per pass.  N <= 2^11 runs as a single row pass.  Column passes put
// COLS adjacent columns in one CTA so every global access is a 128-byte
// segment; row passes put COLS contiguous blocks in one CTA.
//
// Loader / Storer functors give each pass its prologue / epilogue, so
// rescale, ModUp and ModDown fuse their basis conversions into the NTT
// instead of making extra passes over HBM.
#pragma once
#include <type_traits>

#include "ctx.cuh"
#include "prof.cuh"

#ifndef HELR_NTT_EPI_UNROLL
#define HELR_NTT_EPI_UNROLL 4  // tile-epilogue pairs per thread in flight
#endif
constexpr int kNttEpiUnroll = HELR_NTT_EPI_UNROLL;
#ifndef HELR_NTT_COLTW_SMEM
#define HELR_NTT_COLTW_SMEM 1
#endif
constexpr bool kColTwSmem = HELR_NTT_COLTW_SMEM;
#ifndef HELR_NTT_ROW_WARPSYNC
#define HELR_NTT_ROW_WARPSYNC 1
#endif
constexpr bool kRowWarpSync = HELR_NTT_ROW_WARPSYNC;

void count_launches(int k);

struct NttPassArgs {
    int log_n;
    int st0;        // first global stage of this pass (forward numbering)
    int final_out;  // 1: reduce outputs to [0, q)
    // fp64 limbs only: the intermediate buffer between the two passes of one
    // transform holds raw doubles (integer-valued, |x| < 2^46) instead of
    // canonical residues — saves the canonicalisation and the conversion back
    int raw_in, raw_out;
    int dbl_out;  // fp64 limbs, final pass: canonical residues stored as exact doubles
};

template <int LOG_T, int LOG_R>
struct NttShape {
    static constexpr int T = 1 << LOG_T;
    static constexpr int R = 1 << LOG_R;
    static constexpr int NG = (LOG_T + LOG_R - 1) / LOG_R;
};

// insert LOG_R zero bits at bit position lo of s
__device__ __forceinline__ int spread_index(int s, int lo, int log_r) {
    return ((s >> lo) << (lo + log_r)) | (s & ((1 << lo) - 1));
}

// Loader: u64 operator()(int z, int li, int prime, int off) const
//         (+ optional kVec / load2 for 16-byte contiguous pairs)
// Storer: void operator()(int z, int li, int prime, int off, u64 v) const
//         (+ optional kVec / store2)
// grid: x = sub-transform tiles, y = limb index in map, z = batch item.
template <class F, class = void>
struct has_vec { static constexpr bool value = false; };
template <class F>
struct has_vec<F, decltype((void)F::kVec)> { static constexpr bool value = F::kVec; };
// kTile: the last row pass stages its outputs through shared memory and calls
// store2 on coalesced consecutive pairs (storers that read other global
// arrays at the output position, e.g. StCombine)
template <class F, class = void>
struct has_tile { static constexpr bool value = false; };
template <class F>
struct has_tile<F, decltype((void)F::kTile)> { static constexpr bool value = F::kTile; };

// One radix-2 stage on a thread's R registers: pairs (i, i + 2^H), the
// twiddle shared by every pair with the same i >> (H + 1).  H is a template
// parameter so every register index is static (no local-memory arrays).
// q2 below is the lazy half-range 4q: forward inputs/outputs in [0, 8q).
template <int R, int H>
__device__ __forceinline__ void fwd_stage(u64 (&x)[R], const ulonglong2* __restrict__ W2, int tb0, u64 q, u64 q2) {
#pragma unroll
    for (int j = 0; j < (R >> (H + 1)); j++) {
        const ulonglong2 w = __ldg(W2 + tb0 + j);
#pragma unroll
        for (int t = 0; t < (1 << H); t++) {
            const int i = (j << (H + 1)) + t;
            u64 u = x[i];
            u = u >= q2 ? u - q2 : u;
            const u64 v = shoup_lazy4(x[i + (1 << H)], w.x, w.y, q);
            x[i] = u + v;
            x[i + (1 << H)] = u + q2 - v;
        }
    }
}
template <int R, int H>
__device__ __forceinline__ void inv_stage(u64 (&x)[R], const ulonglong2* __restrict__ W2, int tb0, u64 q, u64 q2) {
#pragma unroll
    for (int j = 0; j < (R >> (H + 1)); j++) {
        const ulonglong2 w = __ldg(W2 + tb0 + j);
#pragma unroll
        for (int t = 0; t < (1 << H); t++) {
            const int i = (j << (H + 1)) + t;
            const u64 u = x[i], v = x[i + (1 << H)];
            const u64 sum = u + v;
            x[i] = sum >= q2 ? sum - q2 : sum;
            x[i + (1 << H)] = shoup_lazy4(u + q2 - v, w.x, w.y, q);
        }
    }
}
// last inverse stage (psi^-brv(1)) with N^-1 folded into both outputs
template <int R, int H>
__device__ __forceinline__ void inv_last_stage(u64 (&x)[R], u64 ni, u64 nis, u64 wl, u64 wls, u64 q, u64 q2) {
#pragma unroll
    for (int i = 0; i < R; i++) {
        if (i & (1 << H)) continue;
        const u64 u = x[i], v = x[i + (1 << H)];
        x[i] = shoup_lazy4(u + v, ni, nis, q);
        x[i + (1 << H)] = shoup_lazy4(u + q2 - v, wl, wls, q);
    }
}
template <int R>
__device__ __forceinline__ void fwd_stage_h(int h, u64 (&x)[R], const ulonglong2* W2, int tb0, u64 q, u64 q2) {
    switch (h) {
        case 0: fwd_stage<R, 0>(x, W2, tb0, q, q2); break;
        case 1: if constexpr (R > 2) fwd_stage<R, 1>(x, W2, tb0, q, q2); break;
        case 2: if constexpr (R > 4) fwd_stage<R, 2>(x, W2, tb0, q, q2); break;
        default: if constexpr (R > 8) fwd_stage<R, 3>(x, W2, tb0, q, q2); break;
    }
}
template <int R>
__device__ __forceinline__ void inv_stage_h(int h, u64 (&x)[R], const ulonglong2* W2, int tb0, u64 q, u64 q2) {
    switch (h) {
        case 0: inv_stage<R, 0>(x, W2, tb0, q, q2); break;
        case 1: if constexpr (R > 2) inv_stage<R, 1>(x, W2, tb0, q, q2); break;
        case 2: if constexpr (R > 4) inv_stage<R, 2>(x, W2, tb0, q, q2); break;
        default: if constexpr (R > 8) inv_stage<R, 3>(x, W2, tb0, q, q2); break;
    }
}
template <int R>
__device__ __forceinline__ void inv_last_h(int h, u64 (&x)[R], u64 ni, u64 nis, u64 wl, u64 wls, u64 q, u64 q2) {
    switch (h) {
        case 0: inv_last_stage<R, 0>(x, ni, nis, wl, wls, q, q2); break;
        case 1: if constexpr (R > 2) inv_last_stage<R, 1>(x, ni, nis, wl, wls, q, q2); break;
        case 2: if constexpr (R > 4) inv_last_stage<R, 2>(x, ni, nis, wl, wls, q, q2); break;
        default: if constexpr (R > 8) inv_last_stage<R, 3>(x, ni, nis, wl, wls, q, q2); break;
    }
}

// ---- fp64 path for primes < 2^41 ------------------------------------------
// Residues of primes below 2^41 are exact doubles.  A twiddle product is
// computed on the FP64 pipe (idle otherwise; DFMA issues at the IMAD rate,
// 2.5x IMAD.WIDE): p = fl(a w), e = fma(a, w, -p) (exact), h = rint(p / q) as
// fma(p, 1/q, 1.5 2^52) - 1.5 2^52 (one rounding, to nearest), r = fma(-h, q,
// p) + e = a w - h q exactly, |r| < 0.6 q: six fp64 instructions.
// Signed values grow by < 0.6 q per forward stage and at most double per
// inverse stage; a pass (<= 8 stages) starting from canonical inputs stays
// below 2^50, so every intermediate is an exact integer-valued double, and
// every pass ends with an exact reduction to [0, q).  Identical residues to
// the integer path and the oracle.
constexpr double NTT_MAGIC = 6755399441055744.0;  // 1.5 * 2^52
constexpr double NTT_TWO52 = 4503599627370496.0;  // 2^52
struct DblC { double q, qinv; };
// rint(x * m) for |x * m| < 2^51: the fma rounds the exact product + 1.5 2^52
// to an integer, the subtraction is exact
__device__ __forceinline__ double drint_mul(double x, double m) {
    return __dsub_rn(__fma_rn(x, m, NTT_MAGIC), NTT_MAGIC);
}
__device__ __forceinline__ double mulmod_d(double a, double w, const DblC& c) {
    const double p = __dmul_rn(a, w);
    const double e = __fma_rn(a, w, -p);
    const double h = drint_mul(p, c.qinv);
    return __dadd_rn(__fma_rn(-h, c.q, p), e);
}
// integer-valued |x| < 2^50 -> x - rint(x / q) q, |result| <= q / 2 + 1 (exact)
__device__ __forceinline__ double reduce_d(double x, const DblC& c) {
    return __fma_rn(-drint_mul(x, c.qinv), c.q, x);
}
__device__ __forceinline__ double u2d(u64 x) {  // x < 2^52
    return __dsub_rn(__longlong_as_double((long long)(x | 0x4330000000000000ull)), NTT_TWO52);
}
// r < 0 ? r + q : r with the sign test on the integer pipe (an exact zero
// difference is +0 in round-to-nearest, so the sign bit alone decides): the
// fp64 pipe, which bounds these kernels, is spared the DSETP
__device__ __forceinline__ double wrap_neg(double r, double q) {
    const double rq = __dadd_rn(r, q);
    return __double2hiint(r) < 0 ? rq : r;
}
__device__ __forceinline__ u64 d2u_canon(double x, const DblC& c) {  // integer-valued |x| < 2^50 -> [0, q)
    const double r = wrap_neg(reduce_d(x, c), c.q);
    return (u64)__double_as_longlong(__dadd_rn(r, NTT_TWO52)) & 0x000FFFFFFFFFFFFFull;
}
// integer-valued |x| < 2^50 -> its residue in [0, q) as a double
__device__ __forceinline__ double d2d_canon(double x, const DblC& c) {
    return wrap_neg(reduce_d(x, c), c.q);
}
// A stage's R / 2^(H+1) twiddles are contiguous and, when there are two or
// more, start at an even index (the low bits of the register group's base
// are zero above bit lo), so they load as 16-byte pairs, all issued before
// the butterflies.
#ifndef HELR_NTT_EXP
#define HELR_NTT_EXP 0  // timing experiments only (wrong results), bit mask: 1 no twiddle loads, 2 no butterflies, 4 no global loads, 8 no global stores
#endif
template <int NW, bool SM = false>
__device__ __forceinline__ void load_tw(double (&w)[NW], const double* __restrict__ W, int tb0) {
#if HELR_NTT_EXP & 1
    if constexpr (SM) {
#pragma unroll
        for (int j = 0; j < NW; j++) w[j] = 3.0 + j;
        return;
    }
#endif
    if constexpr (SM) {  // shared-memory table (column passes): plain loads, LDS after inlining
        if constexpr (NW >= 2) {
#pragma unroll
            for (int j = 0; j < NW; j += 2) {
                const double2 p = *reinterpret_cast<const double2*>(W + tb0 + j);
                w[j] = p.x;
                w[j + 1] = p.y;
            }
        } else {
            w[0] = W[tb0];
        }
        return;
    }
#if HELR_NTT_EXP & 1
#pragma unroll
    for (int j = 0; j < NW; j++) w[j] = 3.0 + j;
    return;
#endif
    if constexpr (NW >= 2) {
#pragma unroll
        for (int j = 0; j < NW; j += 2) {
            const double2 p = __ldg(reinterpret_cast<const double2*>(W + tb0 + j));
            w[j] = p.x;
            w[j + 1] = p.y;
        }
    } else {
        w[0] = __ldg(W + tb0);
    }
}
template <int R, int H, bool SM = false>
__device__ __forceinline__ void fwd_stage_d(double (&x)[R], const double* __restrict__ W, int tb0, const DblC& c) {
    double wv[R >> (H + 1)];
    load_tw<(R >> (H + 1)), SM>(wv, W, tb0);
#pragma unroll
    for (int j = 0; j < (R >> (H + 1)); j++) {
        const double w = wv[j];
#pragma unroll
        for (int t = 0; t < (1 << H); t++) {
            const int i = (j << (H + 1)) + t;
            const double u = x[i], v = mulmod_d(x[i + (1 << H)], w, c);
            x[i] = __dadd_rn(u, v);
            x[i + (1 << H)] = __dsub_rn(u, v);
        }
    }
}
template <int R, int H, bool SM = false>
__device__ __forceinline__ void inv_stage_d(double (&x)[R], const double* __restrict__ W, int tb0, const DblC& c) {
    double wv[R >> (H + 1)];
    load_tw<(R >> (H + 1)), SM>(wv, W, tb0);
#pragma unroll
    for (int j = 0; j < (R >> (H + 1)); j++) {
        const double w = wv[j];
#pragma unroll
        for (int t = 0; t < (1 << H); t++) {
            const int i = (j << (H + 1)) + t;
            const double u = x[i], v = x[i + (1 << H)];
            x[i] = __dadd_rn(u, v);
            x[i + (1 << H)] = mulmod_d(__dsub_rn(u, v), w, c);
        }
    }
}
template <int R, int H>
__device__ __forceinline__ void inv_last_stage_d(double (&x)[R], double ni, double wl, const DblC& c) {
#pragma unroll
    for (int i = 0; i < R; i++) {
        if (i & (1 << H)) continue;
        const double u = x[i], v = x[i + (1 << H)];
        x[i] = mulmod_d(__dadd_rn(u, v), ni, c);
        x[i + (1 << H)] = mulmod_d(__dsub_rn(u, v), wl, c);
    }
}
template <int R, bool SM = false>
__device__ __forceinline__ void fwd_stage_dh(int h, double (&x)[R], const double* W, int tb0, const DblC& c) {
    switch (h) {
        case 0: fwd_stage_d<R, 0, SM>(x, W, tb0, c); break;
        case 1: if constexpr (R > 2) fwd_stage_d<R, 1, SM>(x, W, tb0, c); break;
        case 2: if constexpr (R > 4) fwd_stage_d<R, 2, SM>(x, W, tb0, c); break;
        default: if constexpr (R > 8) fwd_stage_d<R, 3, SM>(x, W, tb0, c); break;
    }
}
template <int R, bool SM = false>
__device__ __forceinline__ void inv_stage_dh(int h, double (&x)[R], const double* W, int tb0, const DblC& c) {
    switch (h) {
        case 0: inv_stage_d<R, 0, SM>(x, W, tb0, c); break;
        case 1: if constexpr (R > 2) inv_stage_d<R, 1, SM>(x, W, tb0, c); break;
        case 2: if constexpr (R > 4) inv_stage_d<R, 2, SM>(x, W, tb0, c); break;
        default: if constexpr (R > 8) inv_stage_d<R, 3, SM>(x, W, tb0, c); break;
    }
}
template <int R>
__device__ __forceinline__ void inv_last_dh(int h, double (&x)[R], double ni, double wl, const DblC& c) {
    switch (h) {
        case 0: inv_last_stage_d<R, 0>(x, ni, wl, c); break;
        case 1: if constexpr (R > 2) inv_last_stage_d<R, 1>(x, ni, wl, c); break;
        case 2: if constexpr (R > 4) inv_last_stage_d<R, 2>(x, ni, wl, c); break;
        default: if constexpr (R > 8) inv_last_stage_d<R, 3>(x, ni, wl, c); break;
    }
}

// Storers with kRawD take fp64 limbs' outputs as raw double bits and a
// per-thread context (prep / store2c / store1c): see StCombine (ks.cuh).
template <class F, class = void>
struct has_rawd { static constexpr bool value = false; };
template <class F>
struct has_rawd<F, decltype((void)F::kRawD)> { static constexpr bool value = F::kRawD; };

template <class F, bool = has_rawd<F>::value>
struct storer_ctx { struct type {}; };
template <class F>
struct storer_ctx<F, true> { using type = typename F::Ctx; };

// Loaders / storers with kPtr expose the base address of limb li of item z
// (plain strided buffers): the pass then addresses its elements as one
// pointer plus compile-time offsets instead of a 64-bit product per element.
template <class F, class = void>
struct has_ptr { static constexpr bool value = false; };
template <class F>
struct has_ptr<F, decltype((void)F::kPtr)> { static constexpr bool value = F::kPtr; };

// Primes below this bound take the fp64 path (uniform per CTA: one limb per CTA).
constexpr u64 NTT_DBL_BOUND = 1ull << 41;

// (bx, li, z) = sub-transform tile, limb index in map, batch item.  S2 =
// log N - LOG_T (column passes: the element stride is 2^S2, a compile-time
// constant so every register's address is an immediate offset).
// PRE: the CTA's input tile is already in `sm` (placed there by a TMA bulk
// tensor copy, ntt_tma.cuh): column tiles dense as [T][COLS], row tiles as
// [T * COLS / 16][16] words with the 128-byte hardware swizzle.  The tile is
// consumed into registers, then the same buffer serves the padded exchange.
__device__ __forceinline__ int swz128(int e) {  // word index -> swizzled word index
    return (e & ~15) | (((((e >> 1) ^ (e >> 4)) & 7) << 1)) | (e & 1);
}
template <int LOG_T, int LOG_R, int COLS, bool IS_COL, bool INV, int S2, bool DBL, class Ld, class St, bool PRE = false,
          bool TWSM = false, bool TWFILL = false>
__device__ __forceinline__ void ntt_body(const Ld& ld, const St& st, const Tables& tb, const LimbMap& map,
                                         const NttPassArgs& a, u64* sm, const int bx, const int li, const int z,
                                         double* tws = nullptr) {
    using S = NttShape<LOG_T, LOG_R>;
    constexpr int T = S::T, R = S::R, NG = S::NG;
    constexpr int TPS = T / R;  // threads per sub-transform
    constexpr int SROW = IS_COL ? (COLS + 1) : (T + T / 16);
    using V = typename std::conditional<DBL, double, u64>::type;
    // Row passes whose sub-transform is held by at most one warp's threads
    // (TPS <= 32): a warp owns 32 / TPS whole rows, stages them itself and
    // exchanges only with its own lanes, so every synchronisation of the pass
    // is a __syncwarp — warps never wait for one another (kRowWarpSync).
    constexpr bool WS = kRowWarpSync && !IS_COL && !PRE && TPS <= 32 && (T * COLS / R) % 32 == 0;
    constexpr int WWORDS = WS ? (32 / TPS) * T : 1;  // contiguous words a warp owns
    auto sync_tile = [&]() {
        if constexpr (WS) __syncwarp();
        else __syncthreads();
    };

    const int prime = map.prime[li];
    const u64 q = tb.q[prime];
    const u64 q2 = 4 * q;  // integer path: lazy half-range (see fwd_stage)
    DblC dc;
    if constexpr (DBL) dc = DblC{tb.qd[prime], tb.qinvd[prime]};
    const int n = 1 << a.log_n;
    const ulonglong2* W2 = reinterpret_cast<const ulonglong2*>(INV ? tb.itw : tb.tw) + (size_t)prime * n;
    const double* WD = (INV ? tb.itwd : tb.twd) + (size_t)prime * n;

    const int tid = threadIdx.x;
    // column passes of fp64 limbs: the pass's 2^LOG_T - 1 twiddles (the same for
    // every column) are staged in shared memory by the kernel, so the
    // per-stage twiddle reads are LDS instead of LDG queued behind the data
    // loads and stores (kColTwSmem)
    const double* WDG = WD;  // the limb's table in global memory
    if constexpr (TWSM) WD = tws;
    int cc, s;
    if (IS_COL) { cc = tid % COLS; s = tid / COLS; }
    else { s = tid % TPS; cc = tid / TPS; }
    const int sub = bx * COLS + cc;  // global column / block index
    const int sub_id = IS_COL ? 0 : sub;
    const int wrow = (1 << a.st0) + sub_id;  // twiddle index = (wrow << ls) + (k >> (qb + 1))

    auto goff = [&](int k) -> int {
        return IS_COL ? (sub + (k << S2)) : ((sub << LOG_T) + k);
    };
    // pointer fast path (kPtr functors): this thread's sub-transform base
    // (lin / lout) and the CTA's contiguous tile base (row passes, lcta / scta)
    constexpr bool LP = has_ptr<Ld>::value, SP = has_ptr<St>::value;
    const u64* lin = nullptr;
    const u64* lcta = nullptr;
    u64* lout = nullptr;
    u64* scta = nullptr;
    if constexpr (LP) {
        const u64* lb = ld.limb_ptr(z, li);
        lin = lb + (IS_COL ? sub : (sub << LOG_T));
        lcta = lb + ((bx * COLS) << LOG_T);
    }
    if constexpr (SP) {
        u64* sb = st.limb_ptr(z, li);
        lout = sb + (IS_COL ? sub : (sub << LOG_T));
        scta = sb + ((bx * COLS) << LOG_T);
    }
    auto loff = [&](int k) -> int { return IS_COL ? (k << S2) : k; };
    auto LD = [&](int k) -> u64 {
#if HELR_NTT_EXP & 4
        return (u64)(k * 3 + tid);
#endif
        if constexpr (LP) return lin[loff(k)];
        else return ld(z, li, prime, goff(k));
    };
    auto LD2 = [&](int k) -> ulonglong2 {
#if HELR_NTT_EXP & 4
        return make_ulonglong2(k * 3 + tid, k * 5 + tid);
#endif
        if constexpr (LP) return *reinterpret_cast<const ulonglong2*>(lin + loff(k));
        else if constexpr (has_vec<Ld>::value) return ld.load2(z, li, prime, goff(k));
        else return make_ulonglong2(0, 0);  // not reached: vector paths need kVec
    };
    typename storer_ctx<St>::type sctx;  // filled right before the stores (keeps it out of the butterflies' registers)
    auto ST = [&](int k, u64 v) {
#if HELR_NTT_EXP & 8
        if (v != 0xDEADBEEFDEADBEEFull) return;
#endif
        if constexpr (SP) lout[loff(k)] = v;
        else if constexpr (has_rawd<St>::value) st.store1c(sctx, goff(k), v);
        else st(z, li, prime, goff(k), v);
    };
    auto ST2 = [&](int k, ulonglong2 v) {
#if HELR_NTT_EXP & 8
        if (v.x != 0xDEADBEEFDEADBEEFull) return;
#endif
        if constexpr (SP) *reinterpret_cast<ulonglong2*>(lout + loff(k)) = v;
        else if constexpr (has_rawd<St>::value) st.store2c(sctx, goff(k), v);
        else if constexpr (has_vec<St>::value) st.store2(z, li, prime, goff(k), v);
    };
    auto sidx = [&](int k) -> int {
        return IS_COL ? (k * SROW + cc) : (cc * SROW + k + (k >> 4));
    };
    const bool raw_in = DBL && a.raw_in;
    // fp64 limbs: loads only reinterpret; canonical u64 inputs are converted in
    // one block after the group-0 load (a single uniform branch per pass
    // instead of a select per element)
    auto in_v = [&](u64 v) -> V {
        if constexpr (DBL) return __longlong_as_double((long long)v);
        else return v;
    };
    auto to_sm = [&](V v) -> u64 {
        if constexpr (DBL) return (u64)__double_as_longlong(v);
        else return v;
    };
    auto from_sm = [&](u64 v) -> V {
        if constexpr (DBL) return __longlong_as_double((long long)v);
        else return v;
    };

    V x[R];
#pragma unroll
    for (int g = 0; g < NG; g++) {
        // free index bits of this register group: [lo, lo + LOG_R)
        const int lo = !INV ? ((LOG_T - g * LOG_R - LOG_R) > 0 ? (LOG_T - g * LOG_R - LOG_R) : 0)
                            : ((g * LOG_R < LOG_T - LOG_R) ? g * LOG_R : LOG_T - LOG_R);
        const int base = spread_index(s, lo, LOG_R);
        if (g == 0) {
            if constexpr (PRE) {
                static_assert(NG >= 2, "preloaded tiles need an exchange");
                if constexpr (IS_COL) {
#pragma unroll
                    for (int i = 0; i < R; i++) x[i] = in_v(sm[(base + (i << lo)) * COLS + cc]);
                } else if (lo == 0) {
#pragma unroll
                    for (int i = 0; i < R; i += 2) {
                        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(sm + swz128(cc * T + base + i));
                        x[i] = in_v(v.x);
                        x[i + 1] = in_v(v.y);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < R; i++) x[i] = in_v(sm[swz128(cc * T + base + (i << lo))]);
                }
            } else if constexpr (!IS_COL && has_tile<Ld>::value) {
                if (lo == 0) {
                    // coalesced prologue: the CTA's T * COLS contiguous inputs
                    // through shared memory (each thread then takes R in a row)
                    constexpr int TOT = T * COLS;
                    constexpr int nthr = T * COLS / R;
                    // constant trip count: every thread moves TOT / (2 nthr) pairs
                    const int e0 = WS ? (tid >> 5) * WWORDS + 2 * (tid & 31) : 2 * tid;
                    constexpr int es = WS ? 64 : 2 * nthr;
                    constexpr int NIT = WS ? WWORDS / 64 : TOT / (2 * nthr);
                    static_assert(NIT * es == (WS ? WWORDS : TOT), "staging loop must tile the CTA's words");
#pragma unroll 4
                    for (int u = 0; u < NIT; u++) {
                        const int e = e0 + u * es;
                        const int c2 = e >> LOG_T, k = e & (T - 1);
                        ulonglong2 v;
#if HELR_NTT_EXP & 4
                        v = make_ulonglong2(e * 3 + tid, e * 5 + tid);
#else
                        if constexpr (LP) v = *reinterpret_cast<const ulonglong2*>(lcta + e);
                        else v = ld.load2(z, li, prime, ((bx * COLS + c2) << LOG_T) + k);
#endif
                        sm[c2 * SROW + k + (k >> 4)] = v.x;
                        sm[c2 * SROW + k + 1 + ((k + 1) >> 4)] = v.y;
                    }
                    sync_tile();
#pragma unroll
                    for (int i = 0; i < R; i++) x[i] = in_v(sm[sidx(base + i)]);
                    sync_tile();
                } else {
#pragma unroll
                    for (int i = 0; i < R; i++) x[i] = in_v(LD(base + (i << lo)));
                }
            } else if constexpr (!IS_COL && has_vec<Ld>::value) {
                if (lo == 0) {
#pragma unroll
                    for (int i = 0; i < R; i += 2) {
                        const ulonglong2 v = LD2(base + i);
                        x[i] = in_v(v.x);
                        x[i + 1] = in_v(v.y);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < R; i++) x[i] = in_v(LD(base + (i << lo)));
                }
            } else {
#pragma unroll
                for (int i = 0; i < R; i++) x[i] = in_v(LD(base + (i << lo)));
            }
            if constexpr (TWFILL) {
                // the twiddle table is fetched AFTER the tile's loads were
                // issued, so its latency and the barrier overlap with them
                if (tid < T) tws[tid] = __ldg(WDG + tid);
                __syncthreads();
            }
            if constexpr (DBL) {
                if (!raw_in) {
#pragma unroll
                    for (int i = 0; i < R; i++) x[i] = u2d((u64)__double_as_longlong(x[i]));
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < R; i++) x[i] = from_sm(sm[sidx(base + (i << lo))]);
            if (NG > 2) sync_tile();
        }
#if HELR_NTT_EXP & 2
        if (false) {
#else
        if (!INV) {
#endif
            const int qhi = LOG_T - g * LOG_R - 1;
            const int qlo = qhi - LOG_R + 1 > 0 ? qhi - LOG_R + 1 : 0;
#pragma unroll
            for (int qb = qhi; qb >= qlo; qb--) {
                const int ls = LOG_T - 1 - qb;
                const int t0 = (wrow << ls) + (base >> (qb + 1));
                if constexpr (DBL) fwd_stage_dh<R, TWSM>(qb - lo, x, WD, t0, dc);
                else fwd_stage_h<R>(qb - lo, x, W2, t0, q, q2);
            }
        } else if (!(HELR_NTT_EXP & 2)) {
            const int qlo = g * LOG_R;
            const int qhi = (g + 1) * LOG_R < LOG_T ? (g + 1) * LOG_R - 1 : LOG_T - 1;
#pragma unroll
            for (int qb = qlo; qb <= qhi; qb++) {
                const int ls = LOG_T - 1 - qb;
                if (a.st0 == 0 && ls == 0) {
                    if constexpr (DBL) inv_last_dh<R>(qb - lo, x, tb.nid[prime], tb.i1d[prime], dc);
                    else inv_last_h<R>(qb - lo, x, tb.ninv[prime], tb.ninv_sh[prime], tb.itw1n[prime],
                                       tb.itw1n_sh[prime], q, q2);
                } else {
                    const int t0 = (wrow << ls) + (base >> (qb + 1));
                    if constexpr (DBL) inv_stage_dh<R, TWSM>(qb - lo, x, WD, t0, dc);
                    else inv_stage_h<R>(qb - lo, x, W2, t0, q, q2);
                }
            }
        }
        if (g == NG - 1) {
            u64 y[R];
            constexpr bool RAWD = has_rawd<St>::value;
            if constexpr (RAWD) sctx = st.prep(z, li);
            if constexpr (DBL && RAWD) {
#pragma unroll
                for (int i = 0; i < R; i++) y[i] = (u64)__double_as_longlong(x[i]);  // the storer reduces
            } else if constexpr (DBL) {
                // one uniform branch per pass, then straight-line conversions
                if (a.raw_out) {  // forward: |x| < 10 q; inverse: reduce the 2^8 growth
#pragma unroll
                    for (int i = 0; i < R; i++) y[i] = (u64)__double_as_longlong(INV ? reduce_d(x[i], dc) : x[i]);
                } else if (a.dbl_out) {
#pragma unroll
                    for (int i = 0; i < R; i++) y[i] = (u64)__double_as_longlong(d2d_canon(x[i], dc));
                } else {
#pragma unroll
                    for (int i = 0; i < R; i++) y[i] = d2u_canon(x[i], dc);  // canonical [0, q)
                }
            } else {
#pragma unroll
                for (int i = 0; i < R; i++) {
                    u64 v = x[i];
                    if (a.final_out) {  // forward [0, 8q), inverse [0, 4q) -> [0, q)
                        if (!INV) v = v >= q2 ? v - q2 : v;
                        v = v >= 2 * q ? v - 2 * q : v;
                        v = v >= q ? v - q : v;
                    }
                    y[i] = v;
                }
            }
            if constexpr (!IS_COL && has_tile<St>::value) {
                if (lo != 0) {
                    // the last group spreads each thread over a stride of 2^lo:
                    // consecutive threads of a block store consecutive words
                    // (full segments), no shared-memory staging needed
#pragma unroll
                    for (int i = 0; i < R; i++) ST(base + (i << lo), y[i]);
                } else {
                if (NG > 1) sync_tile();  // this group's shared-memory reads are done
#pragma unroll
                for (int i = 0; i < R; i++) sm[sidx(base + (i << lo))] = y[i];
                sync_tile();
                constexpr int TOT = T * COLS;
                constexpr int nthr = T * COLS / R;
                const int e0 = WS ? (tid >> 5) * WWORDS + 2 * (tid & 31) : 2 * tid;
                constexpr int es = WS ? 64 : 2 * nthr;
                constexpr int NIT = WS ? WWORDS / 64 : TOT / (2 * nthr);
                static_assert(NIT * es == (WS ? WWORDS : TOT), "staging loop must tile the CTA's words");
#pragma unroll (kNttEpiUnroll)
                for (int u = 0; u < NIT; u++) {
                    const int e = e0 + u * es;
                    const int c2 = e >> LOG_T, k = e & (T - 1);
                    const u64 v0 = sm[c2 * SROW + k + (k >> 4)], v1 = sm[c2 * SROW + k + 1 + ((k + 1) >> 4)];
#if HELR_NTT_EXP & 8
                    if (v0 != 0xDEADBEEFDEADBEEFull) continue;
#endif
                    if constexpr (SP) *reinterpret_cast<ulonglong2*>(scta + e) = make_ulonglong2(v0, v1);
                    else if constexpr (has_rawd<St>::value)
                        st.store2c(sctx, ((bx * COLS + c2) << LOG_T) + k, make_ulonglong2(v0, v1));
                    else st.store2(z, li, prime, ((bx * COLS + c2) << LOG_T) + k, make_ulonglong2(v0, v1));
                }
                }
            } else if constexpr (!IS_COL && has_vec<St>::value) {
                if (lo == 0) {
#pragma unroll
                    for (int i = 0; i < R; i += 2) ST2(base + i, make_ulonglong2(y[i], y[i + 1]));
                } else {
#pragma unroll
                    for (int i = 0; i < R; i++) ST(base + (i << lo), y[i]);
                }
            } else {
#pragma unroll
                for (int i = 0; i < R; i++) ST(base + (i << lo), y[i]);
            }
        } else {
            if constexpr (PRE) {
                if (g == 0) __syncthreads();  // every thread has consumed the preloaded tile
            }
#pragma unroll
            for (int i = 0; i < R; i++) sm[sidx(base + (i << lo))] = to_sm(x[i]);
            sync_tile();
        }
    }
}

#ifndef NTT_LIMB_MAJOR
#define NTT_LIMB_MAJOR 1
#endif
static inline dim3 ntt_grid(int tiles, int limbs, int items) {
    return NTT_LIMB_MAJOR ? dim3(tiles, items, limbs) : dim3(tiles, limbs, items);
}

template <int LOG_T, int LOG_R, int COLS, bool IS_COL, bool INV, int S2, class Ld, class St>
#ifndef HELR_NTT_MINB
#define HELR_NTT_MINB 4  // resident 256-thread CTAs per SM the register budget is sized for
#endif
#ifndef HELR_NTT_MINB512
#define HELR_NTT_MINB512 3  // 512-thread CTAs (radix-8 register groups, HELR_NTT_LOGR=3)
#endif
#ifndef HELR_NTT_COLTW_SMEM
#define HELR_NTT_COLTW_SMEM 1
#endif
#ifndef HELR_NTT_STAGGER
#define HELR_NTT_STAGGER 0  // ns: delay a hashed half of the first wave's CTAs (phase-stagger experiment)
#endif
__global__ void __launch_bounds__((1 << LOG_T) * COLS / (1 << LOG_R),
                                  ((1 << LOG_T) * COLS / (1 << LOG_R)) >= 512 ? HELR_NTT_MINB512 :
                                  ((1 << LOG_T) * COLS / (1 << LOG_R)) >= 256 ? HELR_NTT_MINB : 1)
ntt_pass(Ld ld, St st, Tables tb, LimbMap map, NttPassArgs a) {
    pdl_begin();
    constexpr int T = 1 << LOG_T;
    __shared__ u64 sm[IS_COL ? T * (COLS + 1) : COLS * (T + T / 16)];
    // grid: x = tiles, y = batch item, z = limb (NTT_LIMB_MAJOR) — the limb is
    // the slowest index, so the slower integer-path limb (q_0, listed first)
    // is scheduled in the first waves rather than in the tail
    const int li = NTT_LIMB_MAJOR ? blockIdx.z : blockIdx.y, z = NTT_LIMB_MAJOR ? blockIdx.y : blockIdx.z;
#if HELR_NTT_STAGGER
    {
        const unsigned lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        if (gridDim.x * gridDim.y * gridDim.z >= 1184 && lin < 592 && ((lin * 2654435761u) >> 31)) {
            unsigned long long t0, t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            do {
                __nanosleep(100);
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            } while (t1 - t0 < HELR_NTT_STAGGER);
        }
    }
#endif
    constexpr bool TWS = kColTwSmem && IS_COL && LOG_T >= 6 && ((1 << LOG_T) <= (1 << LOG_T) * COLS / (1 << LOG_R));
    __shared__ __align__(16) double tws[TWS ? T : 1];
    if (tb.q[map.prime[li]] < NTT_DBL_BOUND) {
        // column passes: one coalesced read of the limb's 2^LOG_T-entry table
        // per CTA, issued by the body behind its tile loads (TWFILL)
        ntt_body<LOG_T, LOG_R, COLS, IS_COL, INV, S2, true, Ld, St, false, TWS, TWS>(ld, st, tb, map, a, sm, blockIdx.x, li, z,
                                                                                     tws);
    } else
        ntt_body<LOG_T, LOG_R, COLS, IS_COL, INV, S2, false>(ld, st, tb, map, a, sm, blockIdx.x, li, z);
}

// ---- plain functors: strided limb buffers -------------------------------
#ifndef HELR_STBUF_TILE
#define HELR_STBUF_TILE true
#endif
struct LdBuf {
    static constexpr bool kVec = true;
    static constexpr bool kTile = HELR_STBUF_TILE;
    static constexpr bool kPtr = true;
    const u64* base;
    long long item_stride;
    LimbMap map;  // copy of the offsets (small)
    int n;
    __device__ __forceinline__ const u64* limb_ptr(int z, int li) const {
        return base + (size_t)z * item_stride + (size_t)map.off[li] * n;
    }
    __device__ __forceinline__ u64 operator()(int z, int li, int, int off) const {
        return base[(size_t)z * item_stride + (size_t)map.off[li] * n + off];
    }
    __device__ __forceinline__ ulonglong2 load2(int z, int li, int, int off) const {
        return *reinterpret_cast<const ulonglong2*>(base + (size_t)z * item_stride + (size_t)map.off[li] * n + off);
    }
};
struct StBuf {
    static constexpr bool kVec = true;
    static constexpr bool kTile = HELR_STBUF_TILE;
    static constexpr bool kPtr = true;
    u64* base;
    long long item_stride;
    LimbMap map;
    int n;
    __device__ __forceinline__ u64* limb_ptr(int z, int li) const {
        return base + (size_t)z * item_stride + (size_t)map.off[li] * n;
    }
    __device__ __forceinline__ void operator()(int z, int li, int, int off, u64 v) const {
        base[(size_t)z * item_stride + (size_t)map.off[li] * n + off] = v;
    }
    __device__ __forceinline__ void store2(int z, int li, int, int off, ulonglong2 v) const {
        *reinterpret_cast<ulonglong2*>(base + (size_t)z * item_stride + (size_t)map.off[li] * n + off) = v;
    }
};

#include "ntt_tma.cuh"

// ---- host-side dispatch ----------------------------------------------------
// Launch one NTT (forward or inverse) over `count` items x map.count limbs.
// The first pass reads through `ld`, the last pass writes through `st`; with
// two passes the intermediate goes through `mid` (item stride mid_stride,
// limb offsets from map) which may alias the storer's buffer.
// Launches of fewer than NTT_SMALL_GRID full-size CTAs (single-ciphertext
// key switches at low levels) use CTAs a quarter the size, so four times as
// many SMs share the latency-bound work.
#ifndef HELR_NTT_SMALL_GRID
#define HELR_NTT_SMALL_GRID (2 * 148)
#endif
constexpr long long NTT_SMALL_GRID = HELR_NTT_SMALL_GRID;
#ifndef HELR_NTT_COLS
#define HELR_NTT_COLS 16  // adjacent columns per column-pass CTA (16 x 8 B = one 128-byte segment)
#endif
#ifndef HELR_NTT_SMALL_LOGR
#define HELR_NTT_SMALL_LOGR 2
#endif
#ifndef HELR_NTT_LOGR
#define HELR_NTT_LOGR 4  // log2 of the elements a thread holds (radix-16 register groups)
#endif

template <int LOG_T, bool IS_COL, bool INV, int S2, class Ld, class St>
static void ntt_pass_launch(const Ld& ld, const St& st, const Tables& tb, const LimbMap& map,
                            int log_n, int st0, int final_out, int count, cudaStream_t s, int raw_in = 0,
                            int raw_out = 0, int dbl_out = 0) {
    constexpr int LOG_R = LOG_T < HELR_NTT_LOGR ? LOG_T : HELR_NTT_LOGR;
    constexpr int T = 1 << LOG_T;
    // column passes: 16 adjacent columns (128-byte rows); row passes: ~4096 elements per CTA
    constexpr int COLS_ROW = (4096 / T) > 0 ? (4096 / T) : 1;
    constexpr int COLS = IS_COL ? HELR_NTT_COLS : COLS_ROW;
    constexpr int COLS_S = COLS >= 4 ? COLS / 4 : 1;
    const int subs = IS_COL ? (1 << (log_n - LOG_T)) : (1 << (log_n - LOG_T));
    const int cols = subs < COLS ? subs : COLS;  // tiny rings: fewer sub-transforms than COLS
    NttPassArgs a{log_n, st0, final_out, raw_in, raw_out, dbl_out};
    count_launches(1);
    // large launches at N = 2^16 from plain buffers: persistent CTAs whose next
    // tile arrives by TMA while the current one computes (ntt_tma.cuh)
    if constexpr (std::is_same<Ld, LdBuf>::value && LOG_T == ntma::LOG_T && COLS == ntma::COLS &&
                  (!IS_COL || S2 == ntma::LOG_N - ntma::LOG_T)) {
        if (ntma::usable(log_n, ld, map, count) && ntma::launch<IS_COL, INV>(ld, st, tb, map, a, count, s)) return;
    }
    if (cols == COLS) {
        const long long full = (long long)(subs / COLS) * map.count * count;
        if (COLS_S < COLS && full < NTT_SMALL_GRID && log_n >= 12) {
            // small grids (single-ciphertext key switches, W/V updates) are
            // latency-bound: quarter-size tiles, and radix-4 register groups
            // so each tile has 4x the threads (more warps per SM in flight)
            constexpr int LOG_RS = LOG_T >= 6 ? HELR_NTT_SMALL_LOGR : LOG_R;
            dim3 grid = ntt_grid(subs / COLS_S, map.count, count);
            launch_pdl(ntt_pass<LOG_T, LOG_RS, COLS_S, IS_COL, INV, S2, Ld, St>, grid,
                       dim3(T * COLS_S / (1 << LOG_RS)), 0, s, ld, st, tb, map, a);
            return;
        }
        dim3 grid = ntt_grid(subs / COLS, map.count, count);
        launch_pdl(ntt_pass<LOG_T, LOG_R, COLS, IS_COL, INV, S2, Ld, St>, grid, dim3(T * COLS / (1 << LOG_R)), 0, s, ld, st, tb,
                   map, a);
    } else {
        // only reachable for single-pass rings (subs == 1)
        dim3 grid = ntt_grid(subs / cols, map.count, count);
        launch_pdl(ntt_pass<LOG_T, LOG_R, 1, IS_COL, INV, S2, Ld, St>, grid, dim3(T / (1 << LOG_R)), 0, s, ld, st, tb, map, a);
    }
}

template <bool INV, class Ld, class St>
static void ntt_single(int log_n, const Ld& ld, const St& st, const Tables& tb, const LimbMap& map,
                       int count, cudaStream_t s, int in_raw, int out_dbl) {
    switch (log_n) {
#define HELR_SP(LT) \
    case LT: ntt_pass_launch<LT, false, INV, 0>(ld, st, tb, map, log_n, 0, 1, count, s, in_raw, 0, out_dbl); break;
        HELR_SP(2) HELR_SP(3) HELR_SP(4) HELR_SP(5) HELR_SP(6) HELR_SP(7) HELR_SP(8) HELR_SP(9)
        HELR_SP(10) HELR_SP(11)
#undef HELR_SP
        default: break;
    }
}

template <bool INV, class Ld, class St>
static void ntt_col(int lt, int log_n, const Ld& ld, const St& st, const Tables& tb, const LimbMap& map,
                    int final_out, int count, cudaStream_t s, int raw_in, int raw_out, int dbl_out) {
    // column pass of log N = LN: LT = floor(LN / 2) stages (= lt), element stride 2^(LN - LT)
    (void)lt;
    switch (log_n) {
#define HELR_CP(LN) \
    case LN: \
        ntt_pass_launch<(LN) / 2, true, INV, (LN) - (LN) / 2>(ld, st, tb, map, log_n, 0, final_out, count, s, raw_in, \
                                                              raw_out, dbl_out); \
        break;
        HELR_CP(12) HELR_CP(13) HELR_CP(14) HELR_CP(15) HELR_CP(16)
#undef HELR_CP
        default: break;
    }
}

template <bool INV, class Ld, class St>
static void ntt_row(int lt, int log_n, const Ld& ld, const St& st, const Tables& tb, const LimbMap& map,
                    int final_out, int count, cudaStream_t s, int raw_in, int raw_out, int dbl_out) {
    const int st0 = log_n - lt;
    switch (lt) {
#define HELR_RP(LT) \
    case LT: \
        ntt_pass_launch<LT, false, INV, 0>(ld, st, tb, map, log_n, st0, final_out, count, s, raw_in, raw_out, dbl_out); \
        break;
        HELR_RP(6) HELR_RP(7) HELR_RP(8) HELR_RP(9)
#undef HELR_RP
        default: break;
    }
}

inline int ntt_split_s1(int log_n) { return log_n / 2; }

// limbs a fused storer reads besides the transform's own input (byte model);
// overloaded for StCombine in ks.cuh
template <class St>
inline double ntt_extra_words(const St&, const LimbMap&, int) { return 0.0; }

// single-pass 8-CTA cluster NTT for N = 2^16 (ntt_cluster.cuh): measured
// slower than the two passes below, so it is only compiled
// with -DHELR_NTT_CLUSTER_BUILD=1 (HELR_NVCC_DEFS) and enabled by HELR_NTT_CLUSTER=1
#ifndef HELR_NTT_CLUSTER_BUILD
#define HELR_NTT_CLUSTER_BUILD 0
#endif
#if HELR_NTT_CLUSTER_BUILD
#include "ntt_cluster.cuh"
#endif


template <bool INV, class Ld, class St>
// in_raw: fp64 limbs arrive as raw integer-valued doubles (|x| < 2^50);
// out_dbl: fp64 limbs leave as canonical residues stored as exact doubles
static void ntt_launch(const helr_ctx* c, const Ld& ld, const St& st, u64* mid, long long mid_stride,
                       const LimbMap& map, int count, cudaStream_t s, int in_raw = 0, int out_dbl = 0) {
    const int log_n = c->log_n;
    // algorithmic bytes: every limb read and written once, plus the extra
    // operands a fused storer reads once (StCombine: ntt_extra_words)
    ProfScope ps(PROF_NTT, 8.0 * c->n * (2.0 * map.count * count + ntt_extra_words(st, map, count)), s);
#if HELR_NTT_CLUSTER_BUILD
    if (log_n == ncl::LOG_N && ntt_cluster_enabled((long long)map.count * count)) {
        ntt_cluster_launch<INV>(ld, st, c->t, map, count, s, in_raw, out_dbl);
        return;
    }
#endif
    if (log_n <= 11) {
        ntt_single<INV>(log_n, ld, st, c->t, map, count, s, in_raw, out_dbl);
        return;
    }
    const int s1 = ntt_split_s1(log_n), s2 = log_n - s1;
    StBuf smid{mid, mid_stride, map, c->n};
    LdBuf lmid{mid, mid_stride, map, c->n};
    if (!INV) {
        ntt_col<false>(s1, log_n, ld, smid, c->t, map, 0, count, s, in_raw, 1, 0);
        ntt_row<false>(s2, log_n, lmid, st, c->t, map, 1, count, s, 1, 0, out_dbl);
    } else {
        ntt_row<true>(s2, log_n, ld, smid, c->t, map, 0, count, s, in_raw, 1, 0);
        ntt_col<true>(s1, log_n, lmid, st, c->t, map, 1, count, s, 1, 0, out_dbl);
    }
}

// Plain buffer-to-buffer NTT (in-place when in == out).
template <bool INV>
static void ntt_buffers(const helr_ctx* c, const u64* in, long long in_stride, u64* out, long long out_stride,
                        const LimbMap& map, int count, cudaStream_t s, int in_raw = 0, int out_dbl = 0) {
    LdBuf ld{in, in_stride, map, c->n};
    StBuf st{out, out_stride, map, c->n};
    ntt_launch<INV>(c, ld, st, out, out_stride, map, count, s, in_raw, out_dbl);
}
