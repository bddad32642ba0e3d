// ntt_tma.cuh — persistent, TMA-fed NTT passes for N = 2^16 (included by ntt.cuh).
//
// The plain passes (ntt_pass) run load -> butterflies -> store once per CTA;
// with ~2 waves of CTAs the load phases of a wave coincide, so a pass costs
// about (memory time + fp64 time) although the two are of similar size.  Here
// each CTA walks a strided list of tiles and the NEXT tile's 32 KB arrive by
// one cp.async.bulk.tensor (UTMALDG, completion on an mbarrier) while the
// current tile's butterflies run: no issue slots, no registers and no LSU
// traffic are spent on the prefetch.
//
//   tile (row pass)    : 4096 contiguous words = [256 rows][16 words], loaded
//                        with the 128-byte hardware swizzle so both register
//                        layouts (stride-16 words, 16 contiguous words) read
//                        it without bank conflicts;
//   tile (column pass) : 16 adjacent columns x 256 rows (row pitch 2 KB),
//                        dense [256][16].
//
// Two 34 KB buffers per CTA: the tile lands in one, is consumed into
// registers, and the same buffer then carries the padded exchange between the
// register groups and the output staging; the other buffer receives the next
// tile meanwhile.  3 CTAs per SM.  Stores stay ordinary coalesced st.global
// (fire-and-forget).  Arithmetic is ntt_body's, so residues are identical to
// the plain passes (tests/test_gpu_parity.py runs both).
#pragma once
#include <cuda.h>

#include "async.cuh"

namespace ntma {

constexpr int LOG_N = 16;
constexpr int LOG_T = 8;
constexpr int LOG_R = 4;
constexpr int COLS = 16;
constexpr int TILE_WORDS = 4096;
constexpr int BUF_WORDS = 4352;  // padded exchange layout (T * 17 = 16 * (T + T / 16))
constexpr int THREADS = 256;
constexpr int TILES_PER_LIMB = (1 << LOG_N) / TILE_WORDS;
constexpr size_t SMEM_BYTES = 2 * BUF_WORDS * 8 + 64 + 1024;  // + barriers + alignment slack
#ifndef HELR_NTT_TMA_CTAS
#define HELR_NTT_TMA_CTAS 3  // resident CTAs per SM
#endif

struct Geom {
    long long item_stride;  // words between batch items in the source buffer
    int count;              // batch items
    int total;              // tiles = TILES_PER_LIMB * limbs * items
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, u64* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

template <bool IS_COL, bool INV, class St>
__global__ void __launch_bounds__(THREADS, HELR_NTT_TMA_CTAS)
ntt_pass_tma(const __grid_constant__ CUtensorMap tmap, Geom g, LdBuf ld, St st, Tables tb, LimbMap map, NttPassArgs a) {
    extern __shared__ unsigned char ntma_raw[];
    u64* buf = reinterpret_cast<u64*>((reinterpret_cast<uintptr_t>(ntma_raw) + 1023) & ~(uintptr_t)1023);
    u64* bars = buf + 2 * BUF_WORDS;
    __shared__ __align__(16) double tws[IS_COL ? (1 << LOG_T) : 1];
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bars + 0, 1);
        mbar_init(bars + 1, 1);
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
    }
    __syncthreads();
    pdl_begin();
    const int G = gridDim.x;
    // tile id = (limb * items + item) * TILES_PER_LIMB + tile: limb slowest, so
    // the integer-path limb (listed first) is scheduled first
    auto issue = [&](int t, int b) {
        const int bx = t % TILES_PER_LIMB, lz = t / TILES_PER_LIMB;
        const int li = lz / g.count, z = lz - li * g.count;
        const long long w0 = (long long)z * g.item_stride + (long long)map.off[li] * (1 << LOG_N);
        mbar_expect_tx(bars + b, TILE_WORDS * 8);
        if (IS_COL) tma_load_2d(buf + b * BUF_WORDS, &tmap, bx * COLS, (int)(w0 >> 8), bars + b);
        else tma_load_2d(buf + b * BUF_WORDS, &tmap, 0, (int)(w0 >> 4) + bx * (TILE_WORDS / 16), bars + b);
    };
    int t = blockIdx.x;
    if (tid == 0 && t < g.total) issue(t, 0);
    for (int it = 0; t < g.total; it++, t += G) {
        const int b = it & 1;
        if (tid == 0 && t + G < g.total) issue(t + G, b ^ 1);  // its buffer was released by the previous tile's closing barrier
        const int bx = t % TILES_PER_LIMB, lz = t / TILES_PER_LIMB;
        const int li = lz / g.count, z = lz - li * g.count;
        constexpr int S2 = IS_COL ? LOG_N - LOG_T : 0;
        constexpr bool TWS = kColTwSmem && IS_COL;
        const bool dbl = tb.q[map.prime[li]] < NTT_DBL_BOUND;
        if constexpr (TWS) {
            // the limb's 255 column-pass twiddles into shared memory (the
            // previous tile's closing barrier released the table)
            if (dbl) tws[tid] = __ldg((INV ? tb.itwd : tb.twd) + ((size_t)map.prime[li] << LOG_N) + tid);
        }
        mbar_wait(bars + b, (it >> 1) & 1);
        if constexpr (TWS) __syncthreads();
        u64* sm = buf + b * BUF_WORDS;
        if (dbl)
            ntt_body<LOG_T, LOG_R, COLS, IS_COL, INV, S2, true, LdBuf, St, true, TWS>(ld, st, tb, map, a, sm, bx, li, z, tws);
        else
            ntt_body<LOG_T, LOG_R, COLS, IS_COL, INV, S2, false, LdBuf, St, true>(ld, st, tb, map, a, sm, bx, li, z);
        // generic-proxy accesses of this buffer are ordered before the bulk
        // copy (async proxy) that refills it two tiles from now
        fence_async_smem();
        __syncthreads();
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline EncodeFn encode_fn() {
    static EncodeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) != cudaSuccess ||
            qr != cudaDriverEntryPointSuccess)
            p = nullptr;
        cudaGetLastError();
        return (EncodeFn)p;
    }();
    return fn;
}

inline int sm_count() {
    static int n = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

// HELR_NTT_TMA=1 turns the path on.  Default off: measured slower than the
// plain passes (0.60 vs 0.50 us per fp64 limb at 112 limbs) —
// ncu shows the passes wait on the per-stage twiddle loads, not on the tile.
inline int mode() {  // 1: both passes, 2: column passes only, 3: row passes only
    static int on = [] {
        const char* v = getenv("HELR_NTT_TMA");
        return v ? atoi(v) : 0;
    }();
    return on;
}
inline bool enabled() { return mode() != 0; }
// launches with fewer tiles keep the quarter-size plain tiles
// (HELR_NTT_TMA_MIN_TILES overrides, e.g. 1 in the parity tests)
inline long long min_tiles() {
    static long long v = [] {
        const char* e = getenv("HELR_NTT_TMA_MIN_TILES");
        return e ? atoll(e) : 2ll * 148;
    }();
    return v;
}

// words spanned by the source buffer from its base: every (item, limb) of the launch
inline long long extent_words(const LdBuf& ld, const LimbMap& map, int count) {
    int mo = 0;
    for (int i = 0; i < map.count; i++) mo = map.off[i] > mo ? map.off[i] : mo;
    return (long long)(count - 1) * ld.item_stride + (long long)(mo + 1) * ld.n;
}

inline bool usable(int log_n, const LdBuf& ld, const LimbMap& map, int count) {
    if (!enabled() || log_n != LOG_N || !encode_fn()) return false;
    if ((long long)TILES_PER_LIMB * map.count * count < min_tiles()) return false;
    if (ld.item_stride < 0 || (ld.item_stride & 255) || (reinterpret_cast<uintptr_t>(ld.base) & 15)) return false;
    return extent_words(ld, map, count) < (1ll << 39);
}

template <bool IS_COL, bool INV, class St>
static bool launch(const LdBuf& ld, const St& st, const Tables& tb, const LimbMap& map, const NttPassArgs& a, int count,
                   cudaStream_t s) {
    if ((mode() == 2 && !IS_COL) || (mode() == 3 && IS_COL)) return false;
    const long long ext = extent_words(ld, map, count);
    CUtensorMap tm;
    cuuint64_t dims[2], strides[1];
    cuuint32_t box[2], es[2] = {1, 1};
    if (IS_COL) {  // [rows of 256 words][256]; box = 16 columns x 256 rows
        dims[0] = 256; dims[1] = (cuuint64_t)((ext + 255) >> 8); strides[0] = 2048; box[0] = COLS; box[1] = 256;
    } else {       // [rows of 16 words][16]; box = one 4096-word tile
        dims[0] = 16; dims[1] = (cuuint64_t)((ext + 15) >> 4); strides[0] = 128; box[0] = 16; box[1] = 256;
    }
    CUresult r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<u64*>(ld.base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, IS_COL ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    auto kern = ntt_pass_tma<IS_COL, INV, St>;
    static bool attr_set = false;  // one flag per instantiation
    if (!attr_set) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        attr_set = true;
    }
    Geom g{ld.item_stride, count, TILES_PER_LIMB * map.count * count};
    const int slots = HELR_NTT_TMA_CTAS * sm_count();
    const int grid = g.total < slots ? g.total : slots;
    launch_pdl(kern, dim3(grid), dim3(THREADS), SMEM_BYTES, s, tm, g, ld, st, tb, map, a);
    return true;
}

}  // namespace ntma
