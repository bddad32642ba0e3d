// ntt_cluster.cuh — single-pass negacyclic NTT for N = 2^16 on one 8-CTA
// thread-block cluster per limb (included at the end of ntt.cuh).
//
// Why.  The two-pass NTT (ntt_pass) moves every element through HBM/L2
// twice per transform (input -> mid buffer -> output) and its passes wait on
// global-load latency.  Here the 512 KB limb lives in the cluster's
// distributed shared memory: 8 CTAs x 64 KB, 2 CTAs per SM (one loads while
// the other computes), so a limb is read once and written once.
//
// Layout.  Index k = 256 row + col.  The first 8 forward stages mix rows
// (bits 15..8, "column" transforms), the last 8 mix columns (bits 7..0,
// "row" transforms).
//   phase A (columns): CTA r of the cluster owns columns 32r..32r+31 of all
//     256 rows: dense smem tile [256][32] (a row segment is 256 contiguous
//     bytes in HBM: cp.async.bulk per row, completion on an mbarrier).
//   exchange: after a cluster barrier every thread writes its 16 values
//     straight into the owning CTA's shared memory (st.shared::cluster,
//     coalesced: a warp writes 32 consecutive columns of one row).
//   phase B (rows): CTA r owns rows 32r..32r+31: smem [32][256] with the
//     column index XOR-swizzled inside each 16-word chunk
//     (phys = col ^ ((col >> 4) & 15)) so both register-group access
//     patterns (col = s + 16 i and col = 16 s + i) are bank-conflict free.
// Each phase is two radix-16 register groups (4 stages each) exchanging
// through shared memory — the same stage kernels, twiddle indexing and
// exact arithmetic (fp64 for primes < 2^41, Harvey/Shoup integers for q_0)
// as ntt_pass, so the results are the same residues.  The inverse runs the
// same plan transposed (rows first), with one exact fp64 reduction before the
// exchange (the Gentleman-Sande sum path doubles per stage).
#pragma once

namespace ncl {
constexpr int LOG_N = 16;
constexpr int NN = 1 << LOG_N;
constexpr int CL = 8;         // CTAs per cluster = per limb
constexpr int TH = 512;       // threads per CTA
constexpr int EL = NN / CL;   // 8192 elements (64 KB) per CTA
constexpr int SMEM = EL * 8;
}  // namespace ncl

struct NttClArgs {
    int in_raw;   // fp64 limbs arrive as raw integer-valued doubles
    int dbl_out;  // fp64 limbs leave as canonical residues stored as exact doubles
    int bulk;     // plain buffers: cp.async.bulk for the dense phase (forward load / inverse store)
    int xasync;   // exchange by st.async + mbarrier (1) or st.shared::cluster + cluster barrier (0)
};

#include "async.cuh"

// row-phase swizzle: permute each 16-word (128-byte) chunk by the chunk index
__device__ __forceinline__ int swz(int col) { return col ^ ((col >> 4) & 15); }

template <bool INV, bool DBL, class Ld, class St>
__device__ __forceinline__ void ntt_cl_body(const Ld& ld, const St& st, const Tables& tb, const LimbMap& map,
                                            const NttClArgs& a, u64* sm, u64* bars, const int li, const int z) {
    u64* bar = bars;        // bulk tile load
    u64* xbar = bars + 1;   // exchange arrivals
    using V = typename std::conditional<DBL, double, u64>::type;
    constexpr int R = 16;
    const int r = (int)cl_rank();
    const int tid = threadIdx.x;
    const int prime = map.prime[li];
    const u64 q = tb.q[prime];
    const u64 q2 = 4 * q;
    DblC dc;
    if constexpr (DBL) dc = DblC{tb.qd[prime], tb.qinvd[prime]};
    const ulonglong2* W2 = reinterpret_cast<const ulonglong2*>(INV ? tb.itw : tb.tw) + (size_t)prime * ncl::NN;
    const double* WD = (INV ? tb.itwd : tb.twd) + (size_t)prime * ncl::NN;

    constexpr bool LP = has_ptr<Ld>::value, SP = has_ptr<St>::value;
    const bool raw_in = DBL && a.in_raw;
    auto in_v = [&](u64 v) -> V {
        if constexpr (DBL) return raw_in ? __longlong_as_double((long long)v) : u2d(v);
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
    auto canon = [&](V v) -> u64 {
        if constexpr (DBL) {
            return a.dbl_out ? (u64)__double_as_longlong(d2d_canon(v, dc)) : d2u_canon(v, dc);
        } else {
            u64 y = v;
            if (!INV) y = y >= q2 ? y - q2 : y;  // forward lazy range [0, 8q)
            y = y >= 2 * q ? y - 2 * q : y;
            return y >= q ? y - q : y;
        }
    };
    auto LD = [&](int off) -> u64 {
        if constexpr (LP) return ld.limb_ptr(z, li)[off];
        else return ld(z, li, prime, off);
    };
    auto LD2 = [&](int off) -> ulonglong2 {
        if constexpr (LP) return *reinterpret_cast<const ulonglong2*>(ld.limb_ptr(z, li) + off);
        else if constexpr (has_vec<Ld>::value) return ld.load2(z, li, prime, off);
        else return make_ulonglong2(ld(z, li, prime, off), ld(z, li, prime, off + 1));
    };
    auto ST = [&](int off, u64 v) {
        if constexpr (SP) st.limb_ptr(z, li)[off] = v;
        else st(z, li, prime, off, v);
    };
    auto ST2 = [&](int off, ulonglong2 v) {
        if constexpr (SP) *reinterpret_cast<ulonglong2*>(st.limb_ptr(z, li) + off) = v;
        else if constexpr (has_vec<St>::value) st.store2(z, li, prime, off, v);
        else { st(z, li, prime, off, v.x); st(z, li, prime, off + 1, v.y); }
    };
    // one forward / inverse stage on bit qb of a 256-point sub-transform whose
    // twiddle row is wrow; base = this thread's index with the register bits zero
    auto fstage = [&](V (&x)[R], int qb, int lo, int wrow, int base) {
        const int ls = 7 - qb;
        const int t0 = (wrow << ls) + (base >> (qb + 1));
        if constexpr (DBL) fwd_stage_dh<R>(qb - lo, x, WD, t0, dc);
        else fwd_stage_h<R>(qb - lo, x, W2, t0, q, q2);
    };
    auto istage = [&](V (&x)[R], int qb, int lo, int wrow, int base, bool last_pass) {
        const int ls = 7 - qb;
        if (last_pass && ls == 0) {
            if constexpr (DBL) inv_last_dh<R>(qb - lo, x, tb.nid[prime], tb.i1d[prime], dc);
            else inv_last_h<R>(qb - lo, x, tb.ninv[prime], tb.ninv_sh[prime], tb.itw1n[prime], tb.itw1n_sh[prime], q, q2);
        } else {
            const int t0 = (wrow << ls) + (base >> (qb + 1));
            if constexpr (DBL) inv_stage_dh<R>(qb - lo, x, WD, t0, dc);
            else inv_stage_h<R>(qb - lo, x, W2, t0, q, q2);
        }
    };

    V x[R];
    if (a.xasync) {
        // every CTA receives exactly its 64 KB tile from the 8 CTAs of the cluster
        if (tid == 0) {
            mbar_init(xbar, 1);
            mbar_expect_tx(xbar, ncl::SMEM);
        }
    }
    auto exch_begin = [&]() {
        if (a.xasync) cl_sync_relaxed();  // tiles read (and xbar initialised) cluster-wide
        else cl_sync();
    };
    auto exch_put = [&](unsigned addr, unsigned rank, u64 v) {
        if (a.xasync) cl_st_async(addr, v, cl_map(smem_u32(xbar), rank));
        else cl_st(addr, v);
    };
    auto exch_end = [&]() {
        if (a.xasync) mbar_wait(xbar, 0);
        else cl_sync();
    };
    // column-phase thread map: cc = column in the CTA's 32, s = 16-thread slot
    const int cc = tid & 31, s = tid >> 5;
    // row-phase thread map: s2 = slot, rr = row in the CTA's 32
    const int s2 = tid & 15, rr = tid >> 4;
    const int col = 32 * r + cc;        // this thread's global column (column phase)
    const int row = 32 * r + rr;        // this thread's global row (row phase)
    u64* rowp = sm + rr * 256;          // this thread's row in the row-phase tile

    if constexpr (!INV) {
        // ---------------- phase A: stages 0..7 on the row index (columns)
        if constexpr (LP) {
            if (a.bulk) {
                if (tid == 0) mbar_init(bar, 1);
                __syncthreads();
                if (tid < 32) {
                    if (tid == 0) mbar_expect_tx(bar, ncl::SMEM);
                    __syncwarp();
                    const u64* g = ld.limb_ptr(z, li) + 32 * r;
#pragma unroll
                    for (int k = tid; k < 256; k += 32) bulk_g2s(sm + k * 32, g + k * 256, 256, bar);
                }
                mbar_wait(bar, 0);
#pragma unroll
                for (int i = 0; i < R; i++) x[i] = in_v(sm[(s + 16 * i) * 32 + cc]);
            } else {
#pragma unroll
                for (int i = 0; i < R; i++) x[i] = in_v(LD((s + 16 * i) * 256 + col));
            }
        } else {
#pragma unroll
            for (int i = 0; i < R; i++) x[i] = in_v(LD((s + 16 * i) * 256 + col));
        }
#pragma unroll
        for (int qb = 7; qb >= 4; qb--) fstage(x, qb, 4, 1, s);
        // (each thread overwrites exactly the words it read: no barrier needed)
#pragma unroll
        for (int i = 0; i < R; i++) sm[(s + 16 * i) * 32 + cc] = to_sm(x[i]);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < R; i++) x[i] = from_sm(sm[(16 * s + i) * 32 + cc]);
#pragma unroll
        for (int qb = 3; qb >= 0; qb--) fstage(x, qb, 0, 1, s << 4);
        // ---------------- exchange: rows k = 16 s + i go to CTA s >> 1
        exch_begin();
        {
            const unsigned dst = cl_map(smem_u32(sm), (unsigned)(s >> 1)) + 8u * (unsigned)((16 * (s & 1)) * 256 + swz(col));
#pragma unroll
            for (int i = 0; i < R; i++) exch_put(dst + 8u * (unsigned)(i * 256), (unsigned)(s >> 1), to_sm(x[i]));
        }
        exch_end();
        // ---------------- phase B: stages 8..15 on the column index (rows)
        const int wrow = 256 + row;
#pragma unroll
        for (int i = 0; i < R; i++) x[i] = from_sm(rowp[swz(s2 + 16 * i)]);
#pragma unroll
        for (int qb = 7; qb >= 4; qb--) fstage(x, qb, 4, wrow, s2);
#pragma unroll
        for (int i = 0; i < R; i++) rowp[swz(s2 + 16 * i)] = to_sm(x[i]);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < R; i++) x[i] = from_sm(rowp[swz(16 * s2 + i)]);
#pragma unroll
        for (int qb = 3; qb >= 0; qb--) fstage(x, qb, 0, wrow, s2 << 4);
        // ---------------- epilogue: canonical outputs (into the words this
        // thread read), then coalesced pair stores
#pragma unroll
        for (int i = 0; i < R; i++) rowp[swz(16 * s2 + i)] = canon(x[i]);
        __syncthreads();
#pragma unroll 4
        for (int e = 2 * tid; e < ncl::EL; e += 2 * ncl::TH) {
            const int rw = e >> 8, c2 = e & 255;
            const int p = swz(c2);  // c2 even: (p, p ^ 1) is an aligned pair
            const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(sm + rw * 256 + (p & ~1));
            ST2((32 * r + rw) * 256 + c2, (p & 1) ? make_ulonglong2(v.y, v.x) : v);
        }
    } else {
        // ---------------- phase 1: inverse stages on the column index (rows)
#pragma unroll 4
        for (int e = 2 * tid; e < ncl::EL; e += 2 * ncl::TH) {
            const int rw = e >> 8, c2 = e & 255;
            const int p = swz(c2);
            const ulonglong2 v = LD2((32 * r + rw) * 256 + c2);
            *reinterpret_cast<ulonglong2*>(sm + rw * 256 + (p & ~1)) = (p & 1) ? make_ulonglong2(v.y, v.x) : v;
        }
        __syncthreads();
        const int wrow = 256 + row;
#pragma unroll
        for (int i = 0; i < R; i++) x[i] = in_v(rowp[swz(16 * s2 + i)]);
#pragma unroll
        for (int qb = 0; qb <= 3; qb++) istage(x, qb, 0, wrow, s2 << 4, false);
#pragma unroll
        for (int i = 0; i < R; i++) rowp[swz(16 * s2 + i)] = to_sm(x[i]);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < R; i++) x[i] = from_sm(rowp[swz(s2 + 16 * i)]);
#pragma unroll
        for (int qb = 4; qb <= 7; qb++) istage(x, qb, 4, wrow, s2, false);
        if constexpr (DBL) {
#pragma unroll
            for (int i = 0; i < R; i++) x[i] = reduce_d(x[i], dc);  // 2^8 growth of the sum path
        }
        // ---------------- exchange: column s2 + 16 i goes to CTA i >> 1 (dense [256][32] tile)
        exch_begin();
        {
            const unsigned base = smem_u32(sm) + 8u * (unsigned)(row * 32 + s2);
#pragma unroll
            for (int i = 0; i < R; i++)
                exch_put(cl_map(base + 8u * (unsigned)(16 * (i & 1)), (unsigned)(i >> 1)), (unsigned)(i >> 1), to_sm(x[i]));
        }
        exch_end();
        // ---------------- phase 2: inverse stages on the row index (columns)
#pragma unroll
        for (int i = 0; i < R; i++) x[i] = from_sm(sm[(16 * s + i) * 32 + cc]);
#pragma unroll
        for (int qb = 0; qb <= 3; qb++) istage(x, qb, 0, 1, s << 4, true);
#pragma unroll
        for (int i = 0; i < R; i++) sm[(16 * s + i) * 32 + cc] = to_sm(x[i]);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < R; i++) x[i] = from_sm(sm[(s + 16 * i) * 32 + cc]);
#pragma unroll
        for (int qb = 4; qb <= 7; qb++) istage(x, qb, 4, 1, s, true);
        if constexpr (SP) {
            if (a.bulk) {
#pragma unroll
                for (int i = 0; i < R; i++) sm[(s + 16 * i) * 32 + cc] = canon(x[i]);
                fence_async_smem();
                __syncthreads();
                if (tid < 32) {
                    u64* g = st.limb_ptr(z, li) + 32 * r;
#pragma unroll
                    for (int k = tid; k < 256; k += 32) bulk_s2g(g + k * 256, sm + k * 32, 256);
                    bulk_commit_wait();
                }
                return;
            }
        }
#pragma unroll
        for (int i = 0; i < R; i++) ST((s + 16 * i) * 256 + col, canon(x[i]));
    }
}

template <bool INV, class Ld, class St>
__global__ void __cluster_dims__(ncl::CL, 1, 1) __launch_bounds__(ncl::TH, 2)
    ntt_cluster(Ld ld, St st, Tables tb, LimbMap map, NttClArgs a) {
    extern __shared__ __align__(128) u64 ncl_sm[];
    __shared__ __align__(8) u64 bars[2];
    pdl_begin();
    const int li = blockIdx.z, z = blockIdx.y;
    if (tb.q[map.prime[li]] < NTT_DBL_BOUND)  // uniform per cluster (one limb per cluster)
        ntt_cl_body<INV, true>(ld, st, tb, map, a, ncl_sm, bars, li, z);
    else
        ntt_cl_body<INV, false>(ld, st, tb, map, a, ncl_sm, bars, li, z);
}

bool ntt_cluster_enabled(long long limb_transforms);
bool ntt_bulk_enabled();
bool ntt_xasync_enabled();

template <bool INV, class Ld, class St>
static void ntt_cluster_launch(const Ld& ld, const St& st, const Tables& tb, const LimbMap& map, int count,
                               cudaStream_t s, int in_raw, int out_dbl) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(ntt_cluster<INV, Ld, St>, cudaFuncAttributeMaxDynamicSharedMemorySize, ncl::SMEM);
        attr = true;
    }
    NttClArgs a{in_raw, out_dbl, ntt_bulk_enabled() ? 1 : 0, ntt_xasync_enabled() ? 1 : 0};
    count_launches(1);
    launch_pdl(ntt_cluster<INV, Ld, St>, dim3(ncl::CL, count, map.count), dim3(ncl::TH), (size_t)ncl::SMEM, s, ld, st,
               tb, map, a);
}
