// conv.cuh — basis conversions fused into the NTT passes (ModUp / ModDown /
// merged ModDown + rescale): the INTT storer pre-scales the sources, the
// first-pass loader of the following NTT evaluates the conversion sum.
#pragma once
#include "ks.cuh"
#include <cstdlib>

// Built, residue-exact (the whole -m gpu suite passes with it), but measured
// slower than the separate conversion kernels (5.99 vs 4.74 ms per Paper-mini
// step: the per-element conversion in the strided first-pass loader
// serialises its source loads); compiled only with -DHELR_FUSE_CONV_BUILD=1
// and then enabled by HELR_FUSE_CONV=1.
#ifndef HELR_FUSE_CONV_BUILD
#define HELR_FUSE_CONV_BUILD 0
#endif

// ---- basis conversions fused into the NTT passes ----------------------------
// A fast basis conversion y -> sum_k [y_k * w_k]_{s_k} * h_k (mod t) has a
// per-source pre-scaling and a per-target sum.  The pre-scaling is applied by
// the storer of the INTT that produces the sources (StScale), the sum by the
// loader of the first pass of the NTT that consumes the targets (LdModUp /
// LdModDown / LdMdr), so no conversion kernel and no round trip of the
// converted limbs through memory remain.  Values and order of
// operations are those of the former k_modup / k_moddown_conv / k_mdr_conv,
// so every residue is unchanged.
#define HELR_FUSE_MAXD 8
static inline bool fuse_conv_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("HELR_FUSE_CONV");
        on = e ? (atoi(e) != 0) : 0;
    }
    return on != 0;
}

// INTT storer: out = x * w_li mod q (canonical); fp64 limbs as exact doubles
// (the pass runs with dbl_out, so v already is one), integer limbs as u64.
struct StScale {
    u64* base;
    long long item_stride;
    int n;
    LimbMap map;
    const u64* tab;                 // d_tab
    int woff[HELR_MAXLIMBS];        // word offset of w_li in tab
    int wsoff[HELR_MAXLIMBS];       // word offset of its Shoup quotient
    const u64* q;
    const double* qd;
    const double* qinvd;
    __device__ __forceinline__ void operator()(int z, int li, int prime, int off, u64 v) const {
        const u64 qq = q[prime];
        u64 r;
        if (qq < NTT_DBL_BOUND) {
            const DblC dc{qd[prime], qinvd[prime]};
            r = (u64)__double_as_longlong(d2d_canon(mulmod_d(__longlong_as_double((long long)v), u2d(tab[woff[li]]), dc), dc));
        } else {
            r = shoup(v, tab[woff[li]], tab[wsoff[li]], qq);
        }
        base[(size_t)z * item_stride + (size_t)map.off[li] * n + off] = r;
    }
};

// INTT loader that also writes the digit's own limbs of the ModUp output:
// the (optionally Galois-permuted) NTT-form input itself, as exact doubles
// for fp64 primes.  li = limb p of the input.
struct LdCopyOwn {
    static constexpr bool kVec = true;
    static constexpr bool kTile = true;
    const u64* d;
    long long d_stride;
    u64* ext;
    long long ext_item_stride, ext_digit_stride;
    int n, alpha;
    unsigned long long dblmask;  // bit p: prime p < 2^41
    __device__ __forceinline__ u64 conv(int p, u64 v) const {
        return ((dblmask >> p) & 1ull) ? (u64)__double_as_longlong(u2d(v)) : v;
    }
    __device__ __forceinline__ u64* dst(int z, int p) const {
        return ext + (size_t)z * ext_item_stride + (size_t)(p / alpha) * ext_digit_stride + (size_t)p * n;
    }
    __device__ __forceinline__ u64 operator()(int z, int li, int, int off) const {
        const u64 v = d[(size_t)z * d_stride + (size_t)li * n + off];
        dst(z, li)[off] = conv(li, v);
        return v;
    }
    __device__ __forceinline__ ulonglong2 load2(int z, int li, int, int off) const {
        const ulonglong2 v = ld2(d + (size_t)z * d_stride + (size_t)li * n + off);
        st2(dst(z, li) + off, conv(li, v.x), conv(li, v.y));
        return v;
    }
};
struct LdPermCopyOwn {
    const u64* d;
    long long d_stride;
    u64* ext;
    long long ext_item_stride, ext_digit_stride;
    int n, log_n, alpha;
    u64 g;
    unsigned long long dblmask;
    __device__ __forceinline__ u64 operator()(int z, int li, int, int off) const {
        const u64 v = d[(size_t)z * d_stride + (size_t)li * n + galois_perm(off, g, log_n)];
        ext[(size_t)z * ext_item_stride + (size_t)(li / alpha) * ext_digit_stride + (size_t)li * n + off] =
            ((dblmask >> li) & 1ull) ? (u64)__double_as_longlong(u2d(v)) : v;
        return v;
    }
};

// First-pass loader of the ModUp NTT: target limb (digit j, target index t)
// = sum_k y_k * hm[k][t] over the digit's ns pre-scaled sources y_k (coef
// buffer: exact doubles for fp64 primes, u64 otherwise).
struct LdModUp {
    const u64* coef;
    long long coef_stride;
    int n;
    const u64* tab;
    int hm_off[HELR_FUSE_MAXD];     // word offset of hm for digit j
    unsigned char lo[HELR_FUSE_MAXD], ns[HELR_FUSE_MAXD], nt[HELR_FUSE_MAXD];
    unsigned char jj[HELR_MAXLIMBS], tt[HELR_MAXLIMBS];
    unsigned long long dblmask;
    const u64* q;
    const double* qd;
    const double* qinvd;
    __device__ __forceinline__ u64 operator()(int z, int li, int prime, int off) const {
        const int j = jj[li], t = tt[li], n_s = ns[j], n_t = nt[j], l0 = lo[j];
        const u64* hm = tab + hm_off[j];
        const u64* hms = hm + (size_t)n_s * n_t;
        const u64* src = coef + (size_t)z * coef_stride + (size_t)l0 * n + off;
        const u64 qq = q[prime];
        if (qq < NTT_DBL_BOUND) {
            const DblC dc{qd[prime], qinvd[prime]};
            double s = 0.0;
            for (int k = 0; k < n_s; k++) {
                const u64 y = src[(size_t)k * n];
                const u64 w = hm[(size_t)k * n_t + t];
                if ((dblmask >> (l0 + k)) & 1ull) s = __dadd_rn(s, mulmod_d(__longlong_as_double((long long)y), u2d(w), dc));
                else s = __dadd_rn(s, u2d(shoup(y, w, hms[(size_t)k * n_t + t], qq)));
            }
            return (u64)__double_as_longlong(reduce_d(s, dc));  // raw signed double (in_raw)
        }
        u64 s = 0;
        for (int k = 0; k < n_s; k++) {
            u64 y = src[(size_t)k * n];
            if ((dblmask >> (l0 + k)) & 1ull) y = dexact(__longlong_as_double((long long)y));
            s = add_mod(s, shoup(y, hm[(size_t)k * n_t + t], hms[(size_t)k * n_t + t], qq), qq);
        }
        return s;
    }
};

// First-pass loader of the ModDown NTT (centred P -> Q_l conversion of
// k_moddown_conv): li = poly * nl + p; sources z_k = the pre-scaled special
// limbs of acc (exact doubles when p_k < 2^41).
struct LdModDown {
    const u64* acc;
    long long acc_item_stride;
    int n, nl, K, L;
    const u64* phm;
    const u64* phms;
    const u64* pinv_dbl;
    const u64* pm;
    const u64* pm_sh;
    const u64* q;
    const double* qd;
    const double* qinvd;
    __device__ __forceinline__ u64 operator()(int z, int li, int prime, int off) const {
        const int poly = li >= nl ? 1 : 0, p = li - poly * nl, ne = nl + K;
        const u64* src = acc + (size_t)z * acc_item_stride + ((size_t)poly * ne + nl) * n + off;
        double v = 0.0;
        bool dsrc = true;
        for (int k = 0; k < K; k++) {
            const u64 x = src[(size_t)k * n];
            const bool dk = q[L + k] < NTT_DBL_BOUND;
            dsrc = dsrc && dk;
            const double d = dk ? __longlong_as_double((long long)x) : __ull2double_rn(x);
            v = __dadd_rn(v, __dmul_rn(d, __longlong_as_double((long long)pinv_dbl[k])));
        }
        const u64 rr = (u64)__double2ull_rd(__dadd_rn(v, 0.5));
        const u64 qq = q[prime];
        if (dsrc && qq < NTT_DBL_BOUND) {
            const DblC dc{qd[prime], qinvd[prime]};
            double s = -__dmul_rn(u2d(rr), u2d(pm[p]));
            for (int k = 0; k < K; k++)
                s = __dadd_rn(s, mulmod_d(__longlong_as_double((long long)src[(size_t)k * n]), u2d(phm[(size_t)k * L + p]), dc));
            return (u64)__double_as_longlong(reduce_d(s, dc));
        }
        u64 s = 0;
        for (int k = 0; k < K; k++) {
            u64 zk = src[(size_t)k * n];
            if (q[L + k] < NTT_DBL_BOUND) zk = dexact(__longlong_as_double((long long)zk));
            s = add_mod(s, shoup(zk, phm[(size_t)k * L + p], phms[(size_t)k * L + p], qq), qq);
        }
        return sub_mod(s, shoup(rr, pm[p], pm_sh[p], qq), qq);
    }
};

struct MrTab {
    const u64 *hv, *hvs, *hm, *hms, *mm, *mms, *mi, *mis, *dinv;
};
static inline MrTab mr_tab(const helr_ctx* c, int level) {
    const int ns = c->K + 1, L = c->L;
    const u64* e = c->d_tab + c->mr_off[level];
    MrTab t;
    t.hv = e; t.hvs = e + ns; t.hm = t.hvs + ns; t.hms = t.hm + (size_t)ns * L; t.mm = t.hms + (size_t)ns * L;
    t.mms = t.mm + L; t.mi = t.mms + L; t.mis = t.mi + L; t.dinv = t.mis + L;
    return t;
}

// First-pass loader of the merged ModDown + rescale NTT (k_mdr_conv):
// sources {p_0..p_{K-1}, q_l} (pre-scaled by the INTT), targets q_0..q_{l-1};
// li = poly * l + p.
struct LdMdr {
    const u64* acc;
    long long acc_item_stride;
    int n, nl, K, L;
    const u64* hm;    // [K+1][L]
    const u64* hms;
    const u64* mm;    // [L] M mod q_i
    const u64* mms;
    const u64* dinv;  // [K+1] 1/m_k (double bits)
    const u64* q;
    const double* qd;
    const double* qinvd;
    __device__ __forceinline__ u64 operator()(int z, int li, int prime, int off) const {
        const int l = nl - 1, ns = K + 1;
        const int poly = li >= l ? 1 : 0, p = li - poly * l, ne = nl + K;
        const u64* ap = acc + (size_t)z * acc_item_stride + (size_t)poly * ne * n + off;
        double v = 0.0;
        bool dsrc = true;
        for (int k = 0; k < ns; k++) {
            const int lim = k < K ? nl + k : l;
            const u64 x = ap[(size_t)lim * n];
            const bool dk = q[k < K ? L + k : l] < NTT_DBL_BOUND;
            dsrc = dsrc && dk;
            const double d = dk ? __longlong_as_double((long long)x) : __ull2double_rn(x);
            v = __dadd_rn(v, __dmul_rn(d, __longlong_as_double((long long)dinv[k])));
        }
        const u64 rr = (u64)__double2ull_rd(__dadd_rn(v, 0.5));
        const u64 qq = q[prime];
        if (dsrc && qq < NTT_DBL_BOUND) {
            const DblC dc{qd[prime], qinvd[prime]};
            double s = -__dmul_rn(u2d(rr), u2d(mm[p]));
            for (int k = 0; k < ns; k++) {
                const int lim = k < K ? nl + k : l;
                s = __dadd_rn(s, mulmod_d(__longlong_as_double((long long)ap[(size_t)lim * n]), u2d(hm[(size_t)k * L + p]), dc));
            }
            return (u64)__double_as_longlong(reduce_d(s, dc));
        }
        u64 s = 0;
        for (int k = 0; k < ns; k++) {
            const int lim = k < K ? nl + k : l;
            u64 zk = ap[(size_t)lim * n];
            if (q[k < K ? L + k : l] < NTT_DBL_BOUND) zk = dexact(__longlong_as_double((long long)zk));
            s = add_mod(s, shoup(zk, hm[(size_t)k * L + p], hms[(size_t)k * L + p], qq), qq);
        }
        return sub_mod(s, shoup(rr, mm[p], mms[p], qq), qq);
    }
};

static inline unsigned long long dbl_mask(const helr_ctx* c) {
    unsigned long long m = 0;
    for (int p = 0; p < (int)c->primes.size() && p < 64; p++)
        if (c->primes[p] < NTT_DBL_BOUND) m |= 1ull << p;
    return m;
}
static inline StScale st_scale(const helr_ctx* c, u64* base, long long is, const LimbMap& map) {
    StScale st;
    st.base = base; st.item_stride = is; st.n = c->n; st.map = map; st.tab = c->d_tab;
    st.q = c->t.q; st.qd = c->t.qd; st.qinvd = c->t.qinvd;
    for (int i = 0; i < HELR_MAXLIMBS; i++) st.woff[i] = st.wsoff[i] = 0;
    return st;
}

