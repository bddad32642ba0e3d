// ks.cuh — pieces shared by the evaluator (ops.cu) and the key inner-product
// kernels (hoist.cu): launch-check macros, index helpers, 64 / 128-bit and
// fp64 multiply-accumulate helpers, the key-switching workspace layout.
#pragma once
#include <cuda_runtime.h>

#include "../../include/helr_ckks.h"
#include "ntt.cuh"
#include "ops_internal.cuh"
#include "prof.cuh"

#define CHECK_LAUNCH(what)                                              \
    do {                                                                \
        if (!cuda_ok(cudaGetLastError(), what)) return HELR_ECUDA;      \
    } while (0)
// one non-NTT kernel launched (NTT passes count themselves in ntt.cuh)
#define CHECK_KERNEL(what)                                              \
    do {                                                                \
        count_launches(1);                                              \
        if (!cuda_ok(cudaGetLastError(), what)) return HELR_ECUDA;      \
    } while (0)

static inline cudaStream_t S(void* s) { return (cudaStream_t)s; }
static inline int blocks_for(long long n, int t) { return (int)((n + t - 1) / t); }

__device__ __forceinline__ int brv_dev(int x, int log_n) { return (int)(__brev((unsigned)x) >> (32 - log_n)); }
__device__ __forceinline__ ulonglong2 ld2(const u64* p) { return *reinterpret_cast<const ulonglong2*>(p); }
__device__ __forceinline__ void st2(u64* p, u64 x, u64 y) { *reinterpret_cast<ulonglong2*>(p) = make_ulonglong2(x, y); }
// NTT-slot permutation of X -> X^g: out[i] = in[perm(i)]
// (2N is a power of two <= 2^17, so the product is needed only mod 2^32:
// 32-bit arithmetic, one IMAD)
__device__ __forceinline__ int galois_perm_e(unsigned e, u64 g, int log_n) {  // e = 2 brv(i) + 1
    const unsigned f = (e * (unsigned)g) & ((2u << log_n) - 1u);
    return brv_dev((int)((f - 1u) >> 1), log_n);
}
__device__ __forceinline__ int galois_perm(int i, u64 g, int log_n) {
    return galois_perm_e(2u * (unsigned)brv_dev(i, log_n) + 1u, g, log_n);
}


struct u128acc { u64 lo, hi; };
// Split accumulator for a sum of 64x64-bit products: lo + hi 2^64 holds
// sum x0 y0 + x1 y1 2^64, mid (+ carries 2^64) holds sum x0 y1 + x1 y0, so each
// product costs four 32x32->64 multiply-adds with carry (aligned register
// pairs, no shuffling) plus one carry count; resolved once per output.
struct macc { u64 lo, hi, mid; u32 mc; };
__device__ __forceinline__ void mac_split(macc& a, u64 x, u64 y) {
    asm("{\n\t"
        ".reg .u32 x0, x1, y0, y1, a0, a1, a2, a3, m0, m1;\n\t"
        "mov.b64 {x0, x1}, %4;\n\t"
        "mov.b64 {y0, y1}, %5;\n\t"
        "mov.b64 {a0, a1}, %0;\n\t"
        "mov.b64 {a2, a3}, %1;\n\t"
        "mov.b64 {m0, m1}, %2;\n\t"
        "mad.lo.cc.u32 a0, x0, y0, a0;\n\t"
        "madc.hi.cc.u32 a1, x0, y0, a1;\n\t"
        "madc.lo.cc.u32 a2, x1, y1, a2;\n\t"
        "madc.hi.u32 a3, x1, y1, a3;\n\t"
        "mad.lo.cc.u32 m0, x0, y1, m0;\n\t"
        "madc.hi.cc.u32 m1, x0, y1, m1;\n\t"
        "addc.u32 %3, %3, 0;\n\t"
        "mad.lo.cc.u32 m0, x1, y0, m0;\n\t"
        "madc.hi.cc.u32 m1, x1, y0, m1;\n\t"
        "addc.u32 %3, %3, 0;\n\t"
        "mov.b64 %0, {a0, a1};\n\t"
        "mov.b64 %1, {a2, a3};\n\t"
        "mov.b64 %2, {m0, m1};\n\t"
        "}"
        : "+l"(a.lo), "+l"(a.hi), "+l"(a.mid), "+r"(a.mc)
        : "l"(x), "l"(y));
}
// lo + hi 2^64 + (mid + mc 2^64) 2^32 as a 128-bit value (< 2^128 by the fold bound)
__device__ __forceinline__ u128acc resolve(const macc& a) {
    u128acc r{a.lo, a.hi};
    const u64 add_lo = a.mid << 32;
    const u64 add_hi = (a.mid >> 32) | ((u64)a.mc << 32);
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(r.lo), "+l"(r.hi) : "l"(add_lo), "l"(add_hi));
    return r;
}
__device__ __forceinline__ u64 reduce128(const u128acc& a, u64 q, u64 r1, u64 r0, u64 one_sh) {
    return barrett128(u128v{shoup(a.hi, 1, one_sh, q), a.lo}, q, r1, r0);
}

// fp64 multiply-accumulate for limbs whose prime is below 2^41: operands are
// split at bit 21 into exact doubles (< 2^21), the four partial products
// (< 2^42) accumulate exactly in three doubles for up to 2^11 terms (every
// hoisted group has at most 31 * 8), and the sum is reassembled as a 128-bit
// integer once per output.  DFMA issues at 2.5x the IMAD.WIDE rate on a pipe
// the integer path leaves idle.
struct dacc { double hh, mid, ll; };
__device__ __forceinline__ void split21(u64 x, double& h, double& l) {
    h = u2d(x >> 21);
    l = u2d(x & 0x1FFFFFull);
}
__device__ __forceinline__ void mac_d(dacc& a, double xh, double xl, double yh, double yl) {
    a.hh = __fma_rn(xh, yh, a.hh);
    a.mid = __fma_rn(xh, yl, a.mid);
    a.mid = __fma_rn(xl, yh, a.mid);
    a.ll = __fma_rn(xl, yl, a.ll);
}
__device__ __forceinline__ u64 dexact(double x) {  // integer-valued 0 <= x < 2^52
    return (u64)__double_as_longlong(__dadd_rn(x, NTT_TWO52)) & 0x000FFFFFFFFFFFFFull;
}
// ModUp'd digits of fp64 limbs are stored as exact doubles (ks_modup):
// split x = h 2^21 + l with h = rint(x / 2^21) in [0, 2^20] and signed
// l in [-2^20, 2^20] on the fp64 pipe (no integer shifts or masks).  The
// partial products stay below 2^41 in magnitude; mid / ll may be negative.
__device__ __forceinline__ void split21_d(double x, double& h, double& l) {
    h = drint_mul(x, 4.76837158203125e-07);  // 2^-21
    l = __fma_rn(-h, 2097152.0, x);
}
__device__ __forceinline__ long long dexact_s(double x) {  // integer-valued |x| < 2^51
    return __double_as_longlong(__dadd_rn(x, NTT_MAGIC)) - 0x4338000000000000ll;
}
// hh 2^42 + mid 2^21 + ll with signed mid, ll (the total is non-negative)
__device__ __forceinline__ u128acc dresolve_s(const dacc& a) {
    const u64 H = dexact(a.hh);
    const long long M = dexact_s(a.mid), Lo = dexact_s(a.ll);
    u128acc r{H << 42, H >> 22};
    const u64 m_lo = (u64)M << 21, m_hi = (u64)(M >> 43);
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(r.lo), "+l"(r.hi) : "l"(m_lo), "l"(m_hi));
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(r.lo), "+l"(r.hi) : "l"((u64)Lo), "l"((u64)(Lo >> 63)));
    return r;
}
__device__ __forceinline__ u128acc dresolve(const dacc& a) {  // hh 2^42 + mid 2^21 + ll
    const u64 H = dexact(a.hh), M = dexact(a.mid), Lo = dexact(a.ll);
    u128acc r{H << 42, H >> 22};
    const u64 m_lo = M << 21, m_hi = M >> 43;
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(r.lo), "+l"(r.hi) : "l"(m_lo), "l"(m_hi));
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, 0;" : "+l"(r.lo), "+l"(r.hi) : "l"(Lo));
    return r;
}


// Last-NTT-pass storer that finishes a ModDown / rescale in place of a
// separate combine kernel: out = (x - v) * w_p mod q [+ add_a] [+ sum_t
// sigma_t(add_p) on poly 0], v being the NTT output.  Index decoding:
// per_poly > 0: item = z, li = poly * per_poly + p;  per_poly == 0:
// item = z >> 1, poly = z & 1, p = li.
struct StCombine {
    static constexpr bool kVec = true;
    static constexpr bool kTile = true;
    // fp64 limbs hand the storer the pass's raw doubles (integer-valued, any
    // representative, |v| < 2^46): the combine runs on the fp64 pipe — one
    // exact twiddle-style product and ONE canonicalisation for the whole
    // (x - v) w + addend + sigma-sum — instead of canonicalising v and then
    // doing a 64-bit integer Shoup product
    static constexpr bool kRawD = true;
    // per-thread context of one (item, limb): decoded once per pass, not per pair
    struct Ctx {
        const u64* xb;
        const u64* ab;
        const u64* pb;
        u64* ob;
        u64 qq, wp, wps;
        double wd;
        DblC dc;
        bool dbl;
    };
    u64* out;
    long long out_is, out_ps;
    const u64* x;
    long long x_is, x_ps;
    const u64* w;
    const u64* wsh;
    const u64* q;
    const double* qd;     // q and 1/q as doubles (primes below 2^41: lazy sigma sums)
    const double* qinvd;
    const u64* add_a;
    long long a_is, a_ps;
    const u64* add_p;
    long long p_is;
    int ngal, log_n, n, per_poly;
    long long gal[HELR_MAX_HOIST];
    __device__ __forceinline__ void decode(int z, int li, int& item, int& poly, int& p) const {
        if (per_poly > 0) { item = z; poly = li >= per_poly ? 1 : 0; p = li - poly * per_poly; }
        else { item = z >> 1; poly = z & 1; p = li; }
    }
    __device__ __forceinline__ u64 addends(u64 r, int item, int poly, int p, int off, u64 qq, u64 av) const {
        if (add_a) r = add_mod(r, av, qq);
        if (add_p && poly == 0) {
            const u64* pp = add_p + (size_t)item * p_is + (size_t)p * n;
            for (int t = 0; t < ngal; t++) r = add_mod(r, pp[galois_perm(off, (u64)gal[t], log_n)], qq);
        }
        return r;
    }
    __device__ __forceinline__ void operator()(int z, int li, int, int off, u64 v) const {
        int item, poly, p;
        decode(z, li, item, poly, p);
        const u64 qq = q[p];
        const u64 xv = x[(size_t)item * x_is + (size_t)poly * x_ps + (size_t)p * n + off];
        u64 r = shoup(sub_mod(xv, v, qq), w[p], wsh[p], qq);
        const u64 av = add_a ? add_a[(size_t)item * a_is + (size_t)poly * a_ps + (size_t)p * n + off] : 0;
        out[(size_t)item * out_is + (size_t)poly * out_ps + (size_t)p * n + off] = addends(r, item, poly, p, off, qq, av);
    }
    __device__ __forceinline__ Ctx prep(int z, int li) const {
        int item, poly, p;
        decode(z, li, item, poly, p);
        Ctx c;
        c.qq = q[p]; c.wp = w[p]; c.wps = wsh[p];
        c.dbl = c.qq < NTT_DBL_BOUND;
        c.dc = DblC{qd[p], qinvd[p]};
        c.wd = u2d(c.wp & 0x000FFFFFFFFFFFFFull);  // used only when dbl (w < q < 2^41)
        c.xb = x + (size_t)item * x_is + (size_t)poly * x_ps + (size_t)p * n;
        c.ab = add_a ? add_a + (size_t)item * a_is + (size_t)poly * a_ps + (size_t)p * n : nullptr;
        c.pb = (add_p && poly == 0) ? add_p + (size_t)item * p_is + (size_t)p * n : nullptr;
        c.ob = out + (size_t)item * out_is + (size_t)poly * out_ps + (size_t)p * n;
        return c;
    }
    // v: fp64 limbs -> raw double bits (kRawD), integer limbs -> canonical u64
    __device__ __forceinline__ void store2c(const Ctx& c, int off, ulonglong2 v) const {
        const ulonglong2 xv = ld2(c.xb + off);
        if (c.dbl) {
            double r0 = mulmod_d(__dsub_rn(u2d(xv.x), __longlong_as_double((long long)v.x)), c.wd, c.dc);
            double r1 = mulmod_d(__dsub_rn(u2d(xv.y), __longlong_as_double((long long)v.y)), c.wd, c.dc);
            if (c.ab) {
                const ulonglong2 av = ld2(c.ab + off);
                r0 = __dadd_rn(r0, u2d(av.x));
                r1 = __dadd_rn(r1, u2d(av.y));
            }
            if (c.pb) {
                // plain 64-bit sums of the <= 2^11 gathered residues (< 2^52), added as exact doubles
                const unsigned eo = 2u * (unsigned)brv_dev(off, log_n) + 1u;
                u64 s0 = 0, s1 = 0;
                for (int t = 0; t < ngal; t++) {
                    const int src = galois_perm_e(eo, (u64)gal[t], log_n);
                    const ulonglong2 pr = ld2(c.pb + (src & ~1));
                    s0 += (src & 1) ? pr.y : pr.x;
                    s1 += (src & 1) ? pr.x : pr.y;
                }
                r0 = __dadd_rn(r0, u2d(s0));
                r1 = __dadd_rn(r1, u2d(s1));
            }
            st2(c.ob + off, d2u_canon(r0, c.dc), d2u_canon(r1, c.dc));
            return;
        }
        const u64 qq = c.qq;
        u64 r0 = shoup(sub_mod(xv.x, v.x, qq), c.wp, c.wps, qq);
        u64 r1 = shoup(sub_mod(xv.y, v.y, qq), c.wp, c.wps, qq);
        if (c.ab) {
            const ulonglong2 av = ld2(c.ab + off);
            r0 = add_mod(r0, av.x, qq);
            r1 = add_mod(r1, av.y, qq);
        }
        if (c.pb) {
            const unsigned eo = 2u * (unsigned)brv_dev(off, log_n) + 1u;
            for (int t = 0; t < ngal; t++) {
                const int src = galois_perm_e(eo, (u64)gal[t], log_n);
                const ulonglong2 pr = ld2(c.pb + (src & ~1));
                r0 = add_mod(r0, (src & 1) ? pr.y : pr.x, qq);
                r1 = add_mod(r1, (src & 1) ? pr.x : pr.y, qq);
            }
        }
        st2(c.ob + off, r0, r1);
    }
    // single element (passes whose last register group is strided)
    __device__ __forceinline__ void store1c(const Ctx& c, int off, u64 v) const {
        const u64 xv = c.xb[off];
        if (c.dbl) {
            double r = mulmod_d(__dsub_rn(u2d(xv), __longlong_as_double((long long)v)), c.wd, c.dc);
            if (c.ab) r = __dadd_rn(r, u2d(c.ab[off]));
            if (c.pb) {
                u64 s0 = 0;
                for (int t = 0; t < ngal; t++) s0 += c.pb[galois_perm(off, (u64)gal[t], log_n)];
                r = __dadd_rn(r, u2d(s0));
            }
            c.ob[off] = d2u_canon(r, c.dc);
            return;
        }
        u64 r = shoup(sub_mod(xv, v, c.qq), c.wp, c.wps, c.qq);
        if (c.ab) r = add_mod(r, c.ab[off], c.qq);
        if (c.pb)
            for (int t = 0; t < ngal; t++) r = add_mod(r, c.pb[galois_perm(off, (u64)gal[t], log_n)], c.qq);
        c.ob[off] = r;
    }
    __device__ __forceinline__ void store2(int z, int li, int, int off, ulonglong2 v) const {
        int item, poly, p;
        decode(z, li, item, poly, p);
        const u64 qq = q[p], wp = w[p], wps = wsh[p];
        const ulonglong2 xv = ld2(x + (size_t)item * x_is + (size_t)poly * x_ps + (size_t)p * n + off);
        ulonglong2 av = make_ulonglong2(0, 0);
        if (add_a) av = ld2(add_a + (size_t)item * a_is + (size_t)poly * a_ps + (size_t)p * n + off);
        u64 r0 = shoup(sub_mod(xv.x, v.x, qq), wp, wps, qq);
        u64 r1 = shoup(sub_mod(xv.y, v.y, qq), wp, wps, qq);
        if (add_a) { r0 = add_mod(r0, av.x, qq); r1 = add_mod(r1, av.y, qq); }
        if (add_p && poly == 0) {
            // off is even, and a Galois permutation maps the pair (off, off + 1)
            // onto the aligned pair (s, s ^ 1): one index and one 16-byte load per step
            const u64* pp = add_p + (size_t)item * p_is + (size_t)p * n;
            const unsigned eo = 2u * (unsigned)brv_dev(off, log_n) + 1u;
            if (qq < NTT_DBL_BOUND) {
                // primes below 2^41: plain 64-bit sums of the <= 2^11 gathered
                // residues (< 2^52), one exact fp64 reduction at the end
                for (int t = 0; t < ngal; t++) {
                    const int src = galois_perm_e(eo, (u64)gal[t], log_n);
                    const ulonglong2 pr = ld2(pp + (src & ~1));
                    r0 += (src & 1) ? pr.y : pr.x;
                    r1 += (src & 1) ? pr.x : pr.y;
                }
                const DblC dc{qd[p], qinvd[p]};
                r0 = d2u_canon(u2d(r0), dc);
                r1 = d2u_canon(u2d(r1), dc);
            } else {
                for (int t = 0; t < ngal; t++) {
                    const int src = galois_perm_e(eo, (u64)gal[t], log_n);
                    const ulonglong2 pr = ld2(pp + (src & ~1));
                    r0 = add_mod(r0, (src & 1) ? pr.y : pr.x, qq);
                    r1 = add_mod(r1, (src & 1) ? pr.x : pr.y, qq);
                }
            }
        }
        st2(out + (size_t)item * out_is + (size_t)poly * out_ps + (size_t)p * n + off, r0, r1);
    }
};
// byte model of a StCombine last pass: per output limb the ModDown input x,
// the optional addend, and (poly 0 only) the sigma-gathered c0 limb, each once
inline double ntt_extra_words(const StCombine& st, const LimbMap& m, int count) {
    double poly0 = 0.0;
    if (st.per_poly > 0) poly0 = (double)(m.count < st.per_poly ? m.count : st.per_poly) * count;
    else poly0 = (double)m.count * (count / 2.0);
    return (double)m.count * count * (1.0 + (st.add_a ? 1.0 : 0.0)) + (st.add_p ? poly0 : 0.0);
}
static inline StCombine st_combine(const helr_ctx* c, u64* out, long long out_is, long long out_ps, const u64* x, long long x_is,
                            long long x_ps, const u64* w, const u64* wsh, int per_poly) {
    StCombine f;
    f.out = out; f.out_is = out_is; f.out_ps = out_ps;
    f.x = x; f.x_is = x_is; f.x_ps = x_ps;
    f.w = w; f.wsh = wsh; f.q = c->t.q; f.qd = c->t.qd; f.qinvd = c->t.qinvd;
    f.add_a = nullptr; f.a_is = f.a_ps = 0;
    f.add_p = nullptr; f.p_is = 0;
    f.ngal = 0; f.log_n = c->log_n; f.n = c->n; f.per_poly = per_poly;
    for (int t = 0; t < HELR_MAX_HOIST; t++) f.gal[t] = 1;
    return f;
}

// workspace carve-up for key switching of B items at level l
struct KsWs {
    u64 *coef, *ext, *acc, *mdc, *tensor;
    long long coef_s, ext_s, ext_ds, acc_s, mdc_s;
};
static inline KsWs ks_ws(helr_ctx* c, int B) {
    KsWs w;
    const size_t n = c->n;
    w.coef_s = (long long)c->L * n;
    w.ext_ds = (long long)c->LK * n;
    w.ext_s = (long long)c->beta * w.ext_ds;
    w.acc_s = 2ll * c->LK * n;
    w.mdc_s = 2ll * c->L * n;
    w.coef = c->ws;
    w.ext = w.coef + (size_t)B * w.coef_s;
    w.acc = w.ext + (size_t)B * w.ext_s;
    w.mdc = w.acc + (size_t)B * w.acc_s;
    w.tensor = w.mdc + (size_t)B * w.mdc_s;
    return w;
}

struct HoistKeys {
    int nsteps;
    const u64* key[HELR_MAX_HOIST];
    long long gal[HELR_MAX_HOIST];
};

// key inner product of the ModUp'd digits in w.ext with hk's keys, summed
// over hk.nsteps Galois steps, into w.acc (hoist.cu); dadd (optional) adds
// (P mod q) * (d0, d1) of a [B][3][L][N] tensor to the Q limbs
int key_inner(helr_ctx* c, const KsWs& w, const HoistKeys& hk, int nb, int level, const u64* dadd, long long dadd_is,
              cudaStream_t s);

// ---- key-switching stages shared by ks.cu / ks_modup.cu / ks_moddown.cu
struct KsInput {
    const u64* d;        // NTT-form polynomial of item b at d + b*d_stride, limb stride N
    long long d_stride;
    long long galois;    // 0: none, else apply X -> X^galois to d first
};
struct KsEpilogue {
    u64* out;             // ciphertext of item b at out + b*out_stride
    long long out_stride;
    const u64* add_a;     // optional ciphertext-like addend (both polys), stride add_a_stride
    long long add_a_stride;
    const u64* add_p;     // optional: sum_t sigma_t(poly 0 of add_p) added to out poly 0
    long long add_p_stride;
    int ngal;
    long long gal[HELR_MAX_HOIST];
};
static inline KsEpilogue make_epilogue(u64* out, long long os, const u64* add_a, long long as, const u64* add_p, long long ps,
                                int ngal, const long long* gal) {
    KsEpilogue e;
    e.out = out; e.out_stride = os; e.add_a = add_a; e.add_a_stride = as; e.add_p = add_p; e.add_p_stride = ps;
    e.ngal = ngal;
    for (int t = 0; t < HELR_MAX_HOIST; t++) e.gal[t] = t < ngal ? gal[t] : 0;
    return e;
}

int ks_modup(helr_ctx* c, KsInput in, int level, int B, const KsWs& w, cudaStream_t s);
int ks_moddown(helr_ctx* c, int level, const KsEpilogue& ep, int B, const KsWs& w, cudaStream_t s);
int ks_moddown_rescale(helr_ctx* c, int level, u64* out, long long os, int B, const KsWs& w, cudaStream_t s);
