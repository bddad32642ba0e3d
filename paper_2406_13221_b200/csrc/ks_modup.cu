// ks_modup.cu — ModUp of key switching: INTT, basis conversion Q_l -> Q_l + P
// per digit, NTT (fused conversion by default, k_modup kept behind HELR_FUSE_CONV=0).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "conv.cuh"

// ModUp conversion for digit j; grid (x: coeff tiles, y: digit, z: item)
struct ModUpArgs {
    const u64* coef;   // [B][nl][N] INTT of d
    long long coef_stride;
    const u64* d;      // NTT-form input (own-digit limbs are copied from here)
    long long d_stride;
    long long galois;
    u64* ext;          // [B][beta][ext][N]
    long long ext_item_stride, ext_digit_stride;
    const u64* tab;    // d_tab
    const size_t* offs;// device array of modup offsets for this level (per digit)
    int n, log_n, nl, K, L, alpha;
};
// Two consecutive coefficients per thread, 16-byte accesses; register
// arrays bounded by the template parameter (alpha / K <= MA).

template <int MA>
__global__ void k_modup(ModUpArgs a, Tables tb) {
    pdl_begin();
    const int j = blockIdx.y, b = blockIdx.z;
    const int lo = j * a.alpha, hi = lo + a.alpha < a.nl ? lo + a.alpha : a.nl;
    const int ns = hi - lo;
    const int ne = a.nl + a.K;
    const int nt = ne - ns;
    const u64* T = a.tab + a.offs[j];
    const u64* hv = T;
    const u64* hvs = T + ns;
    const u64* hm = T + 2 * ns;
    const u64* hms = hm + (size_t)ns * nt;
    u64* ext = a.ext + (size_t)b * a.ext_item_stride + (size_t)j * a.ext_digit_stride;
    const u64* coef = a.coef + (size_t)b * a.coef_stride;
    const u64* d = a.d + (size_t)b * a.d_stride;
    // the digit's ns x nt target weights as doubles, converted once per CTA
    // (shared-memory broadcast reads instead of a load + conversion per term)
    constexpr bool WSM = MA <= 8;
    __shared__ double wsm[WSM ? MA * HELR_MAXP : 1];
    if constexpr (WSM) {
        for (int e = threadIdx.x; e < ns * nt; e += blockDim.x) {
            const int k = e / nt, t = e - k * nt;
            wsm[k * HELR_MAXP + t] = u2d(hm[(size_t)k * nt + t] & 0x000FFFFFFFFFFFFFull);
        }
        __syncthreads();
    }
    const int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (i >= a.n) return;
    u64 y0[MA], y1[MA];
#pragma unroll
    for (int k = 0; k < MA; k++) {
        if (k < ns) {
            const int p = lo + k;
            const ulonglong2 c = ld2(coef + (size_t)p * a.n + i);
            y0[k] = shoup(c.x, hv[k], hvs[k], tb.q[p]);
            y1[k] = shoup(c.y, hv[k], hvs[k], tb.q[p]);
            // own-digit limbs: the NTT-form input itself (exact doubles for fp64 limbs)
            ulonglong2 v;
            if (a.galois) {
                const u64* dp = d + (size_t)p * a.n;
                v = make_ulonglong2(dp[galois_perm(i, (u64)a.galois, a.log_n)],
                                    dp[galois_perm(i + 1, (u64)a.galois, a.log_n)]);
            } else {
                v = ld2(d + (size_t)p * a.n + i);
            }
            if (tb.q[p] < NTT_DBL_BOUND)
                v = make_ulonglong2((u64)__double_as_longlong(u2d(v.x)), (u64)__double_as_longlong(u2d(v.y)));
            *reinterpret_cast<ulonglong2*>(ext + (size_t)p * a.n + i) = v;
        }
    }
    // source residues as exact doubles (primes < 2^41) for the fp64 targets
    double yd0[MA], yd1[MA];
    bool ydok[MA];
#pragma unroll
    for (int k = 0; k < MA; k++) {
        ydok[k] = k < ns && tb.q[lo + k] < NTT_DBL_BOUND;
        if (ydok[k]) { yd0[k] = u2d(y0[k]); yd1[k] = u2d(y1[k]); }
    }
    int t = 0;
    for (int e = 0; e < ne; e++) {
        if (e >= lo && e < hi) continue;
        const int p = e < a.nl ? e : a.L + (e - a.nl);
        const u64 q = tb.q[p];
        if (q < NTT_DBL_BOUND) {
            // fp64 target: exact signed products (mulmod_d), one reduction
            const DblC dc{tb.qd[p], tb.qinvd[p]};
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int k = 0; k < MA; k++) {
                if (k < ns) {
                    if (ydok[k]) {
                        const double wd = WSM ? wsm[k * HELR_MAXP + t] : u2d(hm[(size_t)k * nt + t]);
                        s0 = __dadd_rn(s0, mulmod_d(yd0[k], wd, dc));
                        s1 = __dadd_rn(s1, mulmod_d(yd1[k], wd, dc));
                    } else {  // wide source prime (q_0): integer Shoup, result < q
                        const u64 w = hm[(size_t)k * nt + t];
                        const u64 ws = hms[(size_t)k * nt + t];
                        s0 = __dadd_rn(s0, u2d(shoup(y0[k], w, ws, q)));
                        s1 = __dadd_rn(s1, u2d(shoup(y1[k], w, ws, q)));
                    }
                }
            }
            // raw signed double (|x| <= q/2 + 1): the NTT below reads it as is (in_raw)
            st2(ext + (size_t)e * a.n + i, (u64)__double_as_longlong(reduce_d(s0, dc)),
                (u64)__double_as_longlong(reduce_d(s1, dc)));
            t++;
            continue;
        }
        u64 s0 = 0, s1 = 0;
#pragma unroll
        for (int k = 0; k < MA; k++) {
            if (k < ns) {
                const u64 w = hm[(size_t)k * nt + t], ws = hms[(size_t)k * nt + t];
                s0 = add_mod(s0, shoup(y0[k], w, ws, q), q);
                s1 = add_mod(s1, shoup(y1[k], w, ws, q), q);
            }
        }
        st2(ext + (size_t)e * a.n + i, s0, s1);
        t++;
    }
}

// Loader applying the Galois permutation to a plain buffer (rotation input).
struct LdPerm {
    const u64* base;
    long long item_stride;
    int n, log_n;
    u64 g;
    __device__ __forceinline__ u64 operator()(int z, int li, int, int off) const {
        return base[(size_t)z * item_stride + (size_t)li * n + galois_perm(off, g, log_n)];
    }
};

#if HELR_FUSE_CONV_BUILD
static int ks_modup_fused(helr_ctx* c, KsInput in, int level, int B, const KsWs& w, cudaStream_t s);
#endif

// ModUp of B inputs into w.ext (NTT form over Q_l + P for every digit)
int ks_modup(helr_ctx* c, KsInput in, int level, int B, const KsWs& w, cudaStream_t s) {
    const int n = c->n, nl = level + 1, K = c->K, L = c->L, ne = nl + K;
    const int nd = (nl + c->alpha - 1) / c->alpha;
#if HELR_FUSE_CONV_BUILD
    if (fuse_conv_enabled() && nd <= HELR_FUSE_MAXD && c->LK <= 64) return ks_modup_fused(c, in, level, B, w, s);
#endif
    // 1) coef = INTT(sigma(d))
    {
        LimbMap m = limb_range(0, nl);
        StBuf st{w.coef, w.coef_s, m, n};
        if (in.galois) {
            LdPerm ld{in.d, in.d_stride, n, c->log_n, (u64)in.galois};
            ntt_launch<true>(c, ld, st, w.coef, w.coef_s, m, B, s);
        } else {
            LdBuf ld{in.d, in.d_stride, m, n};
            ntt_launch<true>(c, ld, st, w.coef, w.coef_s, m, B, s);
        }
        CHECK_LAUNCH("ks intt");
    }
    // 2) ModUp conversions (+ copy of own-digit NTT limbs)
    {
        ModUpArgs a{w.coef, w.coef_s, in.d, in.d_stride, in.galois, w.ext, w.ext_s, w.ext_ds, c->d_tab,
                    c->d_modup_offs + (size_t)level * c->beta, n, c->log_n, nl, K, L, c->alpha};
        dim3 g(blocks_for(n / 2, 128), nd, B);
        ProfScope ps(PROF_MODUP, 8.0 * n * B * (2.0 * nl + (double)nd * ne), s);
        if (c->alpha <= 4) launch_pdl(k_modup<4>, g, dim3(128), 0, s, a, c->t);
        else if (c->alpha <= 8) launch_pdl(k_modup<8>, g, dim3(128), 0, s, a, c->t);
        else if (c->alpha <= 16) launch_pdl(k_modup<16>, g, dim3(128), 0, s, a, c->t);
        else if (c->alpha <= 32) launch_pdl(k_modup<32>, g, dim3(128), 0, s, a, c->t);
        else launch_pdl(k_modup<HELR_MAXP>, g, dim3(128), 0, s, a, c->t);
        CHECK_KERNEL("ks modup");
    }
    // 3) NTT of every converted limb of every digit (one launch per 128 limbs)
    {
        LimbMap m;
        m.count = 0;
        for (int j = 0; j < nd; j++) {
            const int lo = j * c->alpha, hi = lo + c->alpha < nl ? lo + c->alpha : nl;
            for (int e = 0; e < ne; e++) {
                if (e >= lo && e < hi) continue;
                m.off[m.count] = (unsigned char)(j * c->LK + e);
                m.prime[m.count] = (unsigned char)(e < nl ? e : L + (e - nl));
                if (++m.count == HELR_MAXLIMBS) {
                    ntt_buffers<false>(c, w.ext, w.ext_s, w.ext, w.ext_s, m, B, s, 1, 1);
                    m.count = 0;
                }
            }
        }
        // fp64 limbs: raw doubles in, exact (canonical) doubles out — the inner
        // products split them on the fp64 pipe (split21_d).  Integer-path
        // limbs (q_0) first: the limb is the grid's slowest index, so the
        // slower CTAs start in the first waves.
        if (m.count) {
            LimbMap h;
            h.count = 0;
            for (int pass = 0; pass < 2; pass++)
                for (int i = 0; i < m.count; i++)
                    if ((c->primes[m.prime[i]] >= NTT_DBL_BOUND) == (pass == 0)) {
                        h.off[h.count] = m.off[i];
                        h.prime[h.count++] = m.prime[i];
                    }
            ntt_buffers<false>(c, w.ext, w.ext_s, w.ext, w.ext_s, h, B, s, 1, 1);
        }
        CHECK_LAUNCH("ks modup ntt");
    }
    return HELR_OK;
}

#if HELR_FUSE_CONV_BUILD
// Fused ModUp: INTT(sigma(d)) with the digit pre-scaling in its storer and
// the own-digit copy in its loader, then the NTT of every target limb whose
// first-pass loader evaluates the conversion (no k_modup).
static int ks_modup_fused(helr_ctx* c, KsInput in, int level, int B, const KsWs& w, cudaStream_t s) {
    const int n = c->n, nl = level + 1, K = c->K, L = c->L, ne = nl + K, al = c->alpha;
    const int nd = (nl + al - 1) / al;
    const unsigned long long dm = dbl_mask(c);
    // 1) coef = INTT(sigma(d)) * qhat_j^-1 (per digit), ext own limbs = sigma(d)
    {
        LimbMap m = limb_range(0, nl);
        StScale st = st_scale(c, w.coef, w.coef_s, m);
        for (int p = 0; p < nl; p++) {
            const int j = p / al;
            const size_t o = c->modup_off[(size_t)level * c->beta + j];
            const int ns = ((j * al + al < nl) ? j * al + al : nl) - j * al;
            st.woff[p] = (int)(o + (p - j * al));
            st.wsoff[p] = (int)(o + ns + (p - j * al));
        }
        if (in.galois) {
            LdPermCopyOwn ld{in.d, in.d_stride, w.ext, w.ext_s, w.ext_ds, n, c->log_n, al, (u64)in.galois, dm};
            ntt_launch<true>(c, ld, st, w.coef, w.coef_s, m, B, s, 0, 1);
        } else {
            LdCopyOwn ld{in.d, in.d_stride, w.ext, w.ext_s, w.ext_ds, n, al, dm};
            ntt_launch<true>(c, ld, st, w.coef, w.coef_s, m, B, s, 0, 1);
        }
        CHECK_LAUNCH("ks intt (fused modup)");
    }
    // 2) NTT of every converted limb, integer-path limbs first (<= 128 per launch)
    LdModUp ld;
    ld.coef = w.coef; ld.coef_stride = w.coef_s; ld.n = n; ld.tab = c->d_tab; ld.dblmask = dm;
    ld.q = c->t.q; ld.qd = c->t.qd; ld.qinvd = c->t.qinvd;
    for (int j = 0; j < nd; j++) {
        const int lo = j * al, hi = lo + al < nl ? lo + al : nl;
        ld.hm_off[j] = (int)(c->modup_off[(size_t)level * c->beta + j] + 2 * (hi - lo));
        ld.lo[j] = (unsigned char)lo;
        ld.ns[j] = (unsigned char)(hi - lo);
        ld.nt[j] = (unsigned char)(ne - (hi - lo));
    }
    LimbMap m;
    m.count = 0;
    for (int pass = 0; pass < 2; pass++) {
        for (int j = 0; j < nd; j++) {
            const int lo = j * al, hi = lo + al < nl ? lo + al : nl;
            int t = 0;
            for (int e = 0; e < ne; e++) {
                if (e >= lo && e < hi) continue;
                const int prime = e < nl ? e : L + (e - nl);
                const bool wide = c->primes[prime] >= NTT_DBL_BOUND;
                if (wide == (pass == 0)) {
                    m.off[m.count] = (unsigned char)(j * c->LK + e);
                    m.prime[m.count] = (unsigned char)prime;
                    ld.jj[m.count] = (unsigned char)j;
                    ld.tt[m.count] = (unsigned char)t;
                    if (++m.count == HELR_MAXLIMBS) {
                        StBuf st{w.ext, w.ext_s, m, n};
                        ntt_launch<false>(c, ld, st, w.ext, w.ext_s, m, B, s, 1, 1);
                        m.count = 0;
                    }
                }
                t++;
            }
        }
    }
    if (m.count) {
        StBuf st{w.ext, w.ext_s, m, n};
        ntt_launch<false>(c, ld, st, w.ext, w.ext_s, m, B, s, 1, 1);
    }
    CHECK_LAUNCH("ks modup ntt (fused conversion)");
    return HELR_OK;
}
#endif
