// ks.cu — key switching: ModUp, single-key inner product, ModDown (and the
// merged ModDown + rescale), rotations, hoisted rotate-and-sums, ct x ct
// products.  Hybrid scheme: INTT of the input, per-digit fast basis
// conversion to Q_l + P, NTT, inner product with the key, ModDown by P; all
// `count` ciphertexts of a call go through every stage together so each key
// limb is read once per call.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "ks.cuh"

// ---------------------------------------------------------------------------
// key switching
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
static KsEpilogue make_epilogue(u64* out, long long os, const u64* add_a, long long as, const u64* add_p, long long ps,
                                int ngal, const long long* gal) {
    KsEpilogue e;
    e.out = out; e.out_stride = os; e.add_a = add_a; e.add_a_stride = as; e.add_p = add_p; e.add_p_stride = ps;
    e.ngal = ngal;
    for (int t = 0; t < HELR_MAX_HOIST; t++) e.gal[t] = t < ngal ? gal[t] : 0;
    return e;
}

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
                    const u64 w = hm[(size_t)k * nt + t];
                    if (ydok[k]) {
                        const double wd = u2d(w);
                        s0 = __dadd_rn(s0, mulmod_d(yd0[k], wd, dc));
                        s1 = __dadd_rn(s1, mulmod_d(yd1[k], wd, dc));
                    } else {  // wide source prime (q_0): integer Shoup, result < q
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

// inner product: acc[b][poly][e] = sum_j ext[b][j][e] * evk[j][poly][prime(e)]
// block (64, <= 8): threadIdx.y = ciphertext, so the 8 warps of a block read
// the same key words (one DRAM read, L1 hits for the rest).
// dadd (optional): tensor buffer [B][3][L][N]; for Q limbs the accumulator also
// gets (P mod q) * d0 / d1, so a single division by P*q_l (merged ModDown +
// rescale) yields rescale(d + KS(d2)).
__global__ void k_ks_inner(const u64* ext, long long ext_item_stride, long long ext_digit_stride, const u64* evk,
                           u64* acc, long long acc_item_stride, int n, int nl, int K, int L, int LK, int nd, int B,
                           Tables tb, const u64* dadd, long long dadd_is, const u64* pm, const u64* pm_sh,
                           const u64* one_sh) {
    pdl_begin();
    const int e = blockIdx.y;
    const int b = blockIdx.z * blockDim.y + threadIdx.y;
    const int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (b >= B || i >= n) return;
    const int p = e < nl ? e : L + (e - nl);
    const u64 q = tb.q[p], r1 = tb.br1[p], r0 = tb.br0[p];
    const u64* xb = ext + (size_t)b * ext_item_stride + (size_t)e * n + i;
    u64 o00, o01, o10, o11;
    if (q < NTT_DBL_BOUND) {  // fp64 split-operand MACs (see hoist_body)
        dacc c00{0.0, 0.0, 0.0}, c01{0.0, 0.0, 0.0}, c10{0.0, 0.0, 0.0}, c11{0.0, 0.0, 0.0};
        for (int j = 0; j < nd; j++) {
            const ulonglong2 k0 = ld2(evk + (((size_t)j * 2) * LK + p) * n + i);
            const ulonglong2 k1 = ld2(evk + (((size_t)j * 2 + 1) * LK + p) * n + i);
            const ulonglong2 u = ld2(xb + (size_t)j * ext_digit_stride);
            double uxh, uxl, uyh, uyl, k0xh, k0xl, k0yh, k0yl, k1xh, k1xl, k1yh, k1yl;
            split21_d(__longlong_as_double((long long)u.x), uxh, uxl);  // ext: exact doubles
            split21_d(__longlong_as_double((long long)u.y), uyh, uyl);
            split21(k0.x, k0xh, k0xl); split21(k0.y, k0yh, k0yl);
            split21(k1.x, k1xh, k1xl); split21(k1.y, k1yh, k1yl);
            mac_d(c00, uxh, uxl, k0xh, k0xl);
            mac_d(c01, uyh, uyl, k0yh, k0yl);
            mac_d(c10, uxh, uxl, k1xh, k1xl);
            mac_d(c11, uyh, uyl, k1yh, k1yl);
        }
        // fold on the fp64 pipe (idle here; the integer 128-bit Barrett path
        // was the kernel's bottleneck): hh 2^42 + mid 2^21 + ll, each part
        // reduced first, plus the merged-rescale addend (P mod q) d
        const DblC dc{tb.qd[p], tb.qinvd[p]};
        const double t42 = reduce_d(4398046511104.0, dc);  // 2^42 mod q (signed)
        const double t21 = 2097152.0;
        auto fold = [&](const dacc& c) -> double {
            return __dadd_rn(__dadd_rn(mulmod_d(reduce_d(c.hh, dc), t42, dc), mulmod_d(reduce_d(c.mid, dc), t21, dc)),
                             reduce_d(c.ll, dc));
        };
        double f00 = fold(c00), f01 = fold(c01), f10 = fold(c10), f11 = fold(c11);
        if (dadd && e < nl) {
            const u64* db = dadd + (size_t)b * dadd_is + (size_t)e * n + i;
            const ulonglong2 d0 = ld2(db), d1 = ld2(db + (size_t)L * n);
            const double w = u2d(pm[e]);
            f00 = __dadd_rn(f00, mulmod_d(u2d(d0.x), w, dc));
            f01 = __dadd_rn(f01, mulmod_d(u2d(d0.y), w, dc));
            f10 = __dadd_rn(f10, mulmod_d(u2d(d1.x), w, dc));
            f11 = __dadd_rn(f11, mulmod_d(u2d(d1.y), w, dc));
        }
        u64* ap = acc + (size_t)b * acc_item_stride;
        st2(ap + (size_t)e * n + i, d2u_canon(f00, dc), d2u_canon(f01, dc));
        st2(ap + ((size_t)(nl + K) + e) * n + i, d2u_canon(f10, dc), d2u_canon(f11, dc));
        return;
    } else {
    u128v a00{0, 0}, a01{0, 0}, a10{0, 0}, a11{0, 0};
    for (int j = 0; j < nd; j++) {
        const ulonglong2 k0 = ld2(evk + (((size_t)j * 2) * LK + p) * n + i);
        const ulonglong2 k1 = ld2(evk + (((size_t)j * 2 + 1) * LK + p) * n + i);
        const ulonglong2 u = ld2(xb + (size_t)j * ext_digit_stride);
        acc_wide(a00, u.x, k0.x);
        acc_wide(a01, u.y, k0.y);
        acc_wide(a10, u.x, k1.x);
        acc_wide(a11, u.y, k1.y);
        if ((j & 3) == 3 && j + 1 < nd) {
            a00 = u128v{0, barrett128(a00, q, r1, r0)};
            a01 = u128v{0, barrett128(a01, q, r1, r0)};
            a10 = u128v{0, barrett128(a10, q, r1, r0)};
            a11 = u128v{0, barrett128(a11, q, r1, r0)};
        }
    }
    o00 = barrett128(a00, q, r1, r0); o01 = barrett128(a01, q, r1, r0);
    o10 = barrett128(a10, q, r1, r0); o11 = barrett128(a11, q, r1, r0);
    }
    u64* ap = acc + (size_t)b * acc_item_stride;
    if (dadd && e < nl) {
        const u64* db = dadd + (size_t)b * dadd_is + (size_t)e * n + i;
        const ulonglong2 d0 = ld2(db), d1 = ld2(db + (size_t)L * n);
        const u64 w = pm[e], ws = pm_sh[e];
        o00 = add_mod(o00, shoup(d0.x, w, ws, q), q);
        o01 = add_mod(o01, shoup(d0.y, w, ws, q), q);
        o10 = add_mod(o10, shoup(d1.x, w, ws, q), q);
        o11 = add_mod(o11, shoup(d1.y, w, ws, q), q);
    }
    st2(ap + (size_t)e * n + i, o00, o01);
    st2(ap + ((size_t)(nl + K) + e) * n + i, o10, o11);
}

// ModDown conversion: mdc[b][poly][i] = sum_k [a_k * phinv_k]_{p_k} * phmod[k][i] mod q_i
// Centred conversion (see oracle oc_moddown_convert): subtract r*P with
// r = round(sum_k y_k / p_k) evaluated in IEEE double without contraction,
// so the ModDown error is the zero-mean rounding of x / P.
template <int MK>
__global__ void k_moddown_conv(const u64* acc, long long acc_item_stride, u64* mdc, long long mdc_item_stride, int n,
                               int nl, int K, int L, const u64* phinv, const u64* phinv_sh, const u64* phm,
                               const u64* phms, const u64* pinv_dbl, const u64* pm, const u64* pm_sh, Tables tb) {
    pdl_begin();
    const int it = blockIdx.y;  // item*2 + poly
    const int b = it >> 1, poly = it & 1;
    const int ne = nl + K;
    const u64* ap = acc + (size_t)b * acc_item_stride + (size_t)poly * ne * n;
    u64* mp = mdc + (size_t)b * mdc_item_stride + (size_t)poly * L * n;
    const int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (i >= n) return;
    u64 z0[MK], z1[MK];
    double v0 = 0.0, v1 = 0.0;
#pragma unroll
    for (int k = 0; k < MK; k++) {
        if (k < K) {
            const u64 pk = tb.q[L + k];
            const double inv = __longlong_as_double((long long)pinv_dbl[k]);
            const ulonglong2 x = ld2(ap + (size_t)(nl + k) * n + i);
            double d0, d1;  // canonical z as exact doubles (no u64 -> f64 conversions)
            if (pk < NTT_DBL_BOUND) {
                const DblC dk{tb.qd[L + k], tb.qinvd[L + k]};
                const double w = u2d(phinv[k]);
                d0 = d2d_canon(mulmod_d(u2d(x.x), w, dk), dk);
                d1 = d2d_canon(mulmod_d(u2d(x.y), w, dk), dk);
                z0[k] = dexact(d0);
                z1[k] = dexact(d1);
            } else {
                z0[k] = shoup(x.x, phinv[k], phinv_sh[k], pk);
                z1[k] = shoup(x.y, phinv[k], phinv_sh[k], pk);
                d0 = __ull2double_rn(z0[k]);
                d1 = __ull2double_rn(z1[k]);
            }
            v0 = __dadd_rn(v0, __dmul_rn(d0, inv));
            v1 = __dadd_rn(v1, __dmul_rn(d1, inv));
        }
    }
    const u64 rr0 = (u64)__double2ull_rd(__dadd_rn(v0, 0.5));
    const u64 rr1 = (u64)__double2ull_rd(__dadd_rn(v1, 0.5));
    // sources as exact doubles when every special prime is below 2^41
    bool dsrc = true;
    double zd0[MK], zd1[MK];
#pragma unroll
    for (int k = 0; k < MK; k++) {
        if (k < K) {
            dsrc = dsrc && tb.q[L + k] < NTT_DBL_BOUND;
            zd0[k] = u2d(z0[k] & 0x000FFFFFFFFFFFFFull);
            zd1[k] = u2d(z1[k] & 0x000FFFFFFFFFFFFFull);
        }
    }
    for (int p = 0; p < nl; p++) {
        const u64 q = tb.q[p];
        if (dsrc && q < NTT_DBL_BOUND) {  // fp64 target (see k_modup)
            const DblC dc{tb.qd[p], tb.qinvd[p]};
            const double pmd = u2d(pm[p]);
            double s0 = -__dmul_rn(u2d(rr0), pmd), s1 = -__dmul_rn(u2d(rr1), pmd);  // exact: rr < K + 1
#pragma unroll
            for (int k = 0; k < MK; k++) {
                if (k < K) {
                    const double wd = u2d(phm[(size_t)k * L + p]);
                    s0 = __dadd_rn(s0, mulmod_d(zd0[k], wd, dc));
                    s1 = __dadd_rn(s1, mulmod_d(zd1[k], wd, dc));
                }
            }
            // raw signed doubles: the NTT that follows reads them as is (in_raw)
            st2(mp + (size_t)p * n + i, (u64)__double_as_longlong(reduce_d(s0, dc)),
                (u64)__double_as_longlong(reduce_d(s1, dc)));
            continue;
        }
        u64 s0 = 0, s1 = 0;
#pragma unroll
        for (int k = 0; k < MK; k++) {
            if (k < K) {
                const u64 w = phm[(size_t)k * L + p], ws = phms[(size_t)k * L + p];
                s0 = add_mod(s0, shoup(z0[k], w, ws, q), q);
                s1 = add_mod(s1, shoup(z1[k], w, ws, q), q);
            }
        }
        st2(mp + (size_t)p * n + i, sub_mod(s0, shoup(rr0, pm[p], pm_sh[p], q), q),
            sub_mod(s1, shoup(rr1, pm[p], pm_sh[p], q), q));
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

// ModUp of B inputs into w.ext (NTT form over Q_l + P for every digit)
static int ks_modup(helr_ctx* c, KsInput in, int level, int B, const KsWs& w, cudaStream_t s) {
    const int n = c->n, nl = level + 1, K = c->K, L = c->L, ne = nl + K;
    const int nd = (nl + c->alpha - 1) / c->alpha;
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

// ModDown of w.acc (both polynomials) and the fused epilogue into ep.out
static int ks_moddown(helr_ctx* c, int level, const KsEpilogue& ep, int B, const KsWs& w, cudaStream_t s) {
    const int n = c->n, nl = level + 1, K = c->K, L = c->L, ne = nl + K;
    LimbMap m;
    m.count = 2 * K;  // P limbs of both polynomials in one launch
    for (int poly = 0; poly < 2; poly++)
        for (int k = 0; k < K; k++) {
            m.off[poly * K + k] = (unsigned char)(poly * ne + nl + k);
            m.prime[poly * K + k] = (unsigned char)(L + k);
        }
    ntt_buffers<true>(c, w.acc, w.acc_s, w.acc, w.acc_s, m, B, s);
    CHECK_LAUNCH("ks moddown intt");
    dim3 g(blocks_for(n / 2, 128), 2 * B);
    {
        ProfScope ps(PROF_MODDOWN, 8.0 * n * 2.0 * B * (K + nl), s);
        // register arrays sized to K (dnum 1 rings have K up to ~31)
        auto conv = K <= 4 ? k_moddown_conv<4>
                  : K <= 8 ? k_moddown_conv<8>
                  : K <= 16 ? k_moddown_conv<16>
                  : K <= 32 ? k_moddown_conv<32> : k_moddown_conv<HELR_MAXP>;
        launch_pdl(conv, g, dim3(128), 0, s, (const u64*)w.acc, w.acc_s, w.mdc, w.mdc_s, n, nl, K, L, c->md_phinv,
                   c->md_phinv_sh, c->md_phmod, c->md_phmod_sh, c->md_pinv_dbl, c->pmod, c->pmod_sh, c->t);
        CHECK_KERNEL("ks moddown conv");
    }
    LimbMap mq;
    mq.count = 2 * nl;
    for (int poly = 0; poly < 2; poly++)
        for (int i = 0; i < nl; i++) {
            mq.off[poly * nl + i] = (unsigned char)(poly * L + i);
            mq.prime[poly * nl + i] = (unsigned char)i;
        }
    // NTT of the conversion; its last pass applies (acc - conv) * P^-1 and
    // the epilogue addends while storing (StCombine)
    {
        LdBuf ld{w.mdc, w.mdc_s, mq, n};
        StCombine st = st_combine(c, ep.out, ep.out_stride, (long long)L * n, w.acc, w.acc_s, (long long)ne * n,
                                  c->md_pinv, c->md_pinv_sh, nl);
        st.add_a = ep.add_a; st.a_is = ep.add_a_stride; st.a_ps = (long long)L * n;
        st.add_p = ep.add_p; st.p_is = ep.add_p_stride;
        st.ngal = ep.add_p ? ep.ngal : 0;
        for (int t = 0; t < HELR_MAX_HOIST; t++) st.gal[t] = ep.gal[t];
        ntt_launch<false>(c, ld, st, w.mdc, w.mdc_s, mq, B, s, 1);
        CHECK_LAUNCH("ks moddown ntt+final");
    }
    return HELR_OK;
}

// single-key inner product (relinearisation / one rotation): with one key
// there is no step loop to prefetch across, so the 2-coefficient, ciphertext-
// row kernel (k_ks_inner) is faster than the hoisted kernel here
static int key_inner_single(helr_ctx* c, const KsWs& w, const u64* evk, int B, int level, const u64* dadd,
                            long long dadd_is, cudaStream_t s) {
    const int n = c->n, nl = level + 1, K = c->K, L = c->L, ne = nl + K;
    const int nd = (nl + c->alpha - 1) / c->alpha;
    const int by = B < 8 ? B : 8;
    dim3 g(blocks_for(n / 2, 64), ne, (B + by - 1) / by);
    ProfScope ps(PROF_INNER, 8.0 * n * ((double)B * nd * ne + 2.0 * nd * ne + 2.0 * B * ne + (dadd ? 2.0 * B * nl : 0.0)),
                 s);
    launch_pdl(k_ks_inner, g, dim3(64, by), 0, s, (const u64*)w.ext, w.ext_s, w.ext_ds, evk, w.acc, w.acc_s, n, nl, K, L,
               c->LK, nd, B, c->t, dadd, dadd_is, c->pmod, c->pmod_sh, c->one_sh);
    CHECK_KERNEL("ks inner");
    return HELR_OK;
}

static int keyswitch_batch(helr_ctx* c, KsInput in, const u64* evk, int level, const KsEpilogue& ep, int B,
                           const KsWs& w, cudaStream_t s) {
    int r = ks_modup(c, in, level, B, w, s);
    if (r) return r;
    r = key_inner_single(c, w, evk, B, level, nullptr, 0, s);
    if (r) return r;
    return ks_moddown(c, level, ep, B, w, s);
}

// ---- merged ModDown + rescale --------------------------------------------
// acc (PQ_l basis, Q limbs already holding acc + P d) -> round(acc / (P q_l))
// over Q_{l-1}: centred fast conversion from {p_0..p_{K-1}, q_l} (coefficient
// form) to Q_{l-1}, NTT, then (acc_i - conv_i) * (P q_l)^-1.  Saves the
// separate rescale's INTT + l NTTs per polynomial.
struct MrTab {
    const u64 *hv, *hvs, *hm, *hms, *mm, *mms, *mi, *mis, *dinv;
};
static MrTab mr_tab(const helr_ctx* c, int level) {
    const int ns = c->K + 1, L = c->L;
    const u64* e = c->d_tab + c->mr_off[level];
    MrTab t;
    t.hv = e; t.hvs = e + ns; t.hm = t.hvs + ns; t.hms = t.hm + (size_t)ns * L; t.mm = t.hms + (size_t)ns * L;
    t.mms = t.mm + L; t.mi = t.mms + L; t.mis = t.mi + L; t.dinv = t.mis + L;
    return t;
}
template <int MK>
__global__ void k_mdr_conv(const u64* acc, long long acc_item_stride, u64* mdc, long long mdc_item_stride, int n, int nl,
                           int K, int L, MrTab mt, Tables tb) {
    pdl_begin();
    const int it = blockIdx.y;  // item*2 + poly
    const int b = it >> 1, poly = it & 1;
    const int ne = nl + K, l = nl - 1, ns = K + 1;
    const u64* ap = acc + (size_t)b * acc_item_stride + (size_t)poly * ne * n;
    u64* mp = mdc + (size_t)b * mdc_item_stride + (size_t)poly * L * n;
    const int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (i >= n) return;
    u64 z0[MK], z1[MK];
    double v0 = 0.0, v1 = 0.0;
#pragma unroll
    for (int k = 0; k < MK; k++) {
        if (k < ns) {
            const int lim = k < K ? nl + k : l;
            const u64 m = tb.q[k < K ? L + k : l];
            const double inv = __longlong_as_double((long long)mt.dinv[k]);
            const ulonglong2 x = ld2(ap + (size_t)lim * n + i);
            double d0, d1;  // canonical z as exact doubles (no u64 -> f64 conversions)
            if (m < NTT_DBL_BOUND) {
                const int pm = k < K ? L + k : l;
                const DblC dk{tb.qd[pm], tb.qinvd[pm]};
                const double w = u2d(mt.hv[k]);
                d0 = d2d_canon(mulmod_d(u2d(x.x), w, dk), dk);
                d1 = d2d_canon(mulmod_d(u2d(x.y), w, dk), dk);
                z0[k] = dexact(d0);
                z1[k] = dexact(d1);
            } else {
                z0[k] = shoup(x.x, mt.hv[k], mt.hvs[k], m);
                z1[k] = shoup(x.y, mt.hv[k], mt.hvs[k], m);
                d0 = __ull2double_rn(z0[k]);
                d1 = __ull2double_rn(z1[k]);
            }
            v0 = __dadd_rn(v0, __dmul_rn(d0, inv));
            v1 = __dadd_rn(v1, __dmul_rn(d1, inv));
        }
    }
    const u64 rr0 = (u64)__double2ull_rd(__dadd_rn(v0, 0.5));
    const u64 rr1 = (u64)__double2ull_rd(__dadd_rn(v1, 0.5));
    bool dsrc = true;
    double zd0[MK], zd1[MK];
#pragma unroll
    for (int k = 0; k < MK; k++) {
        if (k < ns) {
            dsrc = dsrc && tb.q[k < K ? L + k : l] < NTT_DBL_BOUND;
            zd0[k] = u2d(z0[k] & 0x000FFFFFFFFFFFFFull);
            zd1[k] = u2d(z1[k] & 0x000FFFFFFFFFFFFFull);
        }
    }
    for (int p = 0; p < l; p++) {
        const u64 q = tb.q[p];
        if (dsrc && q < NTT_DBL_BOUND) {  // fp64 target (see k_modup)
            const DblC dc{tb.qd[p], tb.qinvd[p]};
            const double mmd = u2d(mt.mm[p]);
            double s0 = -__dmul_rn(u2d(rr0), mmd), s1 = -__dmul_rn(u2d(rr1), mmd);  // exact: rr <= K + 1
#pragma unroll
            for (int k = 0; k < MK; k++) {
                if (k < ns) {
                    const double wd = u2d(mt.hm[(size_t)k * L + p]);
                    s0 = __dadd_rn(s0, mulmod_d(zd0[k], wd, dc));
                    s1 = __dadd_rn(s1, mulmod_d(zd1[k], wd, dc));
                }
            }
            st2(mp + (size_t)p * n + i, (u64)__double_as_longlong(reduce_d(s0, dc)),
                (u64)__double_as_longlong(reduce_d(s1, dc)));  // raw (in_raw NTT)
            continue;
        }
        u64 s0 = 0, s1 = 0;
#pragma unroll
        for (int k = 0; k < MK; k++) {
            if (k < ns) {
                const u64 w = mt.hm[(size_t)k * L + p], ws = mt.hms[(size_t)k * L + p];
                s0 = add_mod(s0, shoup(z0[k], w, ws, q), q);
                s1 = add_mod(s1, shoup(z1[k], w, ws, q), q);
            }
        }
        st2(mp + (size_t)p * n + i, sub_mod(s0, shoup(rr0, mt.mm[p], mt.mms[p], q), q),
            sub_mod(s1, shoup(rr1, mt.mm[p], mt.mms[p], q), q));
    }
}

static int ks_moddown_rescale(helr_ctx* c, int level, u64* out, long long os, int B, const KsWs& w, cudaStream_t s) {
    const int n = c->n, nl = level + 1, K = c->K, L = c->L, ne = nl + K, l = level;
    MrTab mt = mr_tab(c, level);
    LimbMap m;
    m.count = 2 * (K + 1);
    for (int poly = 0; poly < 2; poly++) {
        for (int k = 0; k < K; k++) {
            m.off[poly * (K + 1) + k] = (unsigned char)(poly * ne + nl + k);
            m.prime[poly * (K + 1) + k] = (unsigned char)(L + k);
        }
        m.off[poly * (K + 1) + K] = (unsigned char)(poly * ne + l);
        m.prime[poly * (K + 1) + K] = (unsigned char)l;
    }
    ntt_buffers<true>(c, w.acc, w.acc_s, w.acc, w.acc_s, m, B, s);
    CHECK_LAUNCH("mdr intt");
    {
        dim3 g(blocks_for(n / 2, 128), 2 * B);
        ProfScope ps(PROF_MODDOWN, 8.0 * n * 2.0 * B * (K + 1 + l), s);
        auto conv = K + 1 <= 4 ? k_mdr_conv<4>
                  : K + 1 <= 8 ? k_mdr_conv<8>
                  : K + 1 <= 16 ? k_mdr_conv<16>
                  : K + 1 <= 32 ? k_mdr_conv<32> : k_mdr_conv<HELR_MAXP>;
        launch_pdl(conv, g, dim3(128), 0, s, (const u64*)w.acc, w.acc_s, w.mdc, w.mdc_s, n, nl, K, L, mt, c->t);
        CHECK_KERNEL("mdr conv");
    }
    LimbMap mq;
    mq.count = 2 * l;
    for (int poly = 0; poly < 2; poly++)
        for (int i = 0; i < l; i++) {
            mq.off[poly * l + i] = (unsigned char)(poly * L + i);
            mq.prime[poly * l + i] = (unsigned char)i;
        }
    {
        LdBuf ld{w.mdc, w.mdc_s, mq, n};
        const StCombine st = st_combine(c, out, os, (long long)L * n, w.acc, w.acc_s, (long long)ne * n, mt.mi, mt.mis, l);
        ntt_launch<false>(c, ld, st, w.mdc, w.mdc_s, mq, B, s, 1);
        CHECK_LAUNCH("mdr ntt+final");
    }
    return HELR_OK;
}

// ---- hoisted rotate-and-sum ------------------------------------------------
// out = [a +] sum_t rot_{g_t}(a): ONE ModUp of c1, the inner products of every
// rotation summed in the extended basis (sigma_t applied to the ModUp'd digits
// by a warp-coalesced gather: a Galois permutation maps every 32-aligned run of
// NTT slots onto a 32-aligned run), ONE ModDown; sum_t sigma_t(c0) is gathered
// in the ModDown epilogue.  The inner product kernel lives in hoist.cu.
int op_rotsum_hoisted(helr_ctx* c, const u64* a, long long as, int nsteps, const long long* gal, const u64* const* keys,
                      u64* out, long long os, int count, int level, int include_identity, cudaStream_t s) {
    if (level < 0 || level >= c->L) { set_error("bad level"); return HELR_EINVAL; }
    if (nsteps < 1 || nsteps > HELR_MAX_HOIST) { set_error("rotsum: 1..32 rotations per hoisted group"); return HELR_EINVAL; }
    if (a == out) { set_error("rotsum: out must not alias the input"); return HELR_EINVAL; }
    HoistKeys hk;
    hk.nsteps = nsteps;
    long long gg[HELR_MAX_HOIST];
    for (int t = 0; t < HELR_MAX_HOIST; t++) {
        if (t < nsteps) {
            const long long g = gal[t] % (2ll * c->n);
            if (g <= 0 || (g & 1) == 0) { set_error("galois element must be odd and positive"); return HELR_EINVAL; }
            hk.key[t] = keys[t];
            hk.gal[t] = g;
            gg[t] = g;
        } else {
            hk.key[t] = nullptr;
            hk.gal[t] = 1;
        }
    }
    const int n = c->n, nl = level + 1, K = c->K, L = c->L, ne = nl + K;
    const int nd = (nl + c->alpha - 1) / c->alpha;
    const int chunk = c->max_batch;
    for (int b0 = 0; b0 < count; b0 += chunk) {
        const int nb = count - b0 < chunk ? count - b0 : chunk;
        KsWs w = ks_ws(c, chunk);
        const u64* ab = a + (size_t)b0 * as;
        KsInput in{ab + (size_t)L * n, as, 0};
        int r = ks_modup(c, in, level, nb, w, s);
        if (r) return r;
        r = key_inner(c, w, hk, nb, level, nullptr, 0, s);
        if (r) return r;
        KsEpilogue ep = make_epilogue(out + (size_t)b0 * os, os, include_identity ? ab : nullptr, as, ab, as, nsteps, gg);
        r = ks_moddown(c, level, ep, nb, w, s);
        if (r) return r;
    }
    return HELR_OK;
}

extern "C" int helr_rotsum(helr_ctx* c, const uint64_t* a, int nsteps, const int64_t* galois,
                           const uint64_t* const* keys, uint64_t* out, int count, int level, int include_identity,
                           void* s) {
    clear_stale_error("helr_rotsum");
    const long long cs = 2ll * c->L * c->n;
    long long g[HELR_MAX_HOIST];
    for (int t = 0; t < nsteps && t < HELR_MAX_HOIST; t++) g[t] = (long long)galois[t];
    return op_rotsum_hoisted(c, (const u64*)a, cs, nsteps, g, (const u64* const*)keys, (u64*)out, cs, count, level,
                             include_identity, S(s));
}

// tensor sum: d = sum_t a_t (x) b_t  (d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1) into [B][3][L][N]
struct TensorArgs {
    const u64* a; long long a_is, a_ts;
    const u64* b; long long b_is, b_ts;
    int terms;
};
__global__ void k_tensor(TensorArgs ta, u64* d, int n, int L, Tables tb) {
    pdl_begin();
    const int p = blockIdx.y, it = blockIdx.z;
    const u64 q = tb.q[p], r1 = tb.br1[p], r0 = tb.br0[p];
    u64* d0 = d + (size_t)it * 3 * L * n + (size_t)p * n;
    u64* d1 = d0 + (size_t)L * n;
    u64* d2 = d1 + (size_t)L * n;
    if (q < NTT_DBL_BOUND) {  // fp64 limb: exact signed products, one reduction (|sum| < 1.2 q * 2 terms)
        const DblC dc{tb.qd[p], tb.qinvd[p]};
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            double s0 = 0.0, s1 = 0.0, s2 = 0.0;
            for (int t = 0; t < ta.terms; t++) {
                const u64* a0 = ta.a + (size_t)it * ta.a_is + (size_t)t * ta.a_ts + (size_t)p * n;
                const u64* b0 = ta.b + (size_t)it * ta.b_is + (size_t)t * ta.b_ts + (size_t)p * n;
                const double x0 = u2d(a0[i]), x1 = u2d(a0[(size_t)L * n + i]);
                const double y0 = u2d(b0[i]), y1 = u2d(b0[(size_t)L * n + i]);
                s0 = __dadd_rn(s0, mulmod_d(x0, y0, dc));
                s1 = __dadd_rn(s1, __dadd_rn(mulmod_d(x0, y1, dc), mulmod_d(x1, y0, dc)));
                s2 = __dadd_rn(s2, mulmod_d(x1, y1, dc));
            }
            d0[i] = d2u_canon(s0, dc);
            d1[i] = d2u_canon(s1, dc);
            d2[i] = d2u_canon(s2, dc);
        }
        return;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        u128v s0{0, 0}, s1{0, 0}, s2{0, 0};
        for (int t = 0; t < ta.terms; t++) {
            const u64* a0 = ta.a + (size_t)it * ta.a_is + (size_t)t * ta.a_ts + (size_t)p * n;
            const u64* b0 = ta.b + (size_t)it * ta.b_is + (size_t)t * ta.b_ts + (size_t)p * n;
            const u64 x0 = a0[i], x1 = a0[(size_t)L * n + i], y0 = b0[i], y1 = b0[(size_t)L * n + i];
            acc_wide(s0, x0, y0);
            acc_wide(s1, x0, y1);
            acc_wide(s1, x1, y0);
            acc_wide(s2, x1, y1);
            if ((t & 1) == 1 && t + 1 < ta.terms) {
                s0 = u128v{0, barrett128(s0, q, r1, r0)};
                s1 = u128v{0, barrett128(s1, q, r1, r0)};
                s2 = u128v{0, barrett128(s2, q, r1, r0)};
            }
        }
        d0[i] = barrett128(s0, q, r1, r0);
        d1[i] = barrett128(s1, q, r1, r0);
        d2[i] = barrett128(s2, q, r1, r0);
    }
}

int op_mul_relin_sum(helr_ctx* c, const u64* a, long long a_is, long long a_ts, const u64* b, long long b_is,
                     long long b_ts, int terms, const u64* rlk, u64* out, long long os, int count, int level,
                     cudaStream_t s) {
    if (level < 0 || level >= c->L) { set_error("bad level"); return HELR_EINVAL; }
    if (terms < 1) { set_error("need at least one product term"); return HELR_EINVAL; }
    const int chunk = c->max_batch;
    for (int b0 = 0; b0 < count; b0 += chunk) {
        int nb = count - b0 < chunk ? count - b0 : chunk;
        KsWs w = ks_ws(c, chunk);
        dim3 g(blocks_for(c->n, 256), level + 1, nb);
        TensorArgs ta{a + (size_t)b0 * a_is, a_is, a_ts, b + (size_t)b0 * b_is, b_is, b_ts, terms};
        {
            ProfScope ps(PROF_TENSOR, 8.0 * c->n * nb * (level + 1) * (4.0 * terms + 3.0), s);
            launch_pdl(k_tensor, g, dim3(256), 0, s, ta, w.tensor, c->n, c->L, c->t);
            CHECK_KERNEL("tensor");
        }
        const long long ts = 3ll * c->L * c->n;
        KsInput in{w.tensor + 2ll * c->L * c->n, ts, 0};
        KsEpilogue ep = make_epilogue(out + (size_t)b0 * os, os, w.tensor, ts, nullptr, 0, 0, nullptr);
        int r = keyswitch_batch(c, in, rlk, level, ep, nb, w, s);
        if (r) return r;
    }
    return HELR_OK;
}

extern "C" int helr_mul_relin(helr_ctx* c, const uint64_t* a, const uint64_t* b, const uint64_t* rlk, uint64_t* out,
                              int count, int level, void* s) {
    clear_stale_error("helr_mul_relin");
    const long long cs = 2ll * c->L * c->n;
    return op_mul_relin_sum(c, (const u64*)a, cs, 0, (const u64*)b, cs, 0, 1, (const u64*)rlk, (u64*)out, cs, count,
                            level, S(s));
}

// out_i (level-1) = rescale(relin(sum_t a (x) b)) with the rescale merged into
// the key switch's ModDown (one division by P * q_level)
int op_mul_relin_rescale_sum(helr_ctx* c, const u64* a, long long a_is, long long a_ts, const u64* b, long long b_is,
                             long long b_ts, int terms, const u64* rlk, u64* out, long long os, int count, int level,
                             cudaStream_t s) {
    if (level < 1 || level >= c->L) { set_error("mul+rescale needs level >= 1"); return HELR_EINVAL; }
    if (terms < 1) { set_error("need at least one product term"); return HELR_EINVAL; }
    const int n = c->n, nl = level + 1, K = c->K, L = c->L, ne = nl + K;
    const int nd = (nl + c->alpha - 1) / c->alpha;
    const int chunk = c->max_batch;
    for (int b0 = 0; b0 < count; b0 += chunk) {
        int nb = count - b0 < chunk ? count - b0 : chunk;
        KsWs w = ks_ws(c, chunk);
        {
            dim3 g(blocks_for(n, 256), level + 1, nb);
            ProfScope ps(PROF_TENSOR, 8.0 * n * nb * (level + 1) * (4.0 * terms + 3.0), s);
            TensorArgs ta{a + (size_t)b0 * a_is, a_is, a_ts, b + (size_t)b0 * b_is, b_is, b_ts, terms};
            launch_pdl(k_tensor, g, dim3(256), 0, s, ta, w.tensor, n, L, c->t);
            CHECK_KERNEL("tensor");
        }
        const long long ts = 3ll * L * n;
        KsInput in{w.tensor + 2ll * L * n, ts, 0};
        int r = ks_modup(c, in, level, nb, w, s);
        if (r) return r;
        r = key_inner_single(c, w, rlk, nb, level, w.tensor, ts, s);
        if (r) return r;
        r = ks_moddown_rescale(c, level, out + (size_t)b0 * os, os, nb, w, s);
        if (r) return r;
    }
    return HELR_OK;
}

extern "C" int helr_mul_relin_rescale(helr_ctx* c, const uint64_t* a, const uint64_t* b, const uint64_t* rlk,
                                      uint64_t* out, int count, int level, void* s) {
    clear_stale_error("helr_mul_relin_rescale");
    const long long cs = 2ll * c->L * c->n;
    return op_mul_relin_rescale_sum(c, (const u64*)a, cs, 0, (const u64*)b, cs, 0, 1, (const u64*)rlk, (u64*)out, cs,
                                    count, level, S(s));
}

int op_rotate(helr_ctx* c, const u64* a, long long as, long long galois, const u64* gk, u64* out, long long os,
              int count, int level, int accumulate, cudaStream_t s) {
    if (level < 0 || level >= c->L) { set_error("bad level"); return HELR_EINVAL; }
    if (galois <= 0 || (galois & 1) == 0) { set_error("galois element must be odd and positive"); return HELR_EINVAL; }
    if (a == out) { set_error("rotate: out must not alias the input"); return HELR_EINVAL; }
    const int chunk = c->max_batch;
    const long long g = (long long)(galois % (2ll * c->n));
    for (int b0 = 0; b0 < count; b0 += chunk) {
        int nb = count - b0 < chunk ? count - b0 : chunk;
        KsWs w = ks_ws(c, chunk);
        const u64* ab = a + (size_t)b0 * as;
        KsInput in{ab + (size_t)c->L * c->n, as, g};
        KsEpilogue ep = make_epilogue(out + (size_t)b0 * os, os, accumulate ? ab : nullptr, as, ab, as, 1, &g);
        int r = keyswitch_batch(c, in, gk, level, ep, nb, w, s);
        if (r) return r;
    }
    return HELR_OK;
}

extern "C" int helr_rotate(helr_ctx* c, const uint64_t* a, int64_t galois, const uint64_t* gk, uint64_t* out, int count,
                           int level, int accumulate, void* s) {
    clear_stale_error("helr_rotate");
    const long long cs = 2ll * c->L * c->n;
    return op_rotate(c, (const u64*)a, cs, (long long)galois, (const u64*)gk, (u64*)out, cs, count, level, accumulate,
                     S(s));
}

// out = sum_t C_t * X_t  (per-limb constants, both polynomials), no rescale
