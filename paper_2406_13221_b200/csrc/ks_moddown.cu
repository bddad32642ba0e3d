// ks_moddown.cu — ModDown (P -> Q_l, centred) and the merged ModDown +
// rescale, with the conversions fused into the NTT passes by default.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "conv.cuh"

// ModDown conversion: mdc[b][poly][i] = sum_k [a_k * phinv_k]_{p_k} * phmod[k][i] mod q_i
// The conversion kernels write fp64 limbs as raw doubles (read by the NTT with
// in_raw) only when every source prime is below 2^41; with a wide source they
// write canonical residues for every limb and the NTT must read them as such.
static inline bool specials_fp64(const helr_ctx* c) {
    for (int k = 0; k < c->K; k++)
        if (c->primes[c->L + k] >= NTT_DBL_BOUND) return false;
    return true;
}

// Centred conversion (see oracle oc_moddown_convert): subtract r*P with
// r = round(sum_k y_k / p_k) evaluated in IEEE double without contraction,
// so the ModDown error is the zero-mean rounding of x / P.
template <int MK, bool ALLD>
__global__ void k_moddown_conv(const u64* acc, long long acc_item_stride, u64* mdc, long long mdc_item_stride, int n,
                               int nl, int K, int L, const u64* phinv, const u64* phinv_sh, const u64* phm,
                               const u64* phms, const u64* pinv_dbl, const u64* pm, const u64* pm_sh, Tables tb) {
    pdl_begin();
    const int it = blockIdx.y;  // item*2 + poly
    const int b = it >> 1, poly = it & 1;
    const int ne = nl + K;
    const u64* ap = acc + (size_t)b * acc_item_stride + (size_t)poly * ne * n;
    u64* mp = mdc + (size_t)b * mdc_item_stride + (size_t)poly * L * n;
    // the K x nl target weights as doubles, converted once per CTA (every
    // thread used to convert each of them): shared-memory broadcast reads
    __shared__ double wsm[MK <= 8 ? MK * HELR_MAXP : 1];
    constexpr bool WSM = MK <= 8;
    if constexpr (WSM) {
        for (int e = threadIdx.x; e < K * nl; e += blockDim.x) {
            const int k = e / nl, p = e - k * nl;
            wsm[k * HELR_MAXP + p] = u2d(phm[(size_t)k * L + p] & 0x000FFFFFFFFFFFFFull);
        }
        __syncthreads();
    }
    const int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (i >= n) return;
    // ALLD (host: every source prime below 2^41): the sources live only as
    // exact doubles; otherwise integer views are kept as well
    u64 z0[ALLD ? 1 : MK], z1[ALLD ? 1 : MK];
    double zd0[MK], zd1[MK];  // sources as exact doubles (special primes below 2^41)
    double v0 = 0.0, v1 = 0.0;
    bool dsrc = true;
#pragma unroll
    for (int k = 0; k < MK; k++) {
        if (k < K) {
            const u64 pk = tb.q[L + k];
            const double inv = __longlong_as_double((long long)pinv_dbl[k]);
            const ulonglong2 x = ld2(ap + (size_t)(nl + k) * n + i);
            double d0, d1;  // canonical z as exact doubles (no u64 -> f64 conversions)
            if (ALLD || pk < NTT_DBL_BOUND) {
                const DblC dk{tb.qd[L + k], tb.qinvd[L + k]};
                const double w = u2d(phinv[k]);
                d0 = d2d_canon(mulmod_d(u2d(x.x), w, dk), dk);
                d1 = d2d_canon(mulmod_d(u2d(x.y), w, dk), dk);
                zd0[k] = d0;
                zd1[k] = d1;
            } else if constexpr (!ALLD) {
                dsrc = false;
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
    // integer views of the fp64 sources for integer-path targets (ALLD: made at use)
    if constexpr (!ALLD) {
#pragma unroll
        for (int k = 0; k < MK; k++) {
            if (k < K && tb.q[L + k] < NTT_DBL_BOUND) {
                z0[k] = dexact(zd0[k]);
                z1[k] = dexact(zd1[k]);
            }
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
                    const double wd = WSM ? wsm[k * HELR_MAXP + p] : u2d(phm[(size_t)k * L + p]);
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
                const u64 zk0 = ALLD ? dexact(zd0[k]) : z0[ALLD ? 0 : k], zk1 = ALLD ? dexact(zd1[k]) : z1[ALLD ? 0 : k];
                s0 = add_mod(s0, shoup(zk0, w, ws, q), q);
                s1 = add_mod(s1, shoup(zk1, w, ws, q), q);
            }
        }
        // canonical residues: with a wide source prime no limb takes the fp64
        // branch above and the host launches the NTT without in_raw
        st2(mp + (size_t)p * n + i, sub_mod(s0, shoup(rr0, pm[p], pm_sh[p], q), q),
            sub_mod(s1, shoup(rr1, pm[p], pm_sh[p], q), q));
    }
}


// ModDown of w.acc (both polynomials) and the fused epilogue into ep.out
int ks_moddown(helr_ctx* c, int level, const KsEpilogue& ep, int B, const KsWs& w, cudaStream_t s) {
    const int n = c->n, nl = level + 1, K = c->K, L = c->L, ne = nl + K;
#if HELR_FUSE_CONV_BUILD
    if (fuse_conv_enabled() && c->LK <= 64) {
        // INTT of the P limbs pre-scaled by (P/p_k)^-1 (in place), then the
        // NTT whose first pass evaluates the centred conversion (LdModDown)
        LimbMap m;
        m.count = 2 * K;
        StScale st;
        for (int poly = 0; poly < 2; poly++)
            for (int k = 0; k < K; k++) {
                m.off[poly * K + k] = (unsigned char)(poly * ne + nl + k);
                m.prime[poly * K + k] = (unsigned char)(L + k);
            }
        st = st_scale(c, w.acc, w.acc_s, m);
        for (int i = 0; i < 2 * K; i++) {
            st.woff[i] = (int)((c->md_phinv - c->d_tab) + i % K);
            st.wsoff[i] = (int)((c->md_phinv_sh - c->d_tab) + i % K);
        }
        LdBuf ldi{w.acc, w.acc_s, m, n};
        ntt_launch<true>(c, ldi, st, w.acc, w.acc_s, m, B, s, 0, 1);
        CHECK_LAUNCH("ks moddown intt (fused)");
        LimbMap mq;
        mq.count = 2 * nl;
        for (int poly = 0; poly < 2; poly++)
            for (int i = 0; i < nl; i++) {
                mq.off[poly * nl + i] = (unsigned char)(poly * L + i);
                mq.prime[poly * nl + i] = (unsigned char)i;
            }
        LdModDown ld{w.acc, w.acc_s, n, nl, K, L, c->md_phmod, c->md_phmod_sh, c->md_pinv_dbl, c->pmod, c->pmod_sh,
                     c->t.q, c->t.qd, c->t.qinvd};
        StCombine stc = st_combine(c, ep.out, ep.out_stride, (long long)L * n, w.acc, w.acc_s, (long long)ne * n,
                                   c->md_pinv, c->md_pinv_sh, nl);
        stc.add_a = ep.add_a; stc.a_is = ep.add_a_stride; stc.a_ps = (long long)L * n;
        stc.add_p = ep.add_p; stc.p_is = ep.add_p_stride;
        stc.ngal = ep.add_p ? ep.ngal : 0;
        for (int t = 0; t < HELR_MAX_HOIST; t++) stc.gal[t] = ep.gal[t];
        ntt_launch<false>(c, ld, stc, w.mdc, w.mdc_s, mq, B, s, 1);
        CHECK_LAUNCH("ks moddown ntt+final (fused conversion)");
        return HELR_OK;
    }
#endif
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
        bool alld = true;  // every special prime on the fp64 path
        for (int k = 0; k < K; k++) alld = alld && c->primes[L + k] < NTT_DBL_BOUND;
        auto conv = alld ? (K <= 4 ? k_moddown_conv<4, true>
                            : K == 5 ? k_moddown_conv<5, true>
                            : K == 6 ? k_moddown_conv<6, true>
                            : K <= 8 ? k_moddown_conv<8, true>
                            : K <= 16 ? k_moddown_conv<16, true>
                            : K <= 32 ? k_moddown_conv<32, true> : k_moddown_conv<HELR_MAXP, true>)
                         : (K <= 4 ? k_moddown_conv<4, false>
                            : K <= 8 ? k_moddown_conv<8, false>
                            : K <= 16 ? k_moddown_conv<16, false>
                            : K <= 32 ? k_moddown_conv<32, false> : k_moddown_conv<HELR_MAXP, false>);
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
        ntt_launch<false>(c, ld, st, w.mdc, w.mdc_s, mq, B, s, specials_fp64(c) ? 1 : 0);
        CHECK_LAUNCH("ks moddown ntt+final");
    }
    return HELR_OK;
}

// ---- merged ModDown + rescale --------------------------------------------
// acc (PQ_l basis, Q limbs already holding acc + P d) -> round(acc / (P q_l))
// over Q_{l-1}: centred fast conversion from {p_0..p_{K-1}, q_l} (coefficient
// form) to Q_{l-1}, NTT, then (acc_i - conv_i) * (P q_l)^-1.  Saves the
// separate rescale's INTT + l NTTs per polynomial.
template <int MK, bool ALLD>
__global__ void k_mdr_conv(const u64* acc, long long acc_item_stride, u64* mdc, long long mdc_item_stride, int n, int nl,
                           int K, int L, MrTab mt, Tables tb) {
    pdl_begin();
    const int it = blockIdx.y;  // item*2 + poly
    const int b = it >> 1, poly = it & 1;
    const int ne = nl + K, l = nl - 1, ns = K + 1;
    const u64* ap = acc + (size_t)b * acc_item_stride + (size_t)poly * ne * n;
    u64* mp = mdc + (size_t)b * mdc_item_stride + (size_t)poly * L * n;
    __shared__ double wsm[MK <= 8 ? MK * HELR_MAXP : 1];  // target weights as doubles (see k_moddown_conv)
    constexpr bool WSM = MK <= 8;
    if constexpr (WSM) {
        for (int e = threadIdx.x; e < ns * l; e += blockDim.x) {
            const int k = e / l, p = e - k * l;
            wsm[k * HELR_MAXP + p] = u2d(mt.hm[(size_t)k * L + p] & 0x000FFFFFFFFFFFFFull);
        }
        __syncthreads();
    }
    const int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (i >= n) return;
    u64 z0[ALLD ? 1 : MK], z1[ALLD ? 1 : MK];
    double zd0[MK], zd1[MK];
    double v0 = 0.0, v1 = 0.0;
    bool dsrc = true;
#pragma unroll
    for (int k = 0; k < MK; k++) {
        if (k < ns) {
            const int lim = k < K ? nl + k : l;
            const u64 m = tb.q[k < K ? L + k : l];
            const double inv = __longlong_as_double((long long)mt.dinv[k]);
            const ulonglong2 x = ld2(ap + (size_t)lim * n + i);
            double d0, d1;  // canonical z as exact doubles (no u64 -> f64 conversions)
            if (ALLD || m < NTT_DBL_BOUND) {
                const int pm = k < K ? L + k : l;
                const DblC dk{tb.qd[pm], tb.qinvd[pm]};
                const double w = u2d(mt.hv[k]);
                d0 = d2d_canon(mulmod_d(u2d(x.x), w, dk), dk);
                d1 = d2d_canon(mulmod_d(u2d(x.y), w, dk), dk);
                zd0[k] = d0;
                zd1[k] = d1;
            } else if constexpr (!ALLD) {
                dsrc = false;
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
    if constexpr (!ALLD) {
#pragma unroll
        for (int k = 0; k < MK; k++) {
            if (k < ns && tb.q[k < K ? L + k : l] < NTT_DBL_BOUND) {
                z0[k] = dexact(zd0[k]);
                z1[k] = dexact(zd1[k]);
            }
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
                    const double wd = WSM ? wsm[k * HELR_MAXP + p] : u2d(mt.hm[(size_t)k * L + p]);
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
                const u64 zk0 = ALLD ? dexact(zd0[k]) : z0[ALLD ? 0 : k], zk1 = ALLD ? dexact(zd1[k]) : z1[ALLD ? 0 : k];
                s0 = add_mod(s0, shoup(zk0, w, ws, q), q);
                s1 = add_mod(s1, shoup(zk1, w, ws, q), q);
            }
        }
        // canonical residues (see k_moddown_conv)
        st2(mp + (size_t)p * n + i, sub_mod(s0, shoup(rr0, mt.mm[p], mt.mms[p], q), q),
            sub_mod(s1, shoup(rr1, mt.mm[p], mt.mms[p], q), q));
    }
}

int ks_moddown_rescale(helr_ctx* c, int level, u64* out, long long os, int B, const KsWs& w, cudaStream_t s) {
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
#if HELR_FUSE_CONV_BUILD
    if (fuse_conv_enabled() && c->LK <= 64) {
        // pre-scaled INTT of the K + 1 sources (in place), then the NTT whose
        // first pass evaluates the centred conversion (LdMdr)
        StScale st = st_scale(c, w.acc, w.acc_s, m);
        for (int i = 0; i < 2 * (K + 1); i++) {
            st.woff[i] = (int)((mt.hv - c->d_tab) + i % (K + 1));
            st.wsoff[i] = (int)((mt.hvs - c->d_tab) + i % (K + 1));
        }
        LdBuf ldi{w.acc, w.acc_s, m, n};
        ntt_launch<true>(c, ldi, st, w.acc, w.acc_s, m, B, s, 0, 1);
        CHECK_LAUNCH("mdr intt (fused)");
        LimbMap mq;
        mq.count = 2 * l;
        for (int poly = 0; poly < 2; poly++)
            for (int i = 0; i < l; i++) {
                mq.off[poly * l + i] = (unsigned char)(poly * L + i);
                mq.prime[poly * l + i] = (unsigned char)i;
            }
        LdMdr ld{w.acc, w.acc_s, n, nl, K, L, mt.hm, mt.hms, mt.mm, mt.mms, mt.dinv, c->t.q, c->t.qd, c->t.qinvd};
        const StCombine stc = st_combine(c, out, os, (long long)L * n, w.acc, w.acc_s, (long long)ne * n, mt.mi, mt.mis, l);
        ntt_launch<false>(c, ld, stc, w.mdc, w.mdc_s, mq, B, s, 1);
        CHECK_LAUNCH("mdr ntt+final (fused conversion)");
        return HELR_OK;
    }
#endif
    ntt_buffers<true>(c, w.acc, w.acc_s, w.acc, w.acc_s, m, B, s);
    CHECK_LAUNCH("mdr intt");
    {
        dim3 g(blocks_for(n / 2, 128), 2 * B);
        ProfScope ps(PROF_MODDOWN, 8.0 * n * 2.0 * B * (K + 1 + l), s);
        bool alld = c->primes[l] < NTT_DBL_BOUND;  // every source prime (specials and q_l) on the fp64 path
        for (int k = 0; k < K; k++) alld = alld && c->primes[L + k] < NTT_DBL_BOUND;
        auto conv = alld ? (K + 1 <= 4 ? k_mdr_conv<4, true>
                            : K + 1 == 5 ? k_mdr_conv<5, true>
                            : K + 1 == 6 ? k_mdr_conv<6, true>
                            : K + 1 <= 8 ? k_mdr_conv<8, true>
                            : K + 1 <= 16 ? k_mdr_conv<16, true>
                            : K + 1 <= 32 ? k_mdr_conv<32, true> : k_mdr_conv<HELR_MAXP, true>)
                         : (K + 1 <= 4 ? k_mdr_conv<4, false>
                            : K + 1 <= 8 ? k_mdr_conv<8, false>
                            : K + 1 <= 16 ? k_mdr_conv<16, false>
                            : K + 1 <= 32 ? k_mdr_conv<32, false> : k_mdr_conv<HELR_MAXP, false>);
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
        ntt_launch<false>(c, ld, st, w.mdc, w.mdc_s, mq, B, s, specials_fp64(c) && c->primes[l] < NTT_DBL_BOUND ? 1 : 0);
        CHECK_LAUNCH("mdr ntt+final");
    }
    return HELR_OK;
}

