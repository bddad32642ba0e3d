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
        // two consecutive coefficients per thread (16-byte accesses; n is even)
        const DblC dc{tb.qd[p], tb.qinvd[p]};
        const size_t ps = (size_t)L * n;
        for (int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x); i < n; i += 2 * gridDim.x * blockDim.x) {
            double s0x = 0.0, s1x = 0.0, s2x = 0.0, s0y = 0.0, s1y = 0.0, s2y = 0.0;
            for (int t = 0; t < ta.terms; t++) {
                const u64* a0 = ta.a + (size_t)it * ta.a_is + (size_t)t * ta.a_ts + (size_t)p * n + i;
                const u64* b0 = ta.b + (size_t)it * ta.b_is + (size_t)t * ta.b_ts + (size_t)p * n + i;
                const ulonglong2 A0 = ld2(a0), A1 = ld2(a0 + ps), B0 = ld2(b0), B1 = ld2(b0 + ps);
                const double x0 = u2d(A0.x), x1 = u2d(A1.x), y0 = u2d(B0.x), y1 = u2d(B1.x);
                const double z0 = u2d(A0.y), z1 = u2d(A1.y), w0 = u2d(B0.y), w1 = u2d(B1.y);
                s0x = __dadd_rn(s0x, mulmod_d(x0, y0, dc));
                s1x = __dadd_rn(s1x, __dadd_rn(mulmod_d(x0, y1, dc), mulmod_d(x1, y0, dc)));
                s2x = __dadd_rn(s2x, mulmod_d(x1, y1, dc));
                s0y = __dadd_rn(s0y, mulmod_d(z0, w0, dc));
                s1y = __dadd_rn(s1y, __dadd_rn(mulmod_d(z0, w1, dc), mulmod_d(z1, w0, dc)));
                s2y = __dadd_rn(s2y, mulmod_d(z1, w1, dc));
            }
            st2(d0 + i, d2u_canon(s0x, dc), d2u_canon(s0y, dc));
            st2(d1 + i, d2u_canon(s1x, dc), d2u_canon(s1y, dc));
            st2(d2 + i, d2u_canon(s2x, dc), d2u_canon(s2y, dc));
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
        dim3 g(blocks_for(c->n / 2, 256), level + 1, nb);  // two coefficients per thread on fp64 limbs (grid-stride otherwise)
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
