// ops.cu — evaluator operations behind the C ABI (include/helr_ckks.h).
//
// Reference mapping (pkg/src/helr/hesim.py): enc 146-158 -> helr_encrypt,
// dec 160-162 -> helr_decrypt, add 166-175 -> helr_add, cadd 177-184 ->
// helr_add_const / helr_add_plain, mul 186-195 -> helr_mul_relin +
// helr_rescale, cmul 197-206 -> helr_mul_const / helr_mul_plain +
// helr_rescale, imul 208-216 -> helr_imul, rotate 218-226 -> helr_rotate,
// bootstrap 228-236 -> helr_refresh (stand-in).
//
// Key switching (used by mul and rotate) is the hybrid scheme: INTT of the
// input, per-digit fast basis conversion to the extended basis Q_l + P
// (ModUp), NTT, inner product with the key, ModDown by P.  All `count`
// ciphertexts of a call go through every stage together so each key limb is
// read once per call (key batching across the row blocks of a mini-batch).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <utility>
#include <vector>

#include "ks.cuh"

// ---------------------------------------------------------------------------
// elementwise kernels.  Items are ciphertexts (2 polys) unless noted; index
// space: (item, poly, limb, n) flattened with limbs 0..level.
struct EwGeom {
    int n, log_n, L, nl;      // nl = level+1 active limbs
    long long as, bs, os;     // item strides (words) of a, b (ciphertext operands), out
};
__device__ __forceinline__ void ew_decode(long long idx, const EwGeom& g, int& item, int& poly, int& limb, int& k) {
    k = (int)(idx & (g.n - 1));
    const unsigned r = (unsigned)(idx >> g.log_n);  // < items * 2 * limbs: 32-bit division
    const unsigned rq = r / (unsigned)g.nl;
    limb = (int)(r - rq * (unsigned)g.nl);
    poly = (int)(rq & 1u);
    item = (int)(rq >> 1);
}


// one element; op is uniform across the launch
__device__ __forceinline__ u64 ew_apply(int op, u64 x, u64 bv, int poly, u64 q, int limb, const Tables& tb) {
    switch (op) {
        case EW_ADD: return add_mod(x, bv, q);
        case EW_SUB: return sub_mod(x, bv, q);
        case EW_ADDC:
        case EW_ADDPT: return poly == 0 ? add_mod(x, bv, q) : x;
        case EW_REDUCE: return barrett128(u128v{0, x}, q, tb.br1[limb], tb.br0[limb]);
        default:
            if (q < NTT_DBL_BOUND) {
                const DblC dc{tb.qd[limb], tb.qinvd[limb]};
                return d2u_canon(mulmod_d(u2d(x), u2d(bv), dc), dc);
            }
            return mul_mod(x, bv, q, tb.br1[limb], tb.br0[limb]);
    }
}
// Two consecutive coefficients per thread (16-byte accesses, one index
// decode per pair); n is even for every ring.
__global__ void k_elementwise(int op, const u64* a, const u64* b, u64* out, EwGeom g, long long total,
                              Tables tb, const u64* imul_f) {
    pdl_begin();
    const long long pairs = total >> 1;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < pairs;
         idx += (long long)gridDim.x * blockDim.x) {
        int item, poly, limb, k;
        ew_decode(idx << 1, g, item, poly, limb, k);
        const u64 q = tb.q[limb];
        const size_t in_poly = ((size_t)poly * g.L + limb) * g.n + k;
        const ulonglong2 x = ld2(a + (size_t)item * g.as + in_poly);
        ulonglong2 bv;
        switch (op) {
            case EW_ADD:
            case EW_SUB: bv = ld2(b + (size_t)item * g.bs + in_poly); break;
            case EW_ADDC:
            case EW_MULC: bv.x = bv.y = b[limb]; break;
            case EW_ADDPT:
            case EW_MULPT: bv = ld2(b + (size_t)limb * g.n + k); break;
            case EW_REDUCE: bv = make_ulonglong2(0, 0); break;
            default: bv = ld2(imul_f + (size_t)limb * g.n + k); break;
        }
        st2(out + (size_t)item * g.os + in_poly, ew_apply(op, x.x, bv.x, poly, q, limb, tb),
            ew_apply(op, x.y, bv.y, poly, q, limb, tb));
    }
}

int op_ew(helr_ctx* c, int op, const u64* a, long long as, const u64* b, long long bs, u64* out, long long os,
          int count, int level, cudaStream_t s) {
    if (level < 0 || level >= c->L || count < 0) { set_error("bad level/count"); return HELR_EINVAL; }
    if (count == 0) return HELR_OK;
    EwGeom g{c->n, c->log_n, c->L, level + 1, as, bs, os};
    long long total = (long long)count * 2 * (level + 1) * c->n;
    int blocks = blocks_for(total / 2, 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    ProfScope ps(PROF_ELEM, 8.0 * total * ((op == EW_ADD || op == EW_SUB) ? 3 : 2), s);
    if (op == EW_REDUCE) b = a;  // unary
    launch_pdl(k_elementwise, dim3(blocks), dim3(256), 0, s, op, a, b, out, g, total, c->t, c->imul_f);
    CHECK_KERNEL("elementwise");
    return HELR_OK;
}

static int launch_ew(helr_ctx* c, int op, const u64* a, const u64* b, u64* out, int count, int level, void* s) {
    const long long cs = 2ll * c->L * c->n;
    return op_ew(c, op, a, cs, b, cs, out, cs, count, level, S(s));
}

extern "C" int helr_add(helr_ctx* c, const uint64_t* a, const uint64_t* b, uint64_t* out, int count, int level, void* s) {
    clear_stale_error("helr_add");
    return launch_ew(c, EW_ADD, (const u64*)a, (const u64*)b, (u64*)out, count, level, s);
}
extern "C" int helr_sub(helr_ctx* c, const uint64_t* a, const uint64_t* b, uint64_t* out, int count, int level, void* s) {
    clear_stale_error("helr_sub");
    return launch_ew(c, EW_SUB, (const u64*)a, (const u64*)b, (u64*)out, count, level, s);
}
extern "C" int helr_add_const(helr_ctx* c, const uint64_t* a, const uint64_t* k, uint64_t* out, int count, int level, void* s) {
    clear_stale_error("helr_add_const");
    return launch_ew(c, EW_ADDC, (const u64*)a, (const u64*)k, (u64*)out, count, level, s);
}
extern "C" int helr_add_plain(helr_ctx* c, const uint64_t* a, const uint64_t* pt, uint64_t* out, int count, int level, void* s) {
    clear_stale_error("helr_add_plain");
    return launch_ew(c, EW_ADDPT, (const u64*)a, (const u64*)pt, (u64*)out, count, level, s);
}
extern "C" int helr_mul_const(helr_ctx* c, const uint64_t* a, const uint64_t* k, uint64_t* out, int count, int level, void* s) {
    clear_stale_error("helr_mul_const");
    return launch_ew(c, EW_MULC, (const u64*)a, (const u64*)k, (u64*)out, count, level, s);
}
extern "C" int helr_reduce(helr_ctx* c, const uint64_t* a, uint64_t* out, int count, int level, void* s) {
    clear_stale_error("helr_reduce");
    return launch_ew(c, EW_REDUCE, (const u64*)a, nullptr, (u64*)out, count, level, s);
}
extern "C" int helr_mul_plain(helr_ctx* c, const uint64_t* a, const uint64_t* pt, uint64_t* out, int count, int level, void* s) {
    clear_stale_error("helr_mul_plain");
    return launch_ew(c, EW_MULPT, (const u64*)a, (const u64*)pt, (u64*)out, count, level, s);
}
extern "C" int helr_imul(helr_ctx* c, const uint64_t* a, uint64_t* out, int count, int level, void* s) {
    clear_stale_error("helr_imul");
    return launch_ew(c, EW_IMUL, (const u64*)a, nullptr, (u64*)out, count, level, s);
}

// ---------------------------------------------------------------------------
// NTT entry points
extern "C" int helr_ntt_fwd(helr_ctx* c, uint64_t* data, int first_prime, int n_limbs, int count, int64_t stride,
                            void* s) {
    clear_stale_error("helr_ntt_fwd");
    if (first_prime < 0 || n_limbs < 1 || first_prime + n_limbs > c->LK) { set_error("bad limb range"); return HELR_EINVAL; }
    if (count < 1) return HELR_OK;
    LimbMap m = limb_range(first_prime, n_limbs);
    ntt_buffers<false>(c, (const u64*)data, stride, (u64*)data, stride, m, count, S(s));
    CHECK_LAUNCH("ntt_fwd");
    return HELR_OK;
}
extern "C" int helr_ntt_inv(helr_ctx* c, uint64_t* data, int first_prime, int n_limbs, int count, int64_t stride,
                            void* s) {
    clear_stale_error("helr_ntt_inv");
    if (first_prime < 0 || n_limbs < 1 || first_prime + n_limbs > c->LK) { set_error("bad limb range"); return HELR_EINVAL; }
    if (count < 1) return HELR_OK;
    LimbMap m = limb_range(first_prime, n_limbs);
    ntt_buffers<true>(c, (const u64*)data, stride, (u64*)data, stride, m, count, S(s));
    CHECK_LAUNCH("ntt_inv");
    return HELR_OK;
}

// ---------------------------------------------------------------------------
// keys
__global__ void k_fill_secret(u64* sk, int n, int LK, u64 seed, Tables tb) {
    const u64 key = prng_key(seed, stream_id(ST_SK, 0, 0, PU_S));
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const long long sv = (long long)(prng_at(key, (u64)i) % 3ull) - 1;
        for (int p = 0; p < LK; p++) sk[(size_t)p * n + i] = reduce_i64(sv, tb.q[p]);
    }
}

__global__ void k_secret_from_coeffs(u64* sk, const signed char* s8, int n, int LK, Tables tb) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const long long sv = s8[i];
        for (int p = 0; p < LK; p++) sk[(size_t)p * n + i] = reduce_i64(sv, tb.q[p]);
    }
}

extern "C" int helr_keygen_secret(helr_ctx* c, uint64_t* sk, uint64_t seed, void* s) {
    clear_stale_error("helr_keygen_secret");
    k_fill_secret<<<blocks_for(c->n, 256), 256, 0, S(s)>>>((u64*)sk, c->n, c->LK, seed, c->t);
    CHECK_KERNEL("keygen_secret");
    LimbMap m = limb_range(0, c->LK);
    ntt_buffers<false>(c, (const u64*)sk, 0, (u64*)sk, 0, m, 1, S(s));
    CHECK_LAUNCH("keygen_secret ntt");
    return HELR_OK;
}

// Sparse ternary secret with exactly hw nonzero +-1 coefficients (HEAAN's
// default family): positions = the hw smallest prng(seed, SK/0, i), ties by
// index; sign = bit 0 of prng(seed, SK/1, i).  Selected on the host (client
// key generation), identical rule in oracle/ckks_oracle.c oc_secret_coeffs.
extern "C" int helr_keygen_secret_hw(helr_ctx* c, uint64_t* sk, uint64_t seed, int hw, void* s) {
    clear_stale_error("helr_keygen_secret_hw");
    if (hw <= 0) return helr_keygen_secret(c, sk, seed, s);
    const int n = c->n;
    const u64 key = prng_key(seed, stream_id(ST_SK, 0, 0, PU_S));
    const u64 ksg = prng_key(seed, stream_id(ST_SK, 0, 1, PU_S));
    std::vector<std::pair<u64, int>> rk(n);
    for (int i = 0; i < n; i++) rk[i] = {prng_at(key, (u64)i), i};
    std::sort(rk.begin(), rk.end());
    std::vector<signed char> s8(n, 0);
    for (int k = 0; k < hw && k < n; k++) {
        const int i = rk[k].second;
        s8[i] = (prng_at(ksg, (u64)i) & 1) ? 1 : -1;
    }
    signed char* d8 = nullptr;
    if (!cuda_ok(cudaMalloc(&d8, n), "cudaMalloc(secret)")) return HELR_ECUDA;
    if (!cuda_ok(cudaMemcpy(d8, s8.data(), n, cudaMemcpyHostToDevice), "upload secret")) { cudaFree(d8); return HELR_ECUDA; }
    k_secret_from_coeffs<<<blocks_for(n, 256), 256, 0, S(s)>>>((u64*)sk, d8, n, c->LK, c->t);
    CHECK_KERNEL("keygen_secret_hw");
    LimbMap m = limb_range(0, c->LK);
    ntt_buffers<false>(c, (const u64*)sk, 0, (u64*)sk, 0, m, 1, S(s));
    CHECK_LAUNCH("keygen_secret_hw ntt");
    cudaStreamSynchronize(S(s));
    cudaFree(d8);
    return HELR_OK;
}

// evk[j][0][p] := e_j mod q_p  (coefficient form; NTT'd afterwards)
__global__ void k_fill_key_error(u64* evk, int n, int LK, int beta, u64 seed, u64 key_id, int eta, Tables tb) {
    const int j = blockIdx.y;
    const u64 key = prng_key(seed, stream_id(ST_KEY, key_id, (u64)j, PU_E));
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const long long e = cbd_from(prng_at(key, (u64)i), eta);
        for (int p = 0; p < LK; p++) evk[(((size_t)j * 2) * LK + p) * n + i] = reduce_i64(e, tb.q[p]);
    }
}
// b1 = a (uniform), b0 = e - a*s + [p in digit j] * (P mod q_p) * s'
__global__ void k_key_combine(u64* evk, const u64* sk, int n, int log_n, int L, int LK, int alpha, u64 seed,
                              u64 key_id, long long galois, Tables tb, const u64* pmod) {
    const int j = blockIdx.z, p = blockIdx.y;
    const u64 q = tb.q[p], r1 = tb.br1[p], r0 = tb.br0[p];
    const u64 key = prng_key(seed, stream_id(ST_KEY, key_id, (u64)j, PU_A));
    const bool in_digit = p < L && p / alpha == j;
    const u64 f = in_digit ? pmod[p] : 0;
    const u64* sp = sk + (size_t)p * n;
    u64* b0 = evk + (((size_t)j * 2) * LK + p) * n;
    u64* b1 = evk + (((size_t)j * 2 + 1) * LK + p) * n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const u64 ctr = 2ull * ((u64)p * n + i);
        const u64 a = uniform_from(prng_at(key, ctr), prng_at(key, ctr + 1), q, r1, r0);
        u64 v = sub_mod(b0[i], mul_mod(a, sp[i], q, r1, r0), q);
        if (in_digit) {
            u64 s2;
            if (galois == 0) s2 = mul_mod(sp[i], sp[i], q, r1, r0);
            else s2 = sp[galois_perm(i, (u64)galois, log_n)];
            v = add_mod(v, mul_mod(f, s2, q, r1, r0), q);
        }
        b0[i] = v;
        b1[i] = a;
    }
}

extern "C" int helr_keygen_switch(helr_ctx* c, const uint64_t* sk, int64_t galois, uint64_t* evk, uint64_t seed,
                                  uint64_t key_id, void* s) {
    clear_stale_error("helr_keygen_switch");
    if (galois != 0 && ((galois & 1) == 0 || galois < 0)) { set_error("galois element must be odd and positive"); return HELR_EINVAL; }
    galois = galois % (2ll * c->n);
    dim3 g1(blocks_for(c->n, 256), c->beta);
    k_fill_key_error<<<g1, 256, 0, S(s)>>>((u64*)evk, c->n, c->LK, c->beta, seed, key_id, c->eta, c->t);
    CHECK_KERNEL("keygen error");
    LimbMap m = limb_range(0, c->LK);
    const long long st = 2ll * c->LK * c->n;
    ntt_buffers<false>(c, (const u64*)evk, st, (u64*)evk, st, m, c->beta, S(s));
    CHECK_LAUNCH("keygen ntt");
    dim3 g2(blocks_for(c->n, 256), c->LK, c->beta);
    k_key_combine<<<g2, 256, 0, S(s)>>>((u64*)evk, (const u64*)sk, c->n, c->log_n, c->L, c->LK, c->alpha, seed, key_id,
                                        (long long)galois, c->t, c->pmod);
    CHECK_KERNEL("keygen combine");
    return HELR_OK;
}

// ---------------------------------------------------------------------------
// encryption / decryption
__global__ void k_enc_fill(u64* ct, const long long* msg, int n, int L, int nl, u64 seed, u64 first_id, int eta,
                           Tables tb) {
    pdl_begin();
    const int b = blockIdx.y;
    const u64 key = prng_key(seed, stream_id(ST_CT, first_id + (u64)b, 0, PU_E));
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const long long v = msg[(size_t)b * n + i] + cbd_from(prng_at(key, (u64)i), eta);
        for (int p = 0; p < nl; p++) ct[(size_t)b * 2 * L * n + (size_t)p * n + i] = reduce_i64(v, tb.q[p]);
    }
}
__global__ void k_enc_combine(u64* ct, const u64* sk, int n, int L, u64 seed, u64 first_id, Tables tb) {
    pdl_begin();
    const int b = blockIdx.z, p = blockIdx.y;
    const u64 q = tb.q[p], r1 = tb.br1[p], r0 = tb.br0[p];
    const u64 key = prng_key(seed, stream_id(ST_CT, first_id + (u64)b, 0, PU_A));
    u64* c0 = ct + (size_t)b * 2 * L * n + (size_t)p * n;
    u64* c1 = c0 + (size_t)L * n;
    const u64* sp = sk + (size_t)p * n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const u64 ctr = 2ull * ((u64)p * n + i);
        const u64 a = uniform_from(prng_at(key, ctr), prng_at(key, ctr + 1), q, r1, r0);
        c1[i] = a;
        c0[i] = sub_mod(c0[i], mul_mod(a, sp[i], q, r1, r0), q);
    }
}

static int encrypt_dev(helr_ctx* c, const u64* sk, const long long* msg, u64* ct, int count, int level, u64 seed,
                       u64 first_id, cudaStream_t s) {
    dim3 g1(blocks_for(c->n, 256), count);
    launch_pdl(k_enc_fill, g1, dim3(256), 0, s, ct, msg, c->n, c->L, level + 1, seed, first_id, c->eta, c->t);
    CHECK_KERNEL("encrypt fill");
    LimbMap m = limb_range(0, level + 1);
    const long long st = 2ll * c->L * c->n;
    ntt_buffers<false>(c, ct, st, ct, st, m, count, s);
    CHECK_LAUNCH("encrypt ntt");
    dim3 g2(blocks_for(c->n, 256), level + 1, count);
    launch_pdl(k_enc_combine, g2, dim3(256), 0, s, ct, sk, c->n, c->L, seed, first_id, c->t);
    CHECK_KERNEL("encrypt combine");
    return HELR_OK;
}

extern "C" int helr_encrypt(helr_ctx* c, const uint64_t* sk, const int64_t* msg, uint64_t* ct, int count, int level,
                            uint64_t seed, uint64_t first_id, void* s) {
    clear_stale_error("helr_encrypt");
    if (level < 0 || level >= c->L) { set_error("bad level"); return HELR_EINVAL; }
    if (count < 1) return HELR_OK;
    return encrypt_dev(c, (const u64*)sk, (const long long*)msg, (u64*)ct, count, level, seed, first_id, S(s));
}

__global__ void k_dec_combine(const u64* ct, const u64* sk, u64* v, int n, int L, Tables tb) {
    pdl_begin();
    const int b = blockIdx.y;
    const u64 q = tb.q[0], r1 = tb.br1[0], r0 = tb.br0[0];
    const u64* c0 = ct + (size_t)b * 2 * L * n;
    const u64* c1 = c0 + (size_t)L * n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        v[(size_t)b * n + i] = add_mod(c0[i], mul_mod(c1[i], sk[i], q, r1, r0), q);
}
__global__ void k_center(const u64* v, long long* out, long long total, double ratio, Tables tb) {
    pdl_begin();
    const u64 q = tb.q[0];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const u64 x = v[i];
        long long m = x > (q >> 1) ? (long long)x - (long long)q : (long long)x;
        if (ratio != 1.0) m = __double2ll_rn(__dmul_rn(__ll2double_rn(m), ratio));
        out[i] = m;
    }
}

static int decrypt_dev(helr_ctx* c, const u64* sk, const u64* ct, int count, long long* out, double ratio,
                       u64* tmp, cudaStream_t s) {
    dim3 g(blocks_for(c->n, 256), count);
    launch_pdl(k_dec_combine, g, dim3(256), 0, s, ct, sk, tmp, c->n, c->L, c->t);
    CHECK_KERNEL("decrypt combine");
    LimbMap m = limb_range(0, 1);
    ntt_buffers<true>(c, tmp, c->n, tmp, c->n, m, count, s);
    CHECK_LAUNCH("decrypt intt");
    long long total = (long long)count * c->n;
    launch_pdl(k_center, dim3(blocks_for(total, 256) < 4096 ? blocks_for(total, 256) : 4096), dim3(256), 0, s, (const u64*)tmp,
               out, total, ratio, c->t);
    CHECK_KERNEL("decrypt center");
    return HELR_OK;
}

extern "C" int helr_decrypt(helr_ctx* c, const uint64_t* sk, const uint64_t* ct, int count, int level, int64_t* out,
                            void* s) {
    clear_stale_error("helr_decrypt");
    if (level < 0 || level >= c->L) { set_error("bad level"); return HELR_EINVAL; }
    for (int b0 = 0; b0 < count; b0 += c->max_batch) {
        int nb = count - b0 < c->max_batch ? count - b0 : c->max_batch;
        int r = decrypt_dev(c, (const u64*)sk, (const u64*)ct + (size_t)b0 * 2 * c->L * c->n, nb,
                            (long long*)out + (size_t)b0 * c->n, 1.0, c->ws, S(s));
        if (r) return r;
    }
    return HELR_OK;
}

__global__ void k_plain_fill(const long long* msg, u64* pt, int n, int L, int nl, Tables tb) {
    const int b = blockIdx.y;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const long long v = msg[(size_t)b * n + i];
        for (int p = 0; p < nl; p++) pt[((size_t)b * L + p) * n + i] = reduce_i64(v, tb.q[p]);
    }
}
extern "C" int helr_encode_plain(helr_ctx* c, const int64_t* msg, uint64_t* pt, int count, int level, void* s) {
    clear_stale_error("helr_encode_plain");
    if (level < 0 || level >= c->L) { set_error("bad level"); return HELR_EINVAL; }
    if (count < 1) return HELR_OK;
    dim3 g(blocks_for(c->n, 256), count);
    k_plain_fill<<<g, 256, 0, S(s)>>>((const long long*)msg, (u64*)pt, c->n, c->L, level + 1, c->t);
    CHECK_KERNEL("plain fill");
    LimbMap m = limb_range(0, level + 1);
    const long long st = (long long)c->L * c->n;
    ntt_buffers<false>(c, (const u64*)pt, st, (u64*)pt, st, m, count, S(s));
    CHECK_LAUNCH("plain ntt");
    return HELR_OK;
}

extern "C" int helr_refresh(helr_ctx* c, const uint64_t* sk, const uint64_t* a, int in_level, double ratio,
                            uint64_t* out, int out_level, int count, uint64_t seed, uint64_t first_id, void* s) {
    clear_stale_error("helr_refresh");
    if (in_level < 0 || in_level >= c->L || out_level < 0 || out_level >= c->L) { set_error("bad level"); return HELR_EINVAL; }
    // workspace: [B][N] u64 scratch + [B][N] int64 message
    const int chunk = c->max_batch;
    for (int b0 = 0; b0 < count; b0 += chunk) {
        int nb = count - b0 < chunk ? count - b0 : chunk;
        u64* tmp = c->ws;
        long long* msg = (long long*)(c->ws + (size_t)chunk * c->n);
        int r = decrypt_dev(c, (const u64*)sk, (const u64*)a + (size_t)b0 * 2 * c->L * c->n, nb, msg, ratio, tmp, S(s));
        if (r) return r;
        r = encrypt_dev(c, (const u64*)sk, msg, (u64*)out + (size_t)b0 * 2 * c->L * c->n, nb, out_level, seed,
                        first_id + (u64)b0, S(s));
        if (r) return r;
    }
    return HELR_OK;
}

// ---------------------------------------------------------------------------
// rescale: out_i = (x_i - NTT_i([INTT_l(x_l)]_centred mod q_i)) * q_l^-1
// (the combine runs in the storer of the last NTT pass, StCombine)
__global__ void k_rescale_conv(const u64* r, u64* t, int n, int l, Tables tb) {
    pdl_begin();
    // r: [items][N] coefficient form mod q_l;  t: [items][l][N]
    const int it = blockIdx.y;
    const u64 ql = tb.q[l], half = ql >> 1;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const u64 v = r[(size_t)it * n + i];
        for (int p = 0; p < l; p++) {
            const u64 q = tb.q[p];
            const u64 m = v > half ? ql - v : v;  // centred magnitude, < q_l
            // q_l < 2q for every chain here (primes of similar size or q_0
            // wider): one conditional subtraction instead of a 64-bit modulo
            const u64 mr = ql <= 2 * q ? (m >= q ? m - q : m) : m % q;
            t[((size_t)it * l + p) * n + i] = v > half ? neg_mod(mr, q) : mr;
        }
    }
}
// polynomial (item, poly) of a strided ciphertext batch, limb `li` offset added by the caller
struct LdPolyLimb {
    const u64* base;   // points at limb l of poly 0 of item 0
    long long item_stride, poly_stride;
    __device__ __forceinline__ u64 operator()(int z, int, int, int off) const {
        return base[(size_t)(z >> 1) * item_stride + (size_t)(z & 1) * poly_stride + off];
    }
};

static int rescale_dev(helr_ctx* c, const u64* a, long long as, u64* out, long long os, int count, int level,
                       cudaStream_t s) {
    const int n = c->n, L = c->L, l = level;
    const int items = 2 * count;  // polynomials
    u64* r = c->ws;                                // [items][N]
    u64* t = c->ws + (size_t)items * n;            // [items][l][N]
    {
        LimbMap m; m.count = 1; m.off[0] = 0; m.prime[0] = (unsigned char)l;
        LdPolyLimb ld{a + (size_t)l * n, as, (long long)L * n};
        StBuf st{r, (long long)n, m, n};
        ntt_launch<true>(c, ld, st, r, n, m, items, s);
        CHECK_LAUNCH("rescale intt");
    }
    dim3 g1(blocks_for(n, 256), items);
    {
        ProfScope ps(PROF_RESCALE, 8.0 * n * items * (1 + l), s);
        launch_pdl(k_rescale_conv, g1, dim3(256), 0, s, (const u64*)r, t, n, l, c->t);
        CHECK_KERNEL("rescale conv");
    }
    // NTT of the converted limbs; the last pass finishes the rescale in its storer
    LimbMap m = limb_range(0, l);
    LdBuf ld{t, (long long)l * n, m, n};
    const StCombine st = st_combine(c, out, os, (long long)L * n, a, as, (long long)L * n, c->qlinv + (size_t)l * L,
                                    c->qlinv_sh + (size_t)l * L, 0);
    ntt_launch<false>(c, ld, st, t, (long long)l * n, m, items, s);
    CHECK_LAUNCH("rescale ntt+final");
    return HELR_OK;
}

int op_rescale(helr_ctx* c, const u64* a, long long as, u64* out, long long os, int count, int level, cudaStream_t s) {
    if (level < 1 || level >= c->L) { set_error("rescale needs level >= 1"); return HELR_EINVAL; }
    const size_t need = (size_t)2 * (level + 1) * c->n;  // per ciphertext (r + t)
    int chunk = (int)(c->ws_words / need);
    if (chunk < 1) { set_error("workspace too small"); return HELR_ENOMEM; }
    for (int b0 = 0; b0 < count; b0 += chunk) {
        int nb = count - b0 < chunk ? count - b0 : chunk;
        int r = rescale_dev(c, a + (size_t)b0 * as, as, out + (size_t)b0 * os, os, nb, level, s);
        if (r) return r;
    }
    return HELR_OK;
}

extern "C" int helr_rescale(helr_ctx* c, const uint64_t* a, uint64_t* out, int count, int level, void* s) {
    clear_stale_error("helr_rescale");
    const long long cs = 2ll * c->L * c->n;
    return op_rescale(c, (const u64*)a, cs, (u64*)out, cs, count, level, S(s));
}

// ---------------------------------------------------------------------------
// ModRaise (bootstrapping step 1): read a ciphertext modulo q_0 and
// re-interpret its centred coefficients modulo q_0..q_level_out.  The result
// encrypts t = m + q_0 I for a small integer polynomial I.
__global__ void k_modraise_conv(const u64* r, u64* out, int n, int L, int nl, Tables tb) {
    pdl_begin();
    // r: [polys][N] coefficient form mod q_0;  out: [polys][L][N], limbs 0..nl-1 written
    const int it = blockIdx.y;
    const u64 q0 = tb.q[0], half = q0 >> 1;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const u64 v = r[(size_t)it * n + i];
        const bool neg = v > half;
        const u64 m = neg ? q0 - v : v;  // centred magnitude
        for (int p = 0; p < nl; p++) {
            const u64 q = tb.q[p];
            const u64 mr = m % q;
            out[((size_t)it * L + p) * n + i] = neg ? neg_mod(mr, q) : mr;
        }
    }
}

extern "C" int helr_mod_raise(helr_ctx* c, const uint64_t* a, uint64_t* out, int count, int level_out, void* sv) {
    clear_stale_error("helr_mod_raise");
    if (level_out < 0 || level_out >= c->L) { set_error("bad level"); return HELR_EINVAL; }
    cudaStream_t s = S(sv);
    const int n = c->n, L = c->L;
    int chunk = (int)(c->ws_words / ((size_t)2 * n));
    if (chunk < 1) { set_error("workspace too small"); return HELR_ENOMEM; }
    for (int b0 = 0; b0 < count; b0 += chunk) {
        const int nb = count - b0 < chunk ? count - b0 : chunk;
        const int items = 2 * nb;  // polynomials
        const u64* ab = (const u64*)a + (size_t)b0 * 2 * L * n;
        u64* ob = (u64*)out + (size_t)b0 * 2 * L * n;
        u64* r = c->ws;  // [items][N]
        {
            LimbMap m; m.count = 1; m.off[0] = 0; m.prime[0] = 0;
            LdPolyLimb ld{ab, 2ll * L * n, (long long)L * n};
            StBuf st{r, (long long)n, m, n};
            ntt_launch<true>(c, ld, st, r, n, m, items, s);
            CHECK_LAUNCH("mod_raise intt");
        }
        dim3 g1(blocks_for(n, 256), items);
        {
            ProfScope ps(PROF_RESCALE, 8.0 * n * items * (2 + level_out), s);
            launch_pdl(k_modraise_conv, g1, dim3(256), 0, s, (const u64*)r, ob, n, L, level_out + 1, c->t);
            CHECK_KERNEL("mod_raise conv");
        }
        LimbMap m = limb_range(0, level_out + 1);
        ntt_buffers<false>(c, ob, (long long)L * n, ob, (long long)L * n, m, items, s);
        CHECK_LAUNCH("mod_raise ntt");
    }
    return HELR_OK;
}

struct LinArgs {
    const u64* x[4];
    long long xs[4];
    const u64* k[4];
    int terms;
};
__global__ void k_lincomb(LinArgs la, u64* out, long long os, int n, int L, Tables tb) {
    pdl_begin();
    const int p = blockIdx.y, it = blockIdx.z;  // it = item*2 + poly
    const int item = it >> 1, poly = it & 1;
    const u64 q = tb.q[p], r1 = tb.br1[p], r0 = tb.br0[p];
    u64* op = out + (size_t)item * os + ((size_t)poly * L + p) * n;
    if (q < NTT_DBL_BOUND) {  // fp64: exact signed products, one canonicalisation
        const DblC dc{tb.qd[p], tb.qinvd[p]};
        double kd[4];
#pragma unroll
        for (int t = 0; t < 4; t++) kd[t] = t < la.terms ? u2d(la.k[t][p]) : 0.0;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            double acc = 0.0;
#pragma unroll
            for (int t = 0; t < 4; t++)
                if (t < la.terms)
                    acc = __dadd_rn(acc, mulmod_d(u2d(la.x[t][(size_t)item * la.xs[t] + ((size_t)poly * L + p) * n + i]),
                                                  kd[t], dc));
            op[i] = d2u_canon(acc, dc);
        }
        return;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        u128v acc{0, 0};
        for (int t = 0; t < la.terms; t++)
            acc_wide(acc, la.x[t][(size_t)item * la.xs[t] + ((size_t)poly * L + p) * n + i], la.k[t][p]);
        op[i] = barrett128(acc, q, r1, r0);
    }
}

int op_lincomb(helr_ctx* c, int terms, const u64* const* x, const long long* xs, const u64* const* k, u64* out,
               long long os, int count, int level, cudaStream_t s) {
    if (terms < 1 || terms > 4) { set_error("lincomb: 1..4 terms"); return HELR_EINVAL; }
    LinArgs la;
    for (int t = 0; t < 4; t++) {
        la.x[t] = t < terms ? x[t] : nullptr;
        la.xs[t] = t < terms ? xs[t] : 0;
        la.k[t] = t < terms ? k[t] : nullptr;
    }
    la.terms = terms;
    dim3 g(blocks_for(c->n, 256), level + 1, 2 * count);
    ProfScope ps(PROF_ELEM, 8.0 * c->n * 2.0 * count * (level + 1) * (terms + 1), s);
    launch_pdl(k_lincomb, g, dim3(256), 0, s, la, out, os, c->n, c->L, c->t);
    CHECK_KERNEL("lincomb");
    return HELR_OK;
}
