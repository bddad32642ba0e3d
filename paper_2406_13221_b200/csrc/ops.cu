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
__device__ __forceinline__ int galois_perm(int i, u64 g, int log_n) {
    const u64 two_n = 2ull << log_n;
    const u64 e = 2ull * (u64)brv_dev(i, log_n) + 1ull;
    const u64 f = (e * g) & (two_n - 1);
    return brv_dev((int)((f - 1) >> 1), log_n);
}

// ---------------------------------------------------------------------------
// elementwise kernels.  Items are ciphertexts (2 polys) unless noted; index
// space: (item, poly, limb, n) flattened with limbs 0..level.
struct EwGeom {
    int n, log_n, L, nl;      // nl = level+1 active limbs
    long long as, bs, os;     // item strides (words) of a, b (ciphertext operands), out
};
__device__ __forceinline__ void ew_decode(long long idx, const EwGeom& g, int& item, int& poly, int& limb, int& k) {
    k = (int)(idx & (g.n - 1));
    long long r = idx >> g.log_n;
    limb = (int)(r % g.nl);
    r /= g.nl;
    poly = (int)(r & 1);
    item = (int)(r >> 1);
}


__global__ void k_elementwise(int op, const u64* a, const u64* b, u64* out, EwGeom g, long long total,
                              Tables tb, const u64* imul_f) {
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        int item, poly, limb, k;
        ew_decode(idx, g, item, poly, limb, k);
        const u64 q = tb.q[limb];
        const size_t in_poly = ((size_t)poly * g.L + limb) * g.n + k;
        const u64 x = a[(size_t)item * g.as + in_poly];
        u64 r;
        switch (op) {
            case EW_ADD: r = add_mod(x, b[(size_t)item * g.bs + in_poly], q); break;
            case EW_SUB: r = sub_mod(x, b[(size_t)item * g.bs + in_poly], q); break;
            case EW_ADDC: r = poly == 0 ? add_mod(x, b[limb], q) : x; break;
            case EW_ADDPT: r = poly == 0 ? add_mod(x, b[(size_t)limb * g.n + k], q) : x; break;
            default: {
                const u64 y = op == EW_MULC ? b[limb] : (op == EW_MULPT ? b[(size_t)limb * g.n + k] : imul_f[(size_t)limb * g.n + k]);
                if (q < NTT_DBL_BOUND) {
                    const DblC dc{tb.qd[limb], tb.qinvd[limb]};
                    r = d2u_canon(mulmod_d(u2d(x), u2d(y), dc), dc);
                } else {
                    r = mul_mod(x, y, q, tb.br1[limb], tb.br0[limb]);
                }
                break;
            }
        }
        out[(size_t)item * g.os + in_poly] = r;
    }
}

int op_ew(helr_ctx* c, int op, const u64* a, long long as, const u64* b, long long bs, u64* out, long long os,
          int count, int level, cudaStream_t s) {
    if (level < 0 || level >= c->L || count < 0) { set_error("bad level/count"); return HELR_EINVAL; }
    if (count == 0) return HELR_OK;
    EwGeom g{c->n, c->log_n, c->L, level + 1, as, bs, os};
    long long total = (long long)count * 2 * (level + 1) * c->n;
    int blocks = blocks_for(total, 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    ProfScope ps(PROF_ELEM, 8.0 * total * ((op == EW_ADD || op == EW_SUB) ? 3 : 2), s);
    k_elementwise<<<blocks, 256, 0, s>>>(op, a, b, out, g, total, c->t, c->imul_f);
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
    const int b = blockIdx.y;
    const u64 key = prng_key(seed, stream_id(ST_CT, first_id + (u64)b, 0, PU_E));
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const long long v = msg[(size_t)b * n + i] + cbd_from(prng_at(key, (u64)i), eta);
        for (int p = 0; p < nl; p++) ct[(size_t)b * 2 * L * n + (size_t)p * n + i] = reduce_i64(v, tb.q[p]);
    }
}
__global__ void k_enc_combine(u64* ct, const u64* sk, int n, int L, u64 seed, u64 first_id, Tables tb) {
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
    k_enc_fill<<<g1, 256, 0, s>>>(ct, msg, c->n, c->L, level + 1, seed, first_id, c->eta, c->t);
    CHECK_KERNEL("encrypt fill");
    LimbMap m = limb_range(0, level + 1);
    const long long st = 2ll * c->L * c->n;
    ntt_buffers<false>(c, ct, st, ct, st, m, count, s);
    CHECK_LAUNCH("encrypt ntt");
    dim3 g2(blocks_for(c->n, 256), level + 1, count);
    k_enc_combine<<<g2, 256, 0, s>>>(ct, sk, c->n, c->L, seed, first_id, c->t);
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
    const int b = blockIdx.y;
    const u64 q = tb.q[0], r1 = tb.br1[0], r0 = tb.br0[0];
    const u64* c0 = ct + (size_t)b * 2 * L * n;
    const u64* c1 = c0 + (size_t)L * n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        v[(size_t)b * n + i] = add_mod(c0[i], mul_mod(c1[i], sk[i], q, r1, r0), q);
}
__global__ void k_center(const u64* v, long long* out, long long total, double ratio, Tables tb) {
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
    k_dec_combine<<<g, 256, 0, s>>>(ct, sk, tmp, c->n, c->L, c->t);
    CHECK_KERNEL("decrypt combine");
    LimbMap m = limb_range(0, 1);
    ntt_buffers<true>(c, tmp, c->n, tmp, c->n, m, count, s);
    CHECK_LAUNCH("decrypt intt");
    long long total = (long long)count * c->n;
    k_center<<<blocks_for(total, 256) < 4096 ? blocks_for(total, 256) : 4096, 256, 0, s>>>(tmp, out, total, ratio, c->t);
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

// Last-NTT-pass storer that finishes a ModDown / rescale in place of a
// separate combine kernel: out = (x - v) * w_p mod q [+ add_a] [+ sum_t
// sigma_t(add_p) on poly 0], v being the NTT output.  Index decoding:
// per_poly > 0: item = z, li = poly * per_poly + p;  per_poly == 0:
// item = z >> 1, poly = z & 1, p = li.
struct StCombine {
    static constexpr bool kVec = true;
    static constexpr bool kTile = true;
    u64* out;
    long long out_is, out_ps;
    const u64* x;
    long long x_is, x_ps;
    const u64* w;
    const u64* wsh;
    const u64* q;
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
            for (int t = 0; t < ngal; t++) {
                const int src = galois_perm(off, (u64)gal[t], log_n);
                const ulonglong2 pr = ld2(pp + (src & ~1));
                r0 = add_mod(r0, (src & 1) ? pr.y : pr.x, qq);
                r1 = add_mod(r1, (src & 1) ? pr.x : pr.y, qq);
            }
        }
        st2(out + (size_t)item * out_is + (size_t)poly * out_ps + (size_t)p * n + off, r0, r1);
    }
};
static StCombine st_combine(const helr_ctx* c, u64* out, long long out_is, long long out_ps, const u64* x, long long x_is,
                            long long x_ps, const u64* w, const u64* wsh, int per_poly) {
    StCombine f;
    f.out = out; f.out_is = out_is; f.out_ps = out_ps;
    f.x = x; f.x_is = x_is; f.x_ps = x_ps;
    f.w = w; f.wsh = wsh; f.q = c->t.q;
    f.add_a = nullptr; f.a_is = f.a_ps = 0;
    f.add_p = nullptr; f.p_is = 0;
    f.ngal = 0; f.log_n = c->log_n; f.n = c->n; f.per_poly = per_poly;
    for (int t = 0; t < HELR_MAX_HOIST; t++) f.gal[t] = 1;
    return f;
}

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
        k_rescale_conv<<<g1, 256, 0, s>>>(r, t, n, l, c->t);
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
            if (a.galois) {
                const u64* dp = d + (size_t)p * a.n;
                st2(ext + (size_t)p * a.n + i, dp[galois_perm(i, (u64)a.galois, a.log_n)],
                    dp[galois_perm(i + 1, (u64)a.galois, a.log_n)]);
            } else {
                *reinterpret_cast<ulonglong2*>(ext + (size_t)p * a.n + i) = ld2(d + (size_t)p * a.n + i);
            }
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
            st2(ext + (size_t)e * a.n + i, d2u_canon(s0, dc), d2u_canon(s1, dc));
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
__device__ __forceinline__ u128acc dresolve(const dacc& a) {  // hh 2^42 + mid 2^21 + ll
    const u64 H = dexact(a.hh), M = dexact(a.mid), Lo = dexact(a.ll);
    u128acc r{H << 42, H >> 22};
    const u64 m_lo = M << 21, m_hi = M >> 43;
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(r.lo), "+l"(r.hi) : "l"(m_lo), "l"(m_hi));
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, 0;" : "+l"(r.lo), "+l"(r.hi) : "l"(Lo));
    return r;
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
            split21(u.x, uxh, uxl); split21(u.y, uyh, uyl);
            split21(k0.x, k0xh, k0xl); split21(k0.y, k0yh, k0yl);
            split21(k1.x, k1xh, k1xl); split21(k1.y, k1yh, k1yl);
            mac_d(c00, uxh, uxl, k0xh, k0xl);
            mac_d(c01, uyh, uyl, k0yh, k0yl);
            mac_d(c10, uxh, uxl, k1xh, k1xl);
            mac_d(c11, uyh, uyl, k1yh, k1yl);
        }
        o00 = reduce128(dresolve(c00), q, r1, r0, one_sh[p]);
        o01 = reduce128(dresolve(c01), q, r1, r0, one_sh[p]);
        o10 = reduce128(dresolve(c10), q, r1, r0, one_sh[p]);
        o11 = reduce128(dresolve(c11), q, r1, r0, one_sh[p]);
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
            z0[k] = shoup(x.x, phinv[k], phinv_sh[k], pk);
            z1[k] = shoup(x.y, phinv[k], phinv_sh[k], pk);
            v0 = __dadd_rn(v0, __dmul_rn(__ull2double_rn(z0[k]), inv));
            v1 = __dadd_rn(v1, __dmul_rn(__ull2double_rn(z1[k]), inv));
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
            st2(mp + (size_t)p * n + i, d2u_canon(s0, dc), d2u_canon(s1, dc));
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

// workspace carve-up for key switching of B items at level l
struct KsWs {
    u64 *coef, *ext, *acc, *mdc, *tensor;
    long long coef_s, ext_s, ext_ds, acc_s, mdc_s;
};
static KsWs ks_ws(helr_ctx* c, int B) {
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
        if (c->alpha <= 4) k_modup<4><<<g, 128, 0, s>>>(a, c->t);
        else if (c->alpha <= 8) k_modup<8><<<g, 128, 0, s>>>(a, c->t);
        else k_modup<HELR_MAXP><<<g, 128, 0, s>>>(a, c->t);
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
                    ntt_buffers<false>(c, w.ext, w.ext_s, w.ext, w.ext_s, m, B, s);
                    m.count = 0;
                }
            }
        }
        if (m.count) ntt_buffers<false>(c, w.ext, w.ext_s, w.ext, w.ext_s, m, B, s);
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
        auto conv = K <= 4 ? k_moddown_conv<4> : (K <= 8 ? k_moddown_conv<8> : k_moddown_conv<HELR_MAXP>);
        conv<<<g, 128, 0, s>>>(w.acc, w.acc_s, w.mdc, w.mdc_s, n, nl, K, L, c->md_phinv, c->md_phinv_sh, c->md_phmod,
                               c->md_phmod_sh, c->md_pinv_dbl, c->pmod, c->pmod_sh, c->t);
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
        ntt_launch<false>(c, ld, st, w.mdc, w.mdc_s, mq, B, s);
        CHECK_LAUNCH("ks moddown ntt+final");
    }
    return HELR_OK;
}

struct HoistKeys {
    int nsteps;
    const u64* key[HELR_MAX_HOIST];
    long long gal[HELR_MAX_HOIST];
};
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
    k_ks_inner<<<g, dim3(64, by), 0, s>>>(w.ext, w.ext_s, w.ext_ds, evk, w.acc, w.acc_s, n, nl, K, L, c->LK, nd, B,
                                          c->t, dadd, dadd_is, c->pmod, c->pmod_sh, c->one_sh);
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
            z0[k] = shoup(x.x, mt.hv[k], mt.hvs[k], m);
            z1[k] = shoup(x.y, mt.hv[k], mt.hvs[k], m);
            v0 = __dadd_rn(v0, __dmul_rn(__ull2double_rn(z0[k]), inv));
            v1 = __dadd_rn(v1, __dmul_rn(__ull2double_rn(z1[k]), inv));
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
            st2(mp + (size_t)p * n + i, d2u_canon(s0, dc), d2u_canon(s1, dc));
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
        auto conv = K + 1 <= 4 ? k_mdr_conv<4> : (K + 1 <= 8 ? k_mdr_conv<8> : k_mdr_conv<HELR_MAXP>);
        conv<<<g, 128, 0, s>>>(w.acc, w.acc_s, w.mdc, w.mdc_s, n, nl, K, L, mt, c->t);
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
        ntt_launch<false>(c, ld, st, w.mdc, w.mdc_s, mq, B, s);
        CHECK_LAUNCH("mdr ntt+final");
    }
    return HELR_OK;
}

// ---- hoisted rotate-and-sum ------------------------------------------------
// out = [a +] sum_t rot_{g_t}(a): ONE ModUp of c1, the inner products of every
// rotation summed in the extended basis (sigma_t applied to the ModUp'd digits
// by a warp-coalesced gather: a Galois permutation maps every 32-aligned run of
// NTT slots onto a 32-aligned run), ONE ModDown; sum_t sigma_t(c0) is gathered
// in the ModDown epilogue.
// One thread per (coefficient i, extended limb e) carries the accumulators of
// up to NB ciphertexts, so each key word is loaded once per launch chunk and
// reused NB times from a register, and every step issues 2 nd + NB nd
// independent loads (memory-level parallelism without high occupancy).
// Accumulation is 128-bit: every product is < 2^122 (all primes < 2^61), so
// up to 63 products fit; longer sums fold to a residue every `fold` steps
// (host-computed from the largest prime, see hoist_fold).
// Per-thread asynchronous prefetch: every thread copies the key words and
// permuted ext words of rotation step t + S - 1 into its own shared-memory
// slots (cp.async, 8 bytes each) while it multiplies step t, so the gathers'
// latency overlaps the arithmetic without holding them in registers.  Each
// slot is written and read by the same thread, so cp.async.wait_group alone
// orders them (no block barrier).
__device__ __forceinline__ void cp_async8(u64* dst, const u64* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

constexpr int HOIST_T = 128;     // threads per block (coefficients per tile)
constexpr int HOIST_STAGES = 3;  // steps in flight per thread


// grid: x = coefficient tile * chunks + chunk (chunks of NB ciphertexts share
// the tile's key words through L2 at the same time), y = extended limb e.
// Kernel arguments of the key inner product (hoisted or single key).
struct HoistArgs {
    const u64* ext;
    long long ext_item_stride, ext_digit_stride;
    u64* acc;
    long long acc_item_stride;
    int n, log_n, nl, K, L, LK, B, nchunks, fold;
    const u64* one_sh;
    const u64* dadd;  // optional [B][3][L][N] tensor: Q limbs also get (P mod q) * (d0, d1)
    long long dadd_is;
    const u64* pm;
    const u64* pm_sh;
};

template <int ND, int NB, bool DBL>
__device__ __forceinline__ void hoist_body(const HoistKeys& hk, const HoistArgs& A, const Tables& tb) {
    const u64* __restrict__ ext = A.ext;
    const long long ext_item_stride = A.ext_item_stride, ext_digit_stride = A.ext_digit_stride;
    u64* acc = A.acc;
    const long long acc_item_stride = A.acc_item_stride;
    const int n = A.n, log_n = A.log_n, nl = A.nl, K = A.K, L = A.L, LK = A.LK, B = A.B, nchunks = A.nchunks,
              fold = A.fold;
    const u64* one_sh = A.one_sh;
    constexpr int W = (2 + NB) * ND;  // words per thread per stage
    constexpr int S = HOIST_STAGES;
    extern __shared__ u64 hsm[];
    const int tid = threadIdx.x;
    const int e = blockIdx.y;
    const int tile = blockIdx.x / nchunks, chunk = blockIdx.x - tile * nchunks;
    const int i = tile * HOIST_T + tid;
    const int b0 = chunk * NB;
    if (i >= n) return;
    const int p = e < nl ? e : L + (e - nl);
    const u64 q = tb.q[p], r1 = tb.br1[p], r0 = tb.br0[p], osh = one_sh[p];
    const int nb = B - b0 < NB ? B - b0 : NB;
    const u64* xb = ext + (size_t)b0 * ext_item_stride + (size_t)e * n;
    const size_t k0off = ((size_t)p) * n + i;
    const size_t k1off = ((size_t)LK + p) * n + i;
    const size_t kds = (size_t)2 * LK * n;
    auto slot = [&](int stage, int w) -> u64* { return hsm + ((size_t)(stage * W + w) * HOIST_T + tid); };
    auto issue = [&](int t) {
        if (t < hk.nsteps) {
            const int stage = t % S;
            const int src = galois_perm(i, (u64)hk.gal[t], log_n);
            const u64* kt = hk.key[t];
#pragma unroll
            for (int j = 0; j < ND; j++) {
                cp_async8(slot(stage, j), kt + (size_t)j * kds + k0off);
                cp_async8(slot(stage, ND + j), kt + (size_t)j * kds + k1off);
            }
#pragma unroll
            for (int b = 0; b < NB; b++) {
                if (b < nb) {
#pragma unroll
                    for (int j = 0; j < ND; j++)
                        cp_async8(slot(stage, 2 * ND + b * ND + j),
                                  xb + (size_t)b * ext_item_stride + (size_t)j * ext_digit_stride + src);
                }
            }
        }
        cp_async_commit();  // empty groups keep the wait count uniform
    };
    using Acc = typename std::conditional<DBL, dacc, macc>::type;
    Acc a0[NB], a1[NB];
#pragma unroll
    for (int b = 0; b < NB; b++) {
        if constexpr (DBL) a0[b] = a1[b] = dacc{0.0, 0.0, 0.0};
        else a0[b] = a1[b] = macc{0, 0, 0, 0};
    }
#pragma unroll
    for (int t = 0; t < S - 1; t++) issue(t);
    int run = 0;
    for (int t = 0; t < hk.nsteps; t++) {
        issue(t + S - 1);
        cp_async_wait<S - 1>();
        const int stage = t % S;
        if constexpr (DBL) {
            double k0h[ND], k0l[ND], k1h[ND], k1l[ND];
#pragma unroll
            for (int j = 0; j < ND; j++) {
                split21(*slot(stage, j), k0h[j], k0l[j]);
                split21(*slot(stage, ND + j), k1h[j], k1l[j]);
            }
#pragma unroll
            for (int b = 0; b < NB; b++) {
                if (b < nb) {
#pragma unroll
                    for (int j = 0; j < ND; j++) {
                        double uh, ul;
                        split21(*slot(stage, 2 * ND + b * ND + j), uh, ul);
                        mac_d(a0[b], uh, ul, k0h[j], k0l[j]);
                        mac_d(a1[b], uh, ul, k1h[j], k1l[j]);
                    }
                }
            }
        } else {
            if (run == fold) {  // fold into a residue before the 128-bit sum can overflow
#pragma unroll
                for (int b = 0; b < NB; b++) {
                    a0[b] = macc{reduce128(resolve(a0[b]), q, r1, r0, osh), 0, 0, 0};
                    a1[b] = macc{reduce128(resolve(a1[b]), q, r1, r0, osh), 0, 0, 0};
                }
                run = 0;
            }
            run++;
            u64 k0[ND], k1[ND];
#pragma unroll
            for (int j = 0; j < ND; j++) {
                k0[j] = *slot(stage, j);
                k1[j] = *slot(stage, ND + j);
            }
#pragma unroll
            for (int b = 0; b < NB; b++) {
                if (b < nb) {
#pragma unroll
                    for (int j = 0; j < ND; j++) {
                        const u64 u = *slot(stage, 2 * ND + b * ND + j);
                        mac_split(a0[b], u, k0[j]);
                        mac_split(a1[b], u, k1[j]);
                    }
                }
            }
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int b = 0; b < NB; b++) {
        if (b < nb) {
            u64* ap = acc + (size_t)(b0 + b) * acc_item_stride;
            u64 o0, o1;
            if constexpr (DBL) {
                o0 = reduce128(dresolve(a0[b]), q, r1, r0, osh);
                o1 = reduce128(dresolve(a1[b]), q, r1, r0, osh);
            } else {
                o0 = reduce128(resolve(a0[b]), q, r1, r0, osh);
                o1 = reduce128(resolve(a1[b]), q, r1, r0, osh);
            }
            if (A.dadd && e < nl) {  // merged ModDown + rescale: + (P mod q) * (d0, d1)
                const u64* db = A.dadd + (size_t)(b0 + b) * A.dadd_is + (size_t)e * n + i;
                const u64 w = A.pm[e], ws = A.pm_sh[e];
                o0 = add_mod(o0, shoup(db[0], w, ws, q), q);
                o1 = add_mod(o1, shoup(db[(size_t)L * n], w, ws, q), q);
            }
            ap[(size_t)e * n + i] = o0;
            ap[((size_t)(nl + K) + e) * n + i] = o1;
        }
    }
}

template <int ND, int NB>
__global__ void __launch_bounds__(HOIST_T, 3) k_ks_inner_hoisted(HoistKeys hk, HoistArgs A, Tables tb) {
    const int e = blockIdx.y;
    const int p = e < A.nl ? e : A.L + (e - A.nl);
    if (tb.q[p] < NTT_DBL_BOUND)  // uniform per CTA (one limb per CTA)
        hoist_body<ND, NB, true>(hk, A, tb);
    else
        hoist_body<ND, NB, false>(hk, A, tb);
}

// Steps per 128-bit accumulation run: a run adds fold*nd products (each <
// 2^(2 bits)) to a residue (< 2^bits) and must stay below 2^128.
static int hoist_fold(const helr_ctx* c, int nd) {
    int bits = 0;
    for (u64 q : c->primes) {
        int b = 64 - __builtin_clzll(q);
        if (b > bits) bits = b;
    }
    const int room = 128 - 2 * bits;  // 2^room products fit, less one for the residue
    const long long terms = room >= 20 ? (1ll << 20) : (1ll << room) - 1;
    const long long f = terms / nd;
    return f < 1 ? 1 : (f > (1 << 20) ? (1 << 20) : (int)f);
}

template <int ND, int NB>
static void launch_hoisted_nb(dim3 g, cudaStream_t s, const HoistKeys& hk, HoistArgs A, const Tables& tb) {
    A.nchunks = (A.B + NB - 1) / NB;
    const size_t smem = sizeof(u64) * (size_t)HOIST_STAGES * (2 + NB) * ND * HOIST_T;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_ks_inner_hoisted<ND, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    g.x *= A.nchunks;
    k_ks_inner_hoisted<ND, NB><<<g, HOIST_T, smem, s>>>(hk, A, tb);
}
// ciphertexts per thread: HELR_HOIST_NB (1, 2, 4 or 8; default 4) caps it
static int hoist_nb_cap() {
    static int cap = -1;
    if (cap < 0) {
        const char* v = getenv("HELR_HOIST_NB");
        cap = v ? atoi(v) : 4;
        if (cap != 1 && cap != 2 && cap != 8) cap = 4;
    }
    return cap;
}
template <int ND>
static void launch_hoisted(dim3 g, cudaStream_t s, const HoistKeys& hk, const HoistArgs& A, const Tables& tb) {
    const int nb = A.B;
    const int cap = hoist_nb_cap();
    const int want = nb <= 1 ? 1 : nb <= 2 ? 2 : nb <= 4 ? 4 : 8;
    const int NBs = want < cap ? want : cap;
    if (NBs == 1) launch_hoisted_nb<ND, 1>(g, s, hk, A, tb);
    else if (NBs == 2) launch_hoisted_nb<ND, 2>(g, s, hk, A, tb);
    else if (NBs == 4) launch_hoisted_nb<ND, 4>(g, s, hk, A, tb);
    else if constexpr (ND <= 3) launch_hoisted_nb<ND, 8>(g, s, hk, A, tb);
    else launch_hoisted_nb<ND, 4>(g, s, hk, A, tb);
}

// Key inner product of the ModUp'd digits in w.ext with hk's keys (summed over
// hk.nsteps Galois steps) into w.acc; dadd (optional) adds (P mod q)(d0, d1).
static int key_inner(helr_ctx* c, const KsWs& w, const HoistKeys& hk, int nb, int level, const u64* dadd,
                     long long dadd_is, cudaStream_t s) {
    const int n = c->n, nl = level + 1, K = c->K, ne = nl + K;
    const int nd = (nl + c->alpha - 1) / c->alpha;
    dim3 g(blocks_for(n, HOIST_T), ne, 1);
    HoistArgs A{w.ext, w.ext_s, w.ext_ds, w.acc, w.acc_s, n, c->log_n, nl, K, c->L, c->LK, nb, 1, hoist_fold(c, nd),
                c->one_sh, dadd, dadd_is, c->pmod, c->pmod_sh};
    ProfScope ps(PROF_INNER, 8.0 * n * ((double)nb * nd * ne * hk.nsteps + 2.0 * nd * ne * hk.nsteps + 2.0 * nb * ne +
                                        (dadd ? 2.0 * nb * nl : 0.0)), s);
    switch (nd) {
        case 1: launch_hoisted<1>(g, s, hk, A, c->t); break;
        case 2: launch_hoisted<2>(g, s, hk, A, c->t); break;
        case 3: launch_hoisted<3>(g, s, hk, A, c->t); break;
        case 4: launch_hoisted<4>(g, s, hk, A, c->t); break;
        case 5: launch_hoisted<5>(g, s, hk, A, c->t); break;
        case 6: launch_hoisted<6>(g, s, hk, A, c->t); break;
        case 7: launch_hoisted<7>(g, s, hk, A, c->t); break;
        case 8: launch_hoisted<8>(g, s, hk, A, c->t); break;
        default: set_error("key switching: more than 8 digits"); return HELR_EINVAL;
    }
    CHECK_KERNEL("key inner product");
    return HELR_OK;
}

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
            k_tensor<<<g, 256, 0, s>>>(ta, w.tensor, c->n, c->L, c->t);
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
            k_tensor<<<g, 256, 0, s>>>(ta, w.tensor, n, L, c->t);
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
struct LinArgs {
    const u64* x[4];
    long long xs[4];
    const u64* k[4];
    int terms;
};
__global__ void k_lincomb(LinArgs la, u64* out, long long os, int n, int L, Tables tb) {
    const int p = blockIdx.y, it = blockIdx.z;  // it = item*2 + poly
    const int item = it >> 1, poly = it & 1;
    const u64 q = tb.q[p], r1 = tb.br1[p], r0 = tb.br0[p];
    u64* op = out + (size_t)item * os + ((size_t)poly * L + p) * n;
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
    k_lincomb<<<g, 256, 0, s>>>(la, out, os, c->n, c->L, c->t);
    CHECK_KERNEL("lincomb");
    return HELR_OK;
}
