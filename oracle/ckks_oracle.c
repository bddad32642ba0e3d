/*
 * ckks_oracle.c — CPU RNS-CKKS oracle.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the timed CPU baseline.  The product path (paper_2406_13221_b200) never
 * links or calls it.
 *
 * What it restates.  The reference (pkg/src/helr/hesim.py) only simulates
 * ciphertexts as complex slot vectors; it has no ring arithmetic, so ring
 * parity is pinned here by known-answer tests instead (tests/test_oracle_*:
 * NTT vs big-int schoolbook negacyclic products, rescale/ModUp/ModDown vs
 * big-int CRT formulas, decrypt(rotate) == np.roll as in hesim.py:218-226).
 * The algorithms are the textbook ones, written as plain loops with
 * unsigned __int128 arithmetic and no lazy reduction, deliberately unlike
 * the device kernels:
 *   - negacyclic NTT, Cooley-Tukey forward / Gentleman-Sande inverse with
 *     bit-reversed powers of psi (output slot i = a(psi^(2 brv(i) + 1)));
 *   - hybrid key switching: digits of alpha limbs, approximate fast basis
 *     conversion (ModUp), inner product with the key, ModDown by P;
 *   - rescale by the top prime with a centred remainder;
 *   - symmetric encryption with a counter-based generator (SplitMix64
 *     finaliser), uniform residues from 128 random bits, centred-binomial
 *     errors; ternary secret.
 * Mapping to the reference evaluator: enc/dec hesim.py:146-162, add 166-175,
 * cadd 177-184, mul 186-195, cmul 197-206, imul 208-216, rotate 218-226,
 * bootstrap (refresh stand-in) 228-236.
 *
 * Ciphertext layout: u64[2][L][N]; secret key u64[L+K][N] (NTT);
 * switching key u64[beta][2][L+K][N].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;
typedef uint64_t u64;

#define MAXP 64

typedef struct {
    int log_n, n, L, K, dnum, alpha, beta, eta;
    u64 prm[MAXP];
    u64 psi[MAXP];
    u64 ninv[MAXP];
    u64* tw;   /* [L+K][N] psi^brv(k) */
    u64* itw;  /* [L+K][N] psi^-brv(k) */
} oc_ctx;

static u64 mulm(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static u64 addm(u64 a, u64 b, u64 q) { u64 s = a + b; return s >= q ? s - q : s; }
static u64 subm(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
static u64 powm(u64 b, u64 e, u64 q) {
    u64 r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = mulm(r, b, q);
        b = mulm(b, b, q);
        e >>= 1;
    }
    return r;
}
static u64 invm(u64 a, u64 q) { return powm(a, q - 2, q); }
static u64 red_i64(int64_t v, u64 q) {
    if (v >= 0) return (u64)v % q;
    u64 m = (u64)(-(v + 1)) % q; /* -(v+1) >= 0 */
    return q - 1 - m;
}
static unsigned brv(unsigned x, int bits) {
    unsigned r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* ---------------- counter-based randomness (shared spec) ---------------- */
static u64 mix64(u64 z) {
    z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27; z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
}
u64 oc_prng(u64 seed, u64 stream, u64 ctr) {
    u64 key = mix64(seed ^ mix64(stream + 0x9E3779B97F4A7C15ULL));
    return mix64(key + (ctr + 1) * 0x9E3779B97F4A7C15ULL);
}
/* stream ids: kind<<56 | id<<8 | sub<<4 | purpose */
#define ST_SK 1ULL
#define ST_CT 2ULL
#define ST_KEY 3ULL
#define PU_A 1ULL
#define PU_E 2ULL
#define PU_S 3ULL
static u64 stream_id(u64 kind, u64 id, u64 sub, u64 purpose) {
    return (kind << 56) ^ (id << 8) ^ (sub << 4) ^ purpose;
}
static u64 uniform_mod(u64 seed, u64 stream, u64 idx, u64 q) {
    u64 lo = oc_prng(seed, stream, 2 * idx);
    u64 hi = oc_prng(seed, stream, 2 * idx + 1);
    return (u64)((((u128)hi << 64) | lo) % q);
}
static int64_t cbd(u64 seed, u64 stream, u64 idx, int eta) {
    u64 r = oc_prng(seed, stream, idx);
    u64 mask = (eta >= 32) ? 0xffffffffULL : ((1ULL << eta) - 1);
    return (int64_t)__builtin_popcountll(r & mask) - (int64_t)__builtin_popcountll((r >> 32) & mask);
}

/* ---------------- context ---------------- */
oc_ctx* oc_create(int log_n, int L, int K, int dnum, const u64* primes, const u64* psi, int eta) {
    if (L + K > MAXP || log_n < 2 || log_n > 17) return NULL;
    oc_ctx* c = (oc_ctx*)calloc(1, sizeof(oc_ctx));
    c->log_n = log_n; c->n = 1 << log_n; c->L = L; c->K = K; c->dnum = dnum; c->eta = eta;
    c->alpha = (L + dnum - 1) / dnum;
    c->beta = (L + c->alpha - 1) / c->alpha;
    int N = c->n;
    c->tw = (u64*)malloc(sizeof(u64) * (size_t)(L + K) * N);
    c->itw = (u64*)malloc(sizeof(u64) * (size_t)(L + K) * N);
    for (int p = 0; p < L + K; p++) {
        u64 q = primes[p];
        c->prm[p] = q; c->psi[p] = psi[p];
        c->ninv[p] = invm((u64)N, q);
        u64 ip = invm(psi[p], q);
        for (int k = 0; k < N; k++) {
            unsigned e = brv((unsigned)k, log_n);
            c->tw[(size_t)p * N + k] = powm(psi[p], e, q);
            c->itw[(size_t)p * N + k] = powm(ip, e, q);
        }
    }
    return c;
}
void oc_destroy(oc_ctx* c) {
    if (!c) return;
    free(c->tw); free(c->itw); free(c);
}
int oc_beta(oc_ctx* c) { return c->beta; }
int oc_alpha(oc_ctx* c) { return c->alpha; }

/* ---------------- NTT ---------------- */
void oc_ntt(oc_ctx* c, u64* a, int p) {
    int N = c->n; u64 q = c->prm[p];
    const u64* W = c->tw + (size_t)p * N;
    int t = N;
    for (int m = 1; m < N; m <<= 1) {
        t >>= 1;
        for (int i = 0; i < m; i++) {
            u64 w = W[m + i];
            int j1 = 2 * i * t;
            for (int j = j1; j < j1 + t; j++) {
                u64 u = a[j], v = mulm(a[j + t], w, q);
                a[j] = addm(u, v, q);
                a[j + t] = subm(u, v, q);
            }
        }
    }
}
void oc_intt(oc_ctx* c, u64* a, int p) {
    int N = c->n; u64 q = c->prm[p];
    const u64* W = c->itw + (size_t)p * N;
    int t = 1;
    for (int m = N >> 1; m >= 1; m >>= 1) {
        int j1 = 0;
        for (int i = 0; i < m; i++) {
            u64 w = W[m + i];
            for (int j = j1; j < j1 + t; j++) {
                u64 u = a[j], v = a[j + t];
                a[j] = addm(u, v, q);
                a[j + t] = mulm(subm(u, v, q), w, q);
            }
            j1 += 2 * t;
        }
        t <<= 1;
    }
    for (int j = 0; j < N; j++) a[j] = mulm(a[j], c->ninv[p], q);
}

/* batch helpers: data[b*stride + i*N], primes first..first+n_limbs-1 */
void oc_ntt_batch(oc_ctx* c, u64* data, int first, int n_limbs, int count, int64_t stride, int inverse) {
    int tot = n_limbs * count;
#pragma omp parallel for schedule(dynamic)
    for (int x = 0; x < tot; x++) {
        int b = x / n_limbs, i = x % n_limbs;
        u64* a = data + (size_t)b * stride + (size_t)i * c->n;
        if (inverse) oc_intt(c, a, first + i); else oc_ntt(c, a, first + i);
    }
}

/* NTT-domain automorphism X -> X^g: out[i] = in[j], 2brv(j)+1 = g(2brv(i)+1) mod 2N */
static void automorph_poly(oc_ctx* c, const u64* in, u64* out, u64 g) {
    int N = c->n, lg = c->log_n;
    u64 two_n = 2 * (u64)N;
    for (int i = 0; i < N; i++) {
        u64 e = 2 * (u64)brv((unsigned)i, lg) + 1;
        u64 f = (e * (g % two_n)) % two_n;
        unsigned j = brv((unsigned)((f - 1) / 2), lg);
        out[i] = in[j];
    }
}

/* ---------------- keys ---------------- */
/* Secret coefficients.  hw == 0: uniform ternary.  hw > 0: exactly hw
 * nonzero +-1 entries (HEAAN's sparse secret): the hw positions with the
 * smallest prng(seed, SK/0, i) (ties broken by index), sign from bit 0 of
 * prng(seed, SK/1, i).  Host-side client key generation, same rule on device. */
typedef struct { u64 r; int i; } rank_t;
static int rank_cmp(const void* a, const void* b) {
    const rank_t *x = (const rank_t*)a, *y = (const rank_t*)b;
    if (x->r != y->r) return x->r < y->r ? -1 : 1;
    return x->i - y->i;
}
void oc_secret_coeffs(u64 seed, int N, int hw, int64_t* s) {
    u64 st = stream_id(ST_SK, 0, 0, PU_S);
    if (hw <= 0) {
        for (int i = 0; i < N; i++) s[i] = (int64_t)(oc_prng(seed, st, (u64)i) % 3) - 1;
        return;
    }
    rank_t* rk = (rank_t*)malloc(sizeof(rank_t) * N);
    for (int i = 0; i < N; i++) { rk[i].r = oc_prng(seed, st, (u64)i); rk[i].i = i; }
    qsort(rk, N, sizeof(rank_t), rank_cmp);
    u64 sg = stream_id(ST_SK, 0, 1, PU_S);
    for (int i = 0; i < N; i++) s[i] = 0;
    for (int k = 0; k < hw && k < N; k++) {
        int i = rk[k].i;
        s[i] = (oc_prng(seed, sg, (u64)i) & 1) ? 1 : -1;
    }
    free(rk);
}

void oc_keygen_secret_hw(oc_ctx* c, u64 seed, int hw, u64* sk) {
    int N = c->n;
    int64_t* s = (int64_t*)malloc(sizeof(int64_t) * N);
    oc_secret_coeffs(seed, N, hw, s);
#pragma omp parallel for
    for (int p = 0; p < c->L + c->K; p++) {
        u64* d = sk + (size_t)p * N;
        for (int i = 0; i < N; i++) d[i] = red_i64(s[i], c->prm[p]);
        oc_ntt(c, d, p);
    }
    free(s);
}
void oc_keygen_secret(oc_ctx* c, u64 seed, u64* sk) { oc_keygen_secret_hw(c, seed, 0, sk); }

/* P mod q_i for i < L */
static u64 pmod(oc_ctx* c, int i) {
    u64 q = c->prm[i], r = 1;
    for (int k = 0; k < c->K; k++) r = mulm(r, c->prm[c->L + k] % q, q);
    return r;
}

void oc_keygen_switch(oc_ctx* c, const u64* sk, int64_t galois, u64* evk, u64 seed, u64 key_id) {
    int N = c->n, LK = c->L + c->K;
    u64* sp = (u64*)malloc(sizeof(u64) * (size_t)LK * N);
    for (int p = 0; p < LK; p++) {
        const u64* s = sk + (size_t)p * N;
        u64* d = sp + (size_t)p * N;
        if (galois == 0) {
            for (int i = 0; i < N; i++) d[i] = mulm(s[i], s[i], c->prm[p]);
        } else {
            automorph_poly(c, s, d, (u64)galois);
        }
    }
    for (int j = 0; j < c->beta; j++) {
        u64 sa = stream_id(ST_KEY, key_id, (u64)j, PU_A);
        u64 se = stream_id(ST_KEY, key_id, (u64)j, PU_E);
        int64_t* e = (int64_t*)malloc(sizeof(int64_t) * N);
        for (int i = 0; i < N; i++) e[i] = cbd(seed, se, (u64)i, c->eta);
#pragma omp parallel for
        for (int p = 0; p < LK; p++) {
            u64 q = c->prm[p];
            u64* b0 = evk + ((size_t)(j * 2 + 0) * LK + p) * N;
            u64* b1 = evk + ((size_t)(j * 2 + 1) * LK + p) * N;
            const u64* s = sk + (size_t)p * N;
            for (int i = 0; i < N; i++) b1[i] = uniform_mod(seed, sa, (u64)p * N + i, q);
            for (int i = 0; i < N; i++) b0[i] = red_i64(e[i], q);
            oc_ntt(c, b0, p);
            int in_digit = (p < c->L) && (p / c->alpha == j);
            u64 f = in_digit ? pmod(c, p) : 0;
            for (int i = 0; i < N; i++) {
                u64 v = subm(b0[i], mulm(b1[i], s[i], q), q);
                if (in_digit) v = addm(v, mulm(f, sp[(size_t)p * N + i], q), q);
                b0[i] = v;
            }
        }
        free(e);
    }
    free(sp);
}

/* ---------------- encryption ---------------- */
static void encrypt_one(oc_ctx* c, const u64* sk, u64 seed, u64 ct_id, int level, const int64_t* m, u64* ct) {
    int N = c->n, L = c->L;
    u64 sa = stream_id(ST_CT, ct_id, 0, PU_A);
    u64 se = stream_id(ST_CT, ct_id, 0, PU_E);
    int64_t* me = (int64_t*)malloc(sizeof(int64_t) * N);
    for (int i = 0; i < N; i++) me[i] = m[i] + cbd(seed, se, (u64)i, c->eta);
    for (int p = 0; p <= level; p++) {
        u64 q = c->prm[p];
        u64* c0 = ct + (size_t)p * N;
        u64* c1 = ct + ((size_t)L + p) * N;
        const u64* s = sk + (size_t)p * N;
        for (int i = 0; i < N; i++) c1[i] = uniform_mod(seed, sa, (u64)p * N + i, q);
        for (int i = 0; i < N; i++) c0[i] = red_i64(me[i], q);
        oc_ntt(c, c0, p);
        for (int i = 0; i < N; i++) c0[i] = subm(c0[i], mulm(c1[i], s[i], q), q);
    }
    free(me);
}
void oc_encrypt(oc_ctx* c, const u64* sk, const int64_t* msg, u64* ct, int count, int level, u64 seed, u64 first_id) {
#pragma omp parallel for schedule(dynamic)
    for (int b = 0; b < count; b++)
        encrypt_one(c, sk, seed, first_id + (u64)b, level, msg + (size_t)b * c->n, ct + (size_t)b * 2 * c->L * c->n);
}
static void decrypt_one(oc_ctx* c, const u64* sk, const u64* ct, int64_t* out) {
    int N = c->n; u64 q = c->prm[0];
    u64* v = (u64*)malloc(sizeof(u64) * N);
    for (int i = 0; i < N; i++) v[i] = addm(ct[i], mulm(ct[(size_t)c->L * N + i], sk[i], q), q);
    oc_intt(c, v, 0);
    for (int i = 0; i < N; i++) out[i] = v[i] > (q >> 1) ? (int64_t)v[i] - (int64_t)q : (int64_t)v[i];
    free(v);
}
void oc_decrypt(oc_ctx* c, const u64* sk, const u64* ct, int count, int level, int64_t* out) {
    (void)level;
#pragma omp parallel for
    for (int b = 0; b < count; b++)
        decrypt_one(c, sk, ct + (size_t)b * 2 * c->L * c->n, out + (size_t)b * c->n);
}
void oc_encode_plain(oc_ctx* c, const int64_t* msg, u64* pt, int count, int level) {
    int N = c->n;
#pragma omp parallel for collapse(2)
    for (int b = 0; b < count; b++)
        for (int p = 0; p <= level; p++) {
            u64* d = pt + ((size_t)b * c->L + p) * N;
            for (int i = 0; i < N; i++) d[i] = red_i64(msg[(size_t)b * N + i], c->prm[p]);
            oc_ntt(c, d, p);
        }
}

/* ---------------- elementwise ---------------- */
#define CT(base, b, poly, p) ((base) + (((size_t)(b) * 2 + (poly)) * c->L + (p)) * c->n)

void oc_add(oc_ctx* c, const u64* a, const u64* b, u64* out, int count, int level, int sub) {
    for (int x = 0; x < count; x++)
        for (int k = 0; k < 2; k++)
            for (int p = 0; p <= level; p++) {
                const u64 *pa = CT(a, x, k, p), *pb = CT(b, x, k, p);
                u64* po = CT(out, x, k, p);
                u64 q = c->prm[p];
                for (int i = 0; i < c->n; i++) po[i] = sub ? subm(pa[i], pb[i], q) : addm(pa[i], pb[i], q);
            }
}
void oc_add_const(oc_ctx* c, const u64* a, const u64* cst, u64* out, int count, int level) {
    for (int x = 0; x < count; x++)
        for (int k = 0; k < 2; k++)
            for (int p = 0; p <= level; p++) {
                const u64* pa = CT(a, x, k, p);
                u64* po = CT(out, x, k, p);
                for (int i = 0; i < c->n; i++) po[i] = k == 0 ? addm(pa[i], cst[p], c->prm[p]) : pa[i];
            }
}
void oc_add_plain(oc_ctx* c, const u64* a, const u64* pt, u64* out, int count, int level) {
    for (int x = 0; x < count; x++)
        for (int k = 0; k < 2; k++)
            for (int p = 0; p <= level; p++) {
                const u64* pa = CT(a, x, k, p);
                const u64* pp = pt + (size_t)p * c->n;
                u64* po = CT(out, x, k, p);
                for (int i = 0; i < c->n; i++) po[i] = k == 0 ? addm(pa[i], pp[i], c->prm[p]) : pa[i];
            }
}
void oc_mul_const(oc_ctx* c, const u64* a, const u64* cst, u64* out, int count, int level) {
    for (int x = 0; x < count; x++)
        for (int k = 0; k < 2; k++)
            for (int p = 0; p <= level; p++) {
                const u64* pa = CT(a, x, k, p);
                u64* po = CT(out, x, k, p);
                for (int i = 0; i < c->n; i++) po[i] = mulm(pa[i], cst[p], c->prm[p]);
            }
}
void oc_mul_plain(oc_ctx* c, const u64* a, const u64* pt, u64* out, int count, int level) {
    for (int x = 0; x < count; x++)
        for (int k = 0; k < 2; k++)
            for (int p = 0; p <= level; p++) {
                const u64* pa = CT(a, x, k, p);
                const u64* pp = pt + (size_t)p * c->n;
                u64* po = CT(out, x, k, p);
                for (int i = 0; i < c->n; i++) po[i] = mulm(pa[i], pp[i], c->prm[p]);
            }
}
void oc_imul(oc_ctx* c, const u64* a, u64* out, int count, int level) {
    /* multiply by X^(N/2): NTT slot i scales by psi^((2brv(i)+1) N/2) */
    int N = c->n;
    for (int p = 0; p <= level; p++) {
        u64 q = c->prm[p];
        u64* f = (u64*)malloc(sizeof(u64) * N);
        for (int i = 0; i < N; i++) {
            u64 e = ((2 * (u64)brv((unsigned)i, c->log_n) + 1) * (u64)(N / 2)) % (2 * (u64)N);
            f[i] = powm(c->psi[p], e, q);
        }
        for (int x = 0; x < count; x++)
            for (int k = 0; k < 2; k++) {
                const u64* pa = CT(a, x, k, p);
                u64* po = CT(out, x, k, p);
                for (int i = 0; i < N; i++) po[i] = mulm(pa[i], f[i], q);
            }
        free(f);
    }
}

/* ---------------- rescale ---------------- */
static void rescale_poly(oc_ctx* c, const u64* in, u64* out, int level) {
    int N = c->n;
    u64 ql = c->prm[level], half = ql >> 1;
    u64* r = (u64*)malloc(sizeof(u64) * N);
    memcpy(r, in + (size_t)level * N, sizeof(u64) * N);
    oc_intt(c, r, level);
    for (int p = 0; p < level; p++) {
        u64 q = c->prm[p];
        u64 inv = invm(ql % q, q);
        u64* t = (u64*)malloc(sizeof(u64) * N);
        for (int i = 0; i < N; i++) {
            /* centred remainder r_c in (-ql/2, ql/2] */
            t[i] = r[i] > half ? subm(0, (ql - r[i]) % q, q) : r[i] % q;
        }
        oc_ntt(c, t, p);
        const u64* x = in + (size_t)p * N;
        u64* y = out + (size_t)p * N;
        for (int i = 0; i < N; i++) y[i] = mulm(subm(x[i], t[i], q), inv, q);
        free(t);
    }
    free(r);
}
void oc_rescale(oc_ctx* c, const u64* a, u64* out, int count, int level) {
#pragma omp parallel for collapse(2)
    for (int x = 0; x < count; x++)
        for (int k = 0; k < 2; k++)
            rescale_poly(c, CT(a, x, k, 0), CT(out, x, k, 0), level);
}

/* ---------------- basis conversion (fast, approximate) ----------------
 * in: coefficient-form limbs for source primes src[0..ns-1]
 * out: coefficient-form limbs for target primes dst[0..nd-1]
 * out_t = sum_k [x_k * (S/s_k)^-1]_{s_k} * (S/s_k mod t) mod t          */
void oc_basis_convert(oc_ctx* c, const u64* in, const int* src, int ns, u64* out, const int* dst, int nd) {
    int N = c->n;
    u64 hinv[MAXP];
    for (int k = 0; k < ns; k++) {
        u64 sk = c->prm[src[k]], prod = 1;
        for (int k2 = 0; k2 < ns; k2++)
            if (k2 != k) prod = mulm(prod, c->prm[src[k2]] % sk, sk);
        hinv[k] = invm(prod, sk);
    }
    for (int d = 0; d < nd; d++) {
        u64 t = c->prm[dst[d]];
        u64 hmod[MAXP];
        for (int k = 0; k < ns; k++) {
            u64 prod = 1;
            for (int k2 = 0; k2 < ns; k2++)
                if (k2 != k) prod = mulm(prod, c->prm[src[k2]] % t, t);
            hmod[k] = prod;
        }
        u64* o = out + (size_t)d * N;
        for (int i = 0; i < N; i++) {
            u64 acc = 0;
            for (int k = 0; k < ns; k++) {
                u64 y = mulm(in[(size_t)k * N + i], hinv[k], c->prm[src[k]]);
                acc = addm(acc, mulm(y % t, hmod[k], t), t);
            }
            o[i] = acc;
        }
    }
}

/* Centred P -> Q_l conversion for ModDown: the CENTRED representative
 * a_c in (-P/2, P/2] of the integer a given by its residues mod p_k (coefficient
 * form), reduced mod q_i.  With y_k = [a_k (P/p_k)^-1]_{p_k},
 * a = sum_k y_k P/p_k - r P where r = round(sum_k y_k / p_k); r is computed
 * in IEEE double (no FMA: y_k * (1/p_k) then a running sum in k order, then
 * floor(v + 0.5)), exactly as the device does, so both round identically.
 * Removing the [0, K) overflow bias of the plain fast conversion keeps the
 * key-switching error zero-mean (a biased error times the secret key
 * concentrates ~1e-7 on the slots next to zeta^{+-1}). */
void oc_moddown_convert(oc_ctx* c, const u64* in, u64* out, int nl) {
    int N = c->n, L = c->L, K = c->K;
    u64 hinv[MAXP];
    double pinv[MAXP];
    for (int k = 0; k < K; k++) {
        u64 pk = c->prm[L + k], prod = 1;
        for (int k2 = 0; k2 < K; k2++)
            if (k2 != k) prod = mulm(prod, c->prm[L + k2] % pk, pk);
        hinv[k] = invm(prod, pk);
        pinv[k] = 1.0 / (double)pk;
    }
    for (int i = 0; i < nl; i++) {
        u64 q = c->prm[i];
        u64 hmod[MAXP], pm = 1;
        for (int k = 0; k < K; k++) {
            u64 prod = 1;
            for (int k2 = 0; k2 < K; k2++)
                if (k2 != k) prod = mulm(prod, c->prm[L + k2] % q, q);
            hmod[k] = prod;
            pm = mulm(pm, c->prm[L + k] % q, q);
        }
        u64* o = out + (size_t)i * N;
        for (int n = 0; n < N; n++) {
            u64 acc = 0;
            volatile double v = 0.0;
            for (int k = 0; k < K; k++) {
                u64 y = mulm(in[(size_t)k * N + n], hinv[k], c->prm[L + k]);
                volatile double t = (double)y * pinv[k];
                v = v + t;
                acc = addm(acc, mulm(y % q, hmod[k], q), q);
            }
            volatile double vh = v + 0.5;
            u64 r = (u64)floor(vh);
            o[n] = subm(acc, mulm(r % q, pm, q), q);
        }
    }
}

/* ---------------- key switching ----------------
 * d: NTT-form limbs 0..level of one polynomial (limb stride N).
 * evk: u64[beta][2][L+K][N].  k0, k1: outputs, limbs 0..level (stride N). */
/* ModUp of d (NTT form, limbs 0..level) into up[nd][ext][N]: per digit, the
 * digit's own limbs copied, the others by fast basis conversion + NTT. */
static void modup_all(oc_ctx* c, const u64* d, int level, u64* up) {
    int N = c->n, L = c->L, K = c->K, al = c->alpha;
    int nl = level + 1, ext = nl + K, nd = (nl + al - 1) / al;
    int idx[MAXP];
    for (int i = 0; i < nl; i++) idx[i] = i;
    for (int k = 0; k < K; k++) idx[nl + k] = L + k;
    u64* coef = (u64*)malloc(sizeof(u64) * (size_t)nl * N);
    memcpy(coef, d, sizeof(u64) * (size_t)nl * N);
    for (int i = 0; i < nl; i++) oc_intt(c, coef + (size_t)i * N, i);
    for (int j = 0; j < nd; j++) {
        int lo = j * al, hi = lo + al < nl ? lo + al : nl;
        int src[MAXP], dst[MAXP], ns = hi - lo, ndst = 0;
        for (int k = 0; k < ns; k++) src[k] = lo + k;
        for (int e = 0; e < ext; e++)
            if (e < lo || e >= hi) dst[ndst++] = idx[e];
        u64* conv = (u64*)malloc(sizeof(u64) * (size_t)ndst * N);
        oc_basis_convert(c, coef + (size_t)lo * N, src, ns, conv, dst, ndst);
        int w = 0;
        for (int e = 0; e < ext; e++) {
            u64* u = up + ((size_t)j * ext + e) * N;
            if (e >= lo && e < hi) {
                memcpy(u, d + (size_t)e * N, sizeof(u64) * N);
            } else {
                memcpy(u, conv + (size_t)w * N, sizeof(u64) * N);
                oc_ntt(c, u, idx[e]);
                w++;
            }
        }
        free(conv);
    }
    free(coef);
}

/* acc[b][ext][N] += sum_j up_j (.) evk_j[b]   (optionally up_j permuted by galois) */
static void inner_acc(oc_ctx* c, const u64* up, const u64* evk, int level, u64 galois, u64* acc) {
    int N = c->n, L = c->L, K = c->K, LK = L + K, al = c->alpha;
    int nl = level + 1, ext = nl + K, nd = (nl + al - 1) / al;
    u64* tmp = (u64*)malloc(sizeof(u64) * N);
    for (int j = 0; j < nd; j++)
        for (int e = 0; e < ext; e++) {
            int p = e < nl ? e : L + (e - nl);
            u64 q = c->prm[p];
            const u64* u = up + ((size_t)j * ext + e) * N;
            if (galois) { automorph_poly(c, u, tmp, galois); u = tmp; }
            for (int b = 0; b < 2; b++) {
                const u64* kk = evk + ((size_t)(j * 2 + b) * LK + p) * N;
                u64* a = acc + ((size_t)b * ext + e) * N;
                for (int i = 0; i < N; i++) a[i] = addm(a[i], mulm(u[i], kk[i], q), q);
            }
        }
    free(tmp);
}

/* ModDown of acc[2][ext][N] (centred) into k0, k1 (limbs 0..level) */
static void moddown_both(oc_ctx* c, const u64* acc, int level, u64* k0, u64* k1) {
    int N = c->n, L = c->L, K = c->K;
    int nl = level + 1, ext = nl + K;
    u64* pc = (u64*)malloc(sizeof(u64) * (size_t)K * N);
    u64* conv = (u64*)malloc(sizeof(u64) * (size_t)nl * N);
    for (int b = 0; b < 2; b++) {
        const u64* a = acc + (size_t)b * ext * N;
        memcpy(pc, a + (size_t)nl * N, sizeof(u64) * (size_t)K * N);
        for (int k = 0; k < K; k++) oc_intt(c, pc + (size_t)k * N, L + k);
        oc_moddown_convert(c, pc, conv, nl);
        u64* outp = b == 0 ? k0 : k1;
        for (int i = 0; i < nl; i++) {
            u64 q = c->prm[i];
            u64 pinv = invm(pmod(c, i), q);
            u64* t = conv + (size_t)i * N;
            oc_ntt(c, t, i);
            const u64* x = a + (size_t)i * N;
            u64* o = outp + (size_t)i * N;
            for (int n = 0; n < N; n++) o[n] = mulm(subm(x[n], t[n], q), pinv, q);
        }
    }
    free(pc); free(conv);
}

/* d: NTT-form limbs 0..level of one polynomial (limb stride N).
 * evk: u64[beta][2][L+K][N].  k0, k1: outputs, limbs 0..level (stride N). */
void oc_keyswitch(oc_ctx* c, const u64* d, const u64* evk, int level, u64* k0, u64* k1) {
    int N = c->n, K = c->K, al = c->alpha;
    int nl = level + 1, ext = nl + K, nd = (nl + al - 1) / al;
    u64* up = (u64*)malloc(sizeof(u64) * (size_t)nd * ext * N);
    u64* acc = (u64*)calloc((size_t)2 * ext * N, sizeof(u64));
    modup_all(c, d, level, up);
    inner_acc(c, up, evk, level, 0, acc);
    moddown_both(c, acc, level, k0, k1);
    free(up); free(acc);
}

/* ct x ct product, relinearised and rescaled by ONE centred division by
 * M = P * q_l (device helr_mul_relin_rescale): acc = sum_j ModUp(d2)_j evk_j,
 * acc_Q += P * (d0, d1), then out_i = (acc_i - conv_i) * M^-1 for i < l where
 * conv is the centred conversion of acc mod M from {p_0..p_{K-1}, q_l}. */
void oc_tensor(oc_ctx* c, const u64* a, const u64* b, u64* d, int level);
/* from a tensor d = [d0, d1, d2] (u64[3][L][N]) to one ciphertext at level-1 */
void oc_relin_rescale_tensor(oc_ctx* c, const u64* d, const u64* rlk, u64* out, int level) {
    int N = c->n, L = c->L, K = c->K, al = c->alpha;
    int nl = level + 1, ext = nl + K, nd = (nl + al - 1) / al, l = level, ns = K + 1;
    const int x = 0;
    {
        u64* up = (u64*)malloc(sizeof(u64) * (size_t)nd * ext * N);
        u64* acc = (u64*)calloc((size_t)2 * ext * N, sizeof(u64));
        u64* src = (u64*)malloc(sizeof(u64) * (size_t)ns * N);
        u64* conv = (u64*)malloc(sizeof(u64) * (size_t)l * N);
        modup_all(c, d + (size_t)2 * L * N, level, up);
        inner_acc(c, up, rlk, level, 0, acc);
        u64 srcp[MAXP];
        for (int k = 0; k < K; k++) srcp[k] = c->prm[L + k];
        srcp[K] = c->prm[l];
        u64 hinv[MAXP];
        double dinv[MAXP];
        for (int k = 0; k < ns; k++) {
            u64 m = srcp[k], prod = 1;
            for (int k2 = 0; k2 < ns; k2++)
                if (k2 != k) prod = mulm(prod, srcp[k2] % m, m);
            hinv[k] = invm(prod, m);
            dinv[k] = 1.0 / (double)m;
        }
        for (int bb = 0; bb < 2; bb++) {
            u64* ab = acc + (size_t)bb * ext * N;
            for (int i = 0; i < nl; i++) {  /* acc_Q += P * d_bb */
                u64 q = c->prm[i], pm = pmod(c, i);
                const u64* dd = d + ((size_t)bb * L + i) * N;
                for (int n = 0; n < N; n++) ab[(size_t)i * N + n] = addm(ab[(size_t)i * N + n], mulm(pm, dd[n], q), q);
            }
            for (int k = 0; k < K; k++) {
                memcpy(src + (size_t)k * N, ab + (size_t)(nl + k) * N, sizeof(u64) * N);
                oc_intt(c, src + (size_t)k * N, L + k);
            }
            memcpy(src + (size_t)K * N, ab + (size_t)l * N, sizeof(u64) * N);
            oc_intt(c, src + (size_t)K * N, l);
            for (int i = 0; i < l; i++) {
                u64 q = c->prm[i], mm = 1, hm[MAXP];
                for (int k = 0; k < ns; k++) {
                    u64 prod = 1;
                    for (int k2 = 0; k2 < ns; k2++)
                        if (k2 != k) prod = mulm(prod, srcp[k2] % q, q);
                    hm[k] = prod;
                    mm = mulm(mm, srcp[k] % q, q);
                }
                u64* o = conv + (size_t)i * N;
                for (int n = 0; n < N; n++) {
                    u64 s = 0;
                    volatile double v = 0.0;
                    for (int k = 0; k < ns; k++) {
                        u64 y = mulm(src[(size_t)k * N + n], hinv[k], srcp[k]);
                        volatile double t = (double)y * dinv[k];
                        v = v + t;
                        s = addm(s, mulm(y % q, hm[k], q), q);
                    }
                    volatile double vh = v + 0.5;
                    u64 r = (u64)floor(vh);
                    o[n] = subm(s, mulm(r % q, mm, q), q);
                }
                oc_ntt(c, o, i);
                u64 minv = invm(mm, q);
                u64* op = out + (((size_t)x * 2 + bb) * L + i) * N;
                for (int n = 0; n < N; n++) op[n] = mulm(subm(ab[(size_t)i * N + n], o[n], q), minv, q);
            }
        }
        free(up); free(acc); free(src); free(conv);
    }
}
void oc_mul_relin_rescale(oc_ctx* c, const u64* a, const u64* b, const u64* rlk, u64* out, int count, int level) {
    int N = c->n, L = c->L;
#pragma omp parallel for
    for (int x = 0; x < count; x++) {
        u64* d = (u64*)malloc(sizeof(u64) * (size_t)3 * L * N);
        oc_tensor(c, a + (size_t)x * 2 * L * N, b + (size_t)x * 2 * L * N, d, level);
        oc_relin_rescale_tensor(c, d, rlk, out + (size_t)x * 2 * L * N, level);
        free(d);
    }
}

/* Hoisted rotate-and-sum (device helr_rotsum): out = [a +] sum_t rot_{g_t}(a)
 * with one ModUp of c1, sigma_t applied to the ModUp'd digits, the inner
 * products summed in the extended basis and one ModDown. */
void oc_rotsum(oc_ctx* c, const u64* a, int nsteps, const int64_t* gal, const u64* const* keys, u64* out, int count,
               int level, int include_identity) {
    int N = c->n, L = c->L, K = c->K, al = c->alpha;
    int nl = level + 1, ext = nl + K, nd = (nl + al - 1) / al;
#pragma omp parallel for
    for (int x = 0; x < count; x++) {
        const u64* ax = a + (size_t)x * 2 * L * N;
        u64* ox = out + (size_t)x * 2 * L * N;
        u64* up = (u64*)malloc(sizeof(u64) * (size_t)nd * ext * N);
        u64* acc = (u64*)calloc((size_t)2 * ext * N, sizeof(u64));
        u64* k0 = (u64*)malloc(sizeof(u64) * (size_t)nl * N);
        u64* k1 = (u64*)malloc(sizeof(u64) * (size_t)nl * N);
        u64* tmp = (u64*)malloc(sizeof(u64) * N);
        modup_all(c, ax + (size_t)L * N, level, up);
        for (int t = 0; t < nsteps; t++) inner_acc(c, up, keys[t], level, (u64)gal[t], acc);
        moddown_both(c, acc, level, k0, k1);
        for (int p = 0; p < nl; p++) {
            u64 q = c->prm[p];
            const u64 *a0 = ax + (size_t)p * N, *a1 = ax + ((size_t)L + p) * N;
            u64 *o0 = ox + (size_t)p * N, *o1 = ox + ((size_t)L + p) * N;
            for (int i = 0; i < N; i++) {
                o0[i] = k0[(size_t)p * N + i];
                o1[i] = k1[(size_t)p * N + i];
                if (include_identity) { o0[i] = addm(o0[i], a0[i], q); o1[i] = addm(o1[i], a1[i], q); }
            }
            for (int t = 0; t < nsteps; t++) {
                automorph_poly(c, a0, tmp, (u64)gal[t]);
                for (int i = 0; i < N; i++) o0[i] = addm(o0[i], tmp[i], q);
            }
        }
        free(up); free(acc); free(k0); free(k1); free(tmp);
    }
}

/* tensor of one pair: d = [d0, d1, d2] (u64[3][L][N]) for limbs 0..level */
void oc_tensor(oc_ctx* c, const u64* a, const u64* b, u64* d, int level) {
    int N = c->n;
    const int x = 0;
#pragma omp parallel for
    for (int p = 0; p <= level; p++) {
        u64 q = c->prm[p];
        const u64 *a0 = CT(a, x, 0, p), *a1 = CT(a, x, 1, p), *b0 = CT(b, x, 0, p), *b1 = CT(b, x, 1, p);
        u64* d0 = d + (size_t)p * N;
        u64* d1 = d + ((size_t)c->L + p) * N;
        u64* d2 = d + ((size_t)2 * c->L + p) * N;
        for (int i = 0; i < N; i++) {
            d0[i] = mulm(a0[i], b0[i], q);
            d1[i] = addm(mulm(a0[i], b1[i], q), mulm(a1[i], b0[i], q), q);
            d2[i] = mulm(a1[i], b1[i], q);
        }
    }
}

/* ---------------- composite ops ---------------- */
void oc_mul_relin(oc_ctx* c, const u64* a, const u64* b, const u64* rlk, u64* out, int count, int level) {
    int N = c->n, nl = level + 1;
#pragma omp parallel for
    for (int x = 0; x < count; x++) {
        u64* d2 = (u64*)malloc(sizeof(u64) * (size_t)nl * N);
        u64* k0 = (u64*)malloc(sizeof(u64) * (size_t)nl * N);
        u64* k1 = (u64*)malloc(sizeof(u64) * (size_t)nl * N);
        u64* d0 = (u64*)malloc(sizeof(u64) * (size_t)nl * N);
        u64* d1 = (u64*)malloc(sizeof(u64) * (size_t)nl * N);
        for (int p = 0; p < nl; p++) {
            u64 q = c->prm[p];
            const u64 *a0 = CT(a, x, 0, p), *a1 = CT(a, x, 1, p), *b0 = CT(b, x, 0, p), *b1 = CT(b, x, 1, p);
            for (int i = 0; i < N; i++) {
                size_t o = (size_t)p * N + i;
                d0[o] = mulm(a0[i], b0[i], q);
                d1[o] = addm(mulm(a0[i], b1[i], q), mulm(a1[i], b0[i], q), q);
                d2[o] = mulm(a1[i], b1[i], q);
            }
        }
        oc_keyswitch(c, d2, rlk, level, k0, k1);
        for (int p = 0; p < nl; p++) {
            u64 q = c->prm[p];
            u64 *o0 = CT(out, x, 0, p), *o1 = CT(out, x, 1, p);
            for (int i = 0; i < N; i++) {
                size_t o = (size_t)p * N + i;
                o0[i] = addm(d0[o], k0[o], q);
                o1[i] = addm(d1[o], k1[o], q);
            }
        }
        free(d2); free(k0); free(k1); free(d0); free(d1);
    }
}
void oc_automorph(oc_ctx* c, const u64* a, u64* out, int count, int level, int64_t galois) {
    for (int x = 0; x < count; x++)
        for (int k = 0; k < 2; k++)
            for (int p = 0; p <= level; p++)
                automorph_poly(c, CT(a, x, k, p), CT(out, x, k, p), (u64)galois);
}
void oc_rotate(oc_ctx* c, const u64* a, int64_t galois, const u64* gk, u64* out, int count, int level, int accumulate) {
    int N = c->n, nl = level + 1;
#pragma omp parallel for
    for (int x = 0; x < count; x++) {
        u64* r0 = (u64*)malloc(sizeof(u64) * (size_t)nl * N);
        u64* r1 = (u64*)malloc(sizeof(u64) * (size_t)nl * N);
        u64* k0 = (u64*)malloc(sizeof(u64) * (size_t)nl * N);
        u64* k1 = (u64*)malloc(sizeof(u64) * (size_t)nl * N);
        for (int p = 0; p < nl; p++) {
            automorph_poly(c, CT(a, x, 0, p), r0 + (size_t)p * N, (u64)galois);
            automorph_poly(c, CT(a, x, 1, p), r1 + (size_t)p * N, (u64)galois);
        }
        oc_keyswitch(c, r1, gk, level, k0, k1);
        for (int p = 0; p < nl; p++) {
            u64 q = c->prm[p];
            const u64 *a0 = CT(a, x, 0, p), *a1 = CT(a, x, 1, p);
            u64 *o0 = CT(out, x, 0, p), *o1 = CT(out, x, 1, p);
            for (int i = 0; i < N; i++) {
                size_t o = (size_t)p * N + i;
                u64 v0 = addm(r0[o], k0[o], q), v1 = k1[o];
                if (accumulate) { v0 = addm(v0, a0[i], q); v1 = addm(v1, a1[i], q); }
                o0[i] = v0; o1[i] = v1;
            }
        }
        free(r0); free(r1); free(k0); free(k1);
    }
}
/* ModRaise (bootstrapping step 1): coefficients of a modulo q_0, centred to
 * (-q_0/2, q_0/2], re-read modulo q_0..q_level_out.  Textbook definition
 * (Cheon-Han-Kim-Kim-Song 2018, section 4.1); the reference only models the
 * bootstrap's level reset (hesim.py:228-236). */
void oc_mod_raise(oc_ctx* c, const u64* a, u64* out, int count, int level_out) {
    int N = c->n;
    u64 q0 = c->prm[0], half = q0 >> 1;
    for (int x = 0; x < count; x++)
        for (int k = 0; k < 2; k++) {
            u64* r = (u64*)malloc(sizeof(u64) * N);
            memcpy(r, CT(a, x, k, 0), sizeof(u64) * N);
            oc_intt(c, r, 0);
            for (int p = 0; p <= level_out; p++) {
                u64 q = c->prm[p];
                u64* o = CT(out, x, k, p);
                for (int i = 0; i < N; i++) {
                    u64 v = r[i];
                    if (v > half) { u64 m = (q0 - v) % q; o[i] = m ? q - m : 0; }
                    else o[i] = v % q;
                }
                oc_ntt(c, o, p);
            }
            free(r);
        }
}
void oc_refresh(oc_ctx* c, const u64* sk, const u64* a, int in_level, double ratio, u64* out, int out_level,
                int count, u64 seed, u64 first_id) {
    (void)in_level;
    int N = c->n;
    for (int x = 0; x < count; x++) {
        int64_t* m = (int64_t*)malloc(sizeof(int64_t) * N);
        decrypt_one(c, sk, a + (size_t)x * 2 * c->L * N, m);
        if (ratio != 1.0) {
            for (int i = 0; i < N; i++) {
                volatile double v = (double)m[i];
                v = v * ratio;
                m[i] = (int64_t)llrint(v);
            }
        }
        encrypt_one(c, sk, seed, first_id + (u64)x, out_level, m, out + (size_t)x * 2 * c->L * N);
        free(m);
    }
}
