/*
 * helr_ckks.h — C ABI of the B200 RNS-CKKS evaluator behind the reference's
 * evaluator protocol (helr.hesim.SimContext, pkg/src/helr/hesim.py:110-291).
 *
 * The reference is pure Python and binds no FFI; these entry points are what
 * its evaluator methods become once a ciphertext is a real RNS polynomial pair
 * on the device.  Each entry point cites the reference method it replaces.
 *
 * Conventions
 *  - Plain C types only: device pointers are passed as (u)int64_t* living in
 *    device memory (from torch tensors' data_ptr()), streams as void*
 *    (cudaStream_t), sizes as int.  No entry point throws: each returns 0 on
 *    success or a negative HELR_E* code, with a message retrievable through
 *    helr_last_error().  Every call is asynchronous on the given stream.
 *  - Ring: N = 2^log_n, primes[0..L-1] = q_0..q_{L-1} (ciphertext chain),
 *    primes[L..L+K-1] = p_0..p_{K-1} (special primes; key-switching digits
 *    hold alpha = ceil(L/dnum) limbs, P = prod p_k should exceed the largest
 *    digit modulus).  All primes < 2^61, = 1 mod 2N; primes < 2^41 take the
 *    fp64 NTT path.
 *  - Polynomials are limb-major u64[limbs][N] of canonical residues in
 *    [0, q), in negacyclic NTT (evaluation) form unless stated otherwise.
 *    NTT slot i holds a(psi^(2*brv(i)+1)).
 *  - A ciphertext buffer is u64[2][L][N] (c0 limbs, then c1 limbs, always
 *    sized for the top level).  "level" l means limbs 0..l are active; the
 *    rest of the buffer is ignored.  A batch is `count` such buffers back to
 *    back (stride 2*L*N words).
 *  - Secret key buffer: u64[L+K][N] (NTT form over every prime).
 *  - Switching key (relinearisation or Galois): u64[beta][2][L+K][N] with
 *    beta = ceil(L/alpha) digits of the top-level chain.
 *  - Randomness is a counter-based generator keyed by (seed, stream, index)
 *    so device and CPU oracle produce identical keys and ciphertexts.
 */
#ifndef HELR_CKKS_H
#define HELR_CKKS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HELR_OK 0
#define HELR_EINVAL (-1)
#define HELR_ECUDA (-2)
#define HELR_ENOMEM (-3)

typedef struct helr_ctx helr_ctx;

/* Last error message of the calling thread (empty when none). */
int helr_last_error(char* buf, size_t len);

/* Library/ABI version (major*10000 + minor*100 + patch). */
int helr_version(void);

/* Context: builds twiddle, basis-conversion and rescale tables on the device.
 * Replaces SimContext.__init__ (hesim.py:119-122) at ring level.  max_batch
 * sizes the key-switching workspace (ciphertexts per batched call). */
int helr_ctx_create(helr_ctx** out, int log_n, int L, int K, int dnum,
                    const uint64_t* primes, const uint64_t* psi, int cbd_eta,
                    int max_batch);
int helr_ctx_destroy(helr_ctx* ctx);

/* ---- ring primitives (primitive sweep; building blocks) ---------------- */

/* In-place forward / inverse negacyclic NTT of `count` polynomials, each with
 * n_limbs limbs using primes first_prime .. first_prime+n_limbs-1; polynomial
 * b limb i lives at data + b*poly_stride + i*N. */
int helr_ntt_fwd(helr_ctx* ctx, uint64_t* data, int first_prime, int n_limbs,
                 int count, int64_t poly_stride, void* stream);
int helr_ntt_inv(helr_ctx* ctx, uint64_t* data, int first_prime, int n_limbs,
                 int count, int64_t poly_stride, void* stream);

/* ---- keys (client side; not in the reference, which has no keys) ------- */

int helr_keygen_secret(helr_ctx* ctx, uint64_t* sk, uint64_t seed, void* stream);
/* Sparse ternary secret with exactly hw nonzero +-1 coefficients (hw = 0:
 * uniform ternary, as helr_keygen_secret).  Lower secret weight shrinks the
 * rescale / key-switching rounding noise by ~sqrt(hw / (2N/3)). */
int helr_keygen_secret_hw(helr_ctx* ctx, uint64_t* sk, uint64_t seed, int hw, void* stream);
/* galois == 0: relinearisation key (s^2 -> s); otherwise key for X -> X^galois. */
int helr_keygen_switch(helr_ctx* ctx, const uint64_t* sk, int64_t galois,
                       uint64_t* evk, uint64_t seed, uint64_t key_id, void* stream);

/* ---- encryption boundary (SimContext.enc / dec, hesim.py:146-162) ------- */

/* Encode-side integers -> ciphertexts.  msg: int64[count][N] integer
 * coefficients (already scaled and rounded on the host); ciphertext b uses
 * randomness stream id first_ct_id + b. */
int helr_encrypt(helr_ctx* ctx, const uint64_t* sk, const int64_t* msg,
                 uint64_t* ct, int count, int level, uint64_t seed,
                 uint64_t first_ct_id, void* stream);
/* Decrypt through q_0 only: out[b][n] = centred coefficient n of
 * (c0 + c1*s) mod q_0 (valid while |m| < q_0/2). */
int helr_decrypt(helr_ctx* ctx, const uint64_t* sk, const uint64_t* ct,
                 int count, int level, int64_t* out, void* stream);
/* Integer polynomial -> plaintext in NTT form over limbs 0..level. */
int helr_encode_plain(helr_ctx* ctx, const int64_t* msg, uint64_t* pt,
                      int count, int level, void* stream);

/* Device-side CKKS encoding (client side; replaces the
 * host FFT behind SimContext.enc, hesim.py:146-158, as used by client_prepare,
 * enctrain.py:114-152).  re / im (im may be NULL = real slots): count slot
 * vectors of N/2 doubles at slot_stride; coef: count x N int64 = rint(scale *
 * m) of the canonical-embedding polynomial (encoder.py).  Device pointers;
 * synchronises the stream (it reports overflow: |scale * m| >= 2^62). */
int helr_encode(helr_ctx* ctx, const double* re, const double* im, int64_t slot_stride, int count,
                double scale, int64_t* coef, void* stream);
/* Inverse map (SimContext.dec, hesim.py:160-162, via decode_weights,
 * enctrain.py:266-289): integer coefficients -> slots / scale. */
int helr_decode(helr_ctx* ctx, const int64_t* coef, int count, double scale, double* re, double* im,
                int64_t slot_stride, void* stream);

/* ---- arithmetic (SimContext.add/cadd/mul/cmul/imul, hesim.py:166-216) -- */

int helr_add(helr_ctx* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out,
             int count, int level, void* stream);
int helr_sub(helr_ctx* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out,
             int count, int level, void* stream);
/* c0 += c (a constant polynomial); c: u64[level+1] residues (cadd, scalar). */
int helr_add_const(helr_ctx* ctx, const uint64_t* a, const uint64_t* c,
                   uint64_t* out, int count, int level, void* stream);
/* c0 += pt (cadd, vector); pt: u64[L][N] NTT plaintext. */
int helr_add_plain(helr_ctx* ctx, const uint64_t* a, const uint64_t* pt,
                   uint64_t* out, int count, int level, void* stream);
/* Both polynomials times a per-limb constant c (u64[level+1]); no rescale. */
int helr_mul_const(helr_ctx* ctx, const uint64_t* a, const uint64_t* c,
                   uint64_t* out, int count, int level, void* stream);
/* Both polynomials times an NTT plaintext; no rescale. */
int helr_mul_plain(helr_ctx* ctx, const uint64_t* a, const uint64_t* pt,
                   uint64_t* out, int count, int level, void* stream);
/* Fold every residue word (any value < 2^64, e.g. the element-wise sum of up
 * to 8 ranks' residue vectors after an all-reduce) back to [0, q_i).  New:
 * the combine step of the sharded full-batch gradient; the
 * reference sums block gradients with SimContext.add (enctrain.py:374-381). */
int helr_reduce(helr_ctx* ctx, const uint64_t* a, uint64_t* out, int count, int level, void* stream);
/* Drop q_level: out (level-1) = round(in / q_level). */
int helr_rescale(helr_ctx* ctx, const uint64_t* a, uint64_t* out, int count,
                 int level, void* stream);
/* ModRaise, the first step of real CKKS bootstrapping (the reference only
 * models a bootstrap: SimContext.bootstrap, hesim.py:228-236): read `a`
 * modulo q_0 (any level; only limb 0 is used) and re-interpret the centred
 * coefficients modulo q_0..q_level_out.  out encrypts m + q_0 * I. */
int helr_mod_raise(helr_ctx* ctx, const uint64_t* a, uint64_t* out, int count,
                   int level_out, void* stream);
/* ct x ct product with relinearisation (no rescale): out = relin(a*b). */
int helr_mul_relin(helr_ctx* ctx, const uint64_t* a, const uint64_t* b,
                   const uint64_t* rlk, uint64_t* out, int count, int level,
                   void* stream);
/* ct x ct product, relinearised and rescaled in one key switch: the
 * accumulator gets P*(d0, d1) and a single centred ModDown divides by
 * P*q_level (SimContext.mul, hesim.py:186-195).  Output at level-1. */
int helr_mul_relin_rescale(helr_ctx* ctx, const uint64_t* a, const uint64_t* b,
                           const uint64_t* rlk, uint64_t* out, int count, int level,
                           void* stream);
/* Multiply by X^(N/2) (slots * i). */
int helr_imul(helr_ctx* ctx, const uint64_t* a, uint64_t* out, int count,
              int level, void* stream);

/* ---- rotations (SimContext.rotate, sum_col_vec, sum_rows) --------------- */

/* out = rot_galois(a).  With accumulate != 0: out = a + rot_galois(a)
 * (the rotate-and-add step of hesim.py:255-264, 278-280).  All `count`
 * ciphertexts share one read of the key. */
int helr_rotate(helr_ctx* ctx, const uint64_t* a, int64_t galois,
                const uint64_t* gk, uint64_t* out, int count, int level,
                int accumulate, void* stream);

/* Hoisted rotate-and-sum: out = [a +] sum_{t<nsteps} rot_{galois[t]}(a)
 * (include_identity selects the a term).  One ModUp of c1, the inner
 * products of all rotations summed in the extended basis, one ModDown
 * ("double hoisting").  A baby-step/giant-step pair of calls computes
 * sum_{k<g} rot_k(a), i.e. each half of sum_col_vec (hesim.py:255-264)
 * with ~4x fewer NTTs than log2(g) sequential rotate-and-add steps.
 * galois: host array; keys: host array of device key pointers; nsteps <= 32. */
int helr_rotsum(helr_ctx* ctx, const uint64_t* a, int nsteps, const int64_t* galois,
                const uint64_t* const* keys, uint64_t* out, int count, int level,
                int include_identity, void* stream);

/* ---- refresh stand-in (SimContext.bootstrap, hesim.py:228-236) ---------- */

/* NOT bootstrapping: decrypts through q_0 with the secret key, multiplies the
 * integer message by `ratio` (fp64, round-to-nearest; 1.0 keeps it exact) and
 * re-encrypts at `out_level` with fresh randomness (stream first_ct_id + b). */
int helr_refresh(helr_ctx* ctx, const uint64_t* sk, const uint64_t* a,
                 int in_level, double ratio, uint64_t* out, int out_level,
                 int count, uint64_t seed, uint64_t first_ct_id, void* stream);

/* ---- fused training step (enctrain.py:344-398 loop body) ---------------- */

/* One enhanced-NAG iteration over one batch, depth-7 schedule:
 *   P_r  = rescale(relin(sum_j Z_rj (x) W_j))                 level lw-1
 *   R_r  = rotsum_left(P_r)  (log_g rotate-and-add)            (sum_col_vec, left half)
 *   U_r  = rotsum_right(rescale(R_r * mask))                   level lw-2
 *   QU_r = q0 + q1 U + q2 U^2 + q3 U^3 (U^2 and (q3 U) products) level lw-4
 *   G_j  = rescale(relin(sum_r QU_r (x) Z_rj))                 level lw-5
 *   G_j  = rotsum_rows(G_j) (log_m rotate-and-add by g*2^i)   (sum_rows)
 *   D_j  = rescale(relin(G_j (x) Bbar_j))                      level lw-6
 *   V'   = rescale(c_w1 W + c_a1 D);  W' = rescale(c_w2 W + c_v2 V + c_a2 D)  level lw-7
 * Constants are per-limb residues prepared by the host planner
 * (paper_2406_13221_b200/driver.py), consts[k*L + i] for k:
 *   0 C3 (q3 u, level lw-2)   1 C1 (q1 u -> lw-4)   2 C2 (q2 u^2 -> lw-4)
 *   3 C0 (q0 added at lw-4)   4 c_w1  5 c_a1  6 c_w2  7 c_v2  8 c_a2  9 unused
 * Ciphertext arrays are contiguous u64[2][L][N] buffers. */
#define HELR_NAG_NCONST 10
typedef struct helr_nag_args {
    const uint64_t* z;      /* [rows][cols] ciphertexts of this batch, level >= lw */
    int rows, cols;         /* row blocks per batch, column blocks */
    int log_g, log_m;       /* block of m = 2^log_m rows x g = 2^log_g columns, m*g = N/2 */
    uint64_t* w;            /* [cols] weights: level lw in, level lw-7 out (in place) */
    uint64_t* v;            /* [cols] companion weights, same */
    const uint64_t* bbar;   /* [cols] quadratic-gradient scales, level >= lw-5 */
    int lw;                 /* level of w and v on entry, >= 7 */
    const uint64_t* rlk;    /* relinearisation key */
    const uint64_t* const* rot_left;   /* [log_g] keys, left rotation by 2^i */
    const uint64_t* const* rot_right;  /* [log_g] keys, right rotation by 2^i */
    const uint64_t* const* rot_rows;   /* [log_m] keys, left rotation by g*2^i
                                          (or grouped, see log_baby_rows) */
    const uint64_t* mask_pt;           /* [L][N] row-start mask plaintext (NTT) */
    const uint64_t* consts;            /* device [HELR_NAG_NCONST][L] */
    uint64_t* grad;                    /* [cols] gradient accumulator (full batch) */
    int phase;  /* 0: full mini-batch iteration; 1: grad = this batch's gradient;
                   2: grad += this batch's gradient; 3: finish from grad (row sums,
                   Bbar product, update) */
    int log_baby; /* 0: sum_col_vec by log2(g) rotate-and-add steps (rot_left[i] /
                     rot_right[i] rotate by 2^i); b > 0: hoisted groups of at most b
                     bits each (helr_rotsum_groups: ceil(log_g / b) groups, bits
                     spread evenly, larger groups first); group j with offset
                     o_j = bits of the groups before it sums rotations
                     k*2^o_j, k = 1..2^bits_j - 1; rot_left holds the keys of
                     group 0, then group 1, ...; rot_right likewise for the
                     negated steps */
    int log_baby_rows; /* sum_rows: 0 = log_m rotate-and-add steps by g*2^i;
                          b > 0: grouped as above over log_m, steps scaled by g */
} helr_nag_args;

/* Group bit-widths of a grouped rotate-and-sum over 2^log_total rotations
 * with groups of at most max_bits bits: returns the number of groups and
 * writes the widths to bits[] (at most 64 entries). */
int helr_rotsum_groups(int log_total, int max_bits, int* bits);

int helr_nag_iteration(helr_ctx* ctx, const helr_nag_args* args, void* stream);

/* Capture / replay the iteration as a CUDA graph (same arguments each
 * replay; constants are read from args->consts at replay time). */
int helr_nag_graph_capture(helr_ctx* ctx, const helr_nag_args* args, void* stream, void** graph_exec);
/* Re-point a captured graph at new arguments of the same shape (another
 * batch of the resident dataset) by re-capturing and updating it in place. */
int helr_nag_graph_update(helr_ctx* ctx, const helr_nag_args* args, void* stream, void* graph_exec);
int helr_nag_graph_launch(void* graph_exec, void* stream);
int helr_nag_graph_destroy(void* graph_exec);

/* ---- training-harness metrics on the device ----
 * The per-iteration metrics of train_encrypted (enctrain.py:417-436):
 * scores s = X w (X: n x d row-major doubles, bias column included; y in
 * {-1,+1}; w: d doubles; device pointers).  out (host, 4 doubles):
 * log_likelihood (optim.py:123-126), accuracy of sign(s) (optim.py:200-206),
 * midrank AUROC (optim.py:209-229; NaN with one class), n_pos.  scratch:
 * helr_metrics_scratch(n) device doubles.  Synchronises the stream. */
size_t helr_metrics_scratch(int n);
int helr_metrics(helr_ctx* ctx, const double* X, const double* y, const double* w, int n, int d,
                 double* scratch, double* out, void* stream);

/* ---- instrumentation (not part of the reference surface) ---------------- */

/* Per-launch CUDA-event timing by kernel category (0 NTT, 1 ModUp, 2 key
 * inner product, 3 ModDown, 4 tensor, 5 rescale, 6 elementwise, 7 other);
 * bytes are the algorithmic bytes each launch must move. */
#define HELR_PROF_NCAT 8
int helr_prof_enable(int on);
int helr_prof_collect(double* ms, double* bytes, int* launches);
/* Running count of kernels this library has launched (eager launches). */
unsigned long long helr_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* HELR_CKKS_H */
