// ops_internal.cuh — batched, strided evaluator primitives shared by the
// C-ABI wrappers (ops.cu) and the fused training driver (nag.cu).
// Strides are in 64-bit words between consecutive ciphertexts; a stride of 0
// broadcasts one ciphertext to every item.
#pragma once

// rotations per hoisted rotate-and-sum group (op_rotsum_hoisted)
#define HELR_MAX_HOIST 32
#include "ctx.cuh"

enum EwOp { EW_ADD = 0, EW_SUB, EW_ADDC, EW_ADDPT, EW_MULC, EW_MULPT, EW_IMUL, EW_REDUCE };

int op_ew(helr_ctx* c, int op, const u64* a, long long as, const u64* b, long long bs, u64* out, long long os,
          int count, int level, cudaStream_t s);
int op_rescale(helr_ctx* c, const u64* a, long long as, u64* out, long long os, int count, int level, cudaStream_t s);
// out_i = relin( sum_{t<terms} a[i*a_is + t*a_ts] (x) b[i*b_is + t*b_ts] ), no rescale
int op_mul_relin_sum(helr_ctx* c, const u64* a, long long a_is, long long a_ts, const u64* b, long long b_is,
                     long long b_ts, int terms, const u64* rlk, u64* out, long long os, int count, int level,
                     cudaStream_t s);
int op_rotate(helr_ctx* c, const u64* a, long long as, long long galois, const u64* gk, u64* out, long long os,
              int count, int level, int accumulate, cudaStream_t s);
int op_lincomb(helr_ctx* c, int terms, const u64* const* x, const long long* xs, const u64* const* k, u64* out,
               long long os, int count, int level, cudaStream_t s);
// out = [a +] sum_{t < nsteps} rot_{gal[t]}(a): one ModUp, summed inner
// products in the extended basis, one ModDown (double hoisting)
int op_rotsum_hoisted(helr_ctx* c, const u64* a, long long as, int nsteps, const long long* gal, const u64* const* keys,
                      u64* out, long long os, int count, int level, int include_identity, cudaStream_t s);
// out_i (level-1) = rescale(relin(sum_t a (x) b)), the rescale merged into ModDown
int op_mul_relin_rescale_sum(helr_ctx* c, const u64* a, long long a_is, long long a_ts, const u64* b, long long b_is,
                             long long b_ts, int terms, const u64* rlk, u64* out, long long os, int count, int level,
                             cudaStream_t s);
