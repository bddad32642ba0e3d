// modarith.cuh — 64-bit modular arithmetic for sm_100a (INT pipe).
//
// All primes are < 2^62.  Canonical residues live in [0, q); the NTT keeps
// lazy values in [0, 4q) (forward, Harvey butterflies) or [0, 2q) (inverse).
// Constant multiplications use Shoup's precomputed quotient
// w' = floor(w * 2^64 / q); variable x variable products use a 128-bit
// Barrett reduction with ratio floor(2^128 / q) (two words).
#pragma once
#include <cstdint>

typedef uint64_t u64;
typedef unsigned int u32;

#define HD __host__ __device__ __forceinline__
#define DV __device__ __forceinline__

DV u64 mulhi64(u64 a, u64 b) { return __umul64hi(a, b); }

// a * w mod q in [0, 2q) for any a < 2^64, w < q.
DV u64 shoup_lazy(u64 a, u64 w, u64 wsh, u64 q) {
    u64 h = mulhi64(a, wsh);
    return a * w - h * q;
}
// Shoup with an approximate quotient: the high word of a * wsh without the
// low x low partial product and the low halves of the cross products (one
// 32x32->64 and two 32x32->hi32 multiplies instead of four 32x32->64).  The
// quotient is at most 2 below Shoup's, so the result is in [0, 4q) for any
// a < 2^64 — the NTT keeps lazy values in [0, 8q) (all primes < 2^61).
DV u64 shoup_lazy4(u64 a, u64 w, u64 wsh, u64 q) {
    const u32 a0 = (u32)a, a1 = (u32)(a >> 32), w0 = (u32)wsh, w1 = (u32)(wsh >> 32);
    const u64 h = (u64)a1 * w1 + (u64)__umulhi(a1, w0) + (u64)__umulhi(a0, w1);
    return a * w - h * q;
}
DV u64 csub(u64 a, u64 q) { return a >= q ? a - q : a; }
DV u64 shoup(u64 a, u64 w, u64 wsh, u64 q) { return csub(shoup_lazy(a, w, wsh, q), q); }

DV u64 add_mod(u64 a, u64 b, u64 q) { return csub(a + b, q); }
DV u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
DV u64 neg_mod(u64 a, u64 q) { return a ? q - a : 0; }

// 128-bit value as (hi, lo)
struct u128v { u64 hi, lo; };

DV u128v mul_wide(u64 a, u64 b) { return u128v{mulhi64(a, b), a * b}; }
DV void acc_wide(u128v& acc, u64 a, u64 b) {
    u64 lo = a * b, hi = mulhi64(a, b);
    acc.lo += lo;
    acc.hi += hi + (acc.lo < lo ? 1ull : 0ull);
}

// Barrett reduction of x < 2^128 (with x / q < 2^64) modulo q, given
// ratio = floor(2^128 / q) = (r1, r0).  Returns the canonical residue.
DV u64 barrett128(u128v x, u64 q, u64 r1, u64 r0) {
    u64 carry = mulhi64(x.lo, r0);
    u64 t2lo = x.lo * r1, t2hi = mulhi64(x.lo, r1);
    u64 t1 = t2lo + carry;
    u64 t3 = t2hi + (t1 < carry ? 1ull : 0ull);
    u64 slo = x.hi * r0, shi = mulhi64(x.hi, r0);
    u64 s = t1 + slo;
    carry = shi + (s < t1 ? 1ull : 0ull);
    u64 qe = x.hi * r1 + t3 + carry;
    u64 r = x.lo - qe * q;  // in [0, 2q) for x < 2^126, [0, 3q) otherwise
    return csub(csub(r, q), q);
}
DV u64 mul_mod(u64 a, u64 b, u64 q, u64 r1, u64 r0) { return barrett128(mul_wide(a, b), q, r1, r0); }

// ---- counter-based randomness: identical to oracle/ckks_oracle.c --------
HD u64 mix64(u64 z) {
    z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27; z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
}
HD u64 prng_key(u64 seed, u64 stream) { return mix64(seed ^ mix64(stream + 0x9E3779B97F4A7C15ULL)); }
HD u64 prng_at(u64 key, u64 ctr) { return mix64(key + (ctr + 1) * 0x9E3779B97F4A7C15ULL); }
HD u64 stream_id(u64 kind, u64 id, u64 sub, u64 purpose) {
    return (kind << 56) ^ (id << 8) ^ (sub << 4) ^ purpose;
}
#define ST_SK 1ULL
#define ST_CT 2ULL
#define ST_KEY 3ULL
#define PU_A 1ULL
#define PU_E 2ULL
#define PU_S 3ULL

// (hi * 2^64 + lo) mod q, canonical
DV u64 uniform_from(u64 lo, u64 hi, u64 q, u64 r1, u64 r0) {
    // hi*2^64 + lo may exceed q*2^64, so first fold hi below q.
    u64 h = hi % q;
    return barrett128(u128v{h, lo}, q, r1, r0);
}
DV long long cbd_from(u64 r, int eta) {
    u64 mask = eta >= 32 ? 0xffffffffull : ((1ull << eta) - 1);
    return (long long)__popcll(r & mask) - (long long)__popcll((r >> 32) & mask);
}
DV u64 reduce_i64(long long v, u64 q) {
    if (v >= 0) return (u64)v % q;
    u64 m = (u64)(-(v + 1)) % q;
    return q - 1 - m;
}
