// encode.cu — device-side CKKS encoding / decoding (client side; SURVEY.md
// §8(f) row 2: client_prepare at enctrain.py:114-152 and decode_weights at
// enctrain.py:266-289, whose SimContext.enc / dec are hesim.py:146-162).
//
// A slot vector z in C^(N/2) is the real polynomial m with m(zeta^(5^j)) = z_j
// and m(zeta^(-5^j)) = conj(z_j), zeta = exp(i pi / N) — the same canonical
// embedding as the host encoder (encoder.py).  With ev[t] the evaluation at
// zeta^(2t+1), m_i = Re(zeta^(-i) * FFT(ev)_i) / N (FFT sign -1), and the
// coefficients are rint(scale * m_i).  Decoding is the transpose: z_j =
// sum_i c_i zeta^i exp(+2 pi i t i / N) at t = (5^j - 1) / 2, divided by scale.
//
// The length-N complex FFT runs as log2 N radix-2 Stockham passes over a
// whole chunk of messages (fp64, natural order in and out); each pass reads
// and writes the chunk once, so encoding is HBM-bound and the host never
// touches a coefficient.  Results can differ from the host encoder's numpy
// FFT by one unit in a coefficient when a value lies within rounding error of
// a half-integer (a 2^-40 relative change of one coefficient; parity is a
// tolerance test, tests/test_gpu_encode.py).
#include <cstdio>
#include <vector>

#include "../../include/helr_ckks.h"
#include "ks.cuh"

namespace {

struct EncTables {
    int log_n = 0;
    double2* tw = nullptr;  // [N/2] exp(-2 pi i k / N)
    int* tpos = nullptr;    // [N/2] slot j -> evaluation index (5^j - 1) / 2
    int* tneg = nullptr;    // [N/2] conj slot j -> (2N - 5^j - 1) / 2
};

__global__ void k_fft_twiddles(double2* tw, int n) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n / 2) return;
    double s, c;
    sincospi(-2.0 * (double)k / (double)n, &s, &c);
    tw[k] = make_double2(c, s);
}

int enc_tables(helr_ctx* c, EncTables& t, cudaStream_t s) {
    // owned by the context (freed by helr_ctx_destroy)
    t.log_n = c->log_n;
    if (c->enc_tw) {
        t.tw = (double2*)c->enc_tw; t.tpos = c->enc_tpos; t.tneg = c->enc_tneg;
        return HELR_OK;
    }
    const int n = c->n, S = n / 2;
    std::vector<int> tp(S), tn(S);
    long long pw = 1;
    for (int j = 0; j < S; j++) {
        tp[j] = (int)((pw - 1) / 2);
        tn[j] = (int)((2ll * n - pw - 1) / 2);
        pw = (pw * 5) % (2ll * n);
    }
    double2* tw = nullptr;
    int *pos = nullptr, *neg = nullptr;
    if (!cuda_ok(cudaMalloc(&tw, sizeof(double2) * S), "cudaMalloc(fft twiddles)")) return HELR_ENOMEM;
    if (!cuda_ok(cudaMalloc(&pos, sizeof(int) * S), "cudaMalloc(slot map)")) { cudaFree(tw); return HELR_ENOMEM; }
    if (!cuda_ok(cudaMalloc(&neg, sizeof(int) * S), "cudaMalloc(slot map)")) {
        cudaFree(tw); cudaFree(pos); return HELR_ENOMEM;
    }
    cudaMemcpyAsync(pos, tp.data(), sizeof(int) * S, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(neg, tn.data(), sizeof(int) * S, cudaMemcpyHostToDevice, s);
    k_fft_twiddles<<<(S + 255) / 256, 256, 0, s>>>(tw, n);
    if (!cuda_ok(cudaStreamSynchronize(s), "encode tables")) return HELR_ECUDA;
    c->enc_tw = tw; c->enc_tpos = pos; c->enc_tneg = neg;
    t.tw = tw; t.tpos = pos; t.tneg = neg;
    return HELR_OK;
}

// ev[b][tpos[j]] = z_j, ev[b][tneg[j]] = conj(z_j)
__global__ void k_enc_scatter(const double* re, const double* im, long long zs, double2* ev, EncTables t, int n,
                              int count) {
    const int S = n / 2;
    const long long total = (long long)count * S;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(idx / S), j = (int)(idx - (long long)b * S);
        const double x = re[(size_t)b * zs + j];
        const double y = im ? im[(size_t)b * zs + j] : 0.0;
        double2* e = ev + (size_t)b * n;
        e[t.tpos[j]] = make_double2(x, y);
        e[t.tneg[j]] = make_double2(x, -y);
    }
}

// one radix-2 Stockham pass (stage st, n' = N >> st, stride s = 2^st):
// y[q + s 2p] = a + b, y[q + s (2p+1)] = (a - b) w^(p s), a = x[q + s p],
// b = x[q + s (p + n'/2)]; sign < 0: w = exp(-2 pi i / N), else its conjugate
__global__ void k_fft_pass(const double2* __restrict__ x, double2* __restrict__ y, const double2* __restrict__ tw,
                           int log_n, int st, int sign, int count) {
    const int n = 1 << log_n, half = n >> 1;
    const long long total = (long long)count * half;
    const int m = half >> st;  // n' / 2
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(idx >> (log_n - 1));
        const int t = (int)(idx & (half - 1));
        const int q = t & ((1 << st) - 1), p = t >> st;
        const double2* xb = x + (size_t)b * n;
        double2* yb = y + (size_t)b * n;
        const double2 u = xb[q + (p << st)], v = xb[q + ((p + m) << st)];
        double2 w = tw[p << st];
        if (sign > 0) w.y = -w.y;
        const double dx = __dsub_rn(u.x, v.x), dy = __dsub_rn(u.y, v.y);
        yb[q + ((2 * p) << st)] = make_double2(__dadd_rn(u.x, v.x), __dadd_rn(u.y, v.y));
        yb[q + ((2 * p + 1) << st)] =
            make_double2(__dsub_rn(__dmul_rn(dx, w.x), __dmul_rn(dy, w.y)), __dadd_rn(__dmul_rn(dx, w.y), __dmul_rn(dy, w.x)));
    }
}

// coef_i = rint(Re(zeta^-i b_i) * scale / N); flags |value| >= 2^62
__global__ void k_enc_round(const double2* b, long long* coef, int log_n, double scale_over_n, int count, int* bad) {
    const int n = 1 << log_n;
    const long long total = (long long)count * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx & (n - 1));
        double s, c;
        sincospi(-(double)i / (double)n, &s, &c);  // zeta^-i
        const double2 v = b[idx];
        const double re = __dsub_rn(__dmul_rn(v.x, c), __dmul_rn(v.y, s));
        const double m = __dmul_rn(re, scale_over_n);
        if (!(fabs(m) < 4.611686018427387904e18)) { *bad = 1; coef[idx] = 0; continue; }
        coef[idx] = __double2ll_rn(m);
    }
}

// decode prologue: ev_i = c_i zeta^i
__global__ void k_dec_twist(const long long* coef, double2* ev, int log_n, int count) {
    const int n = 1 << log_n;
    const long long total = (long long)count * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx & (n - 1));
        double s, c;
        sincospi((double)i / (double)n, &s, &c);
        const double x = (double)coef[idx];
        ev[idx] = make_double2(__dmul_rn(x, c), __dmul_rn(x, s));
    }
}

__global__ void k_dec_gather(const double2* ev, double* re, double* im, long long zs, EncTables t, int n,
                             double inv_scale, int count) {
    const int S = n / 2;
    const long long total = (long long)count * S;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(idx / S), j = (int)(idx - (long long)b * S);
        const double2 v = ev[(size_t)b * n + t.tpos[j]];
        re[(size_t)b * zs + j] = __dmul_rn(v.x, inv_scale);
        if (im) im[(size_t)b * zs + j] = __dmul_rn(v.y, inv_scale);
    }
}

int grid_for(long long total) {
    long long g = (total + 255) / 256;
    return (int)(g < 148 * 32 ? g : 148 * 32);
}

// log2 N passes ping-ponging between a and b; returns the buffer holding the result
double2* fft_run(double2* a, double2* b, const EncTables& t, int log_n, int sign, int count, cudaStream_t s) {
    const long long total = (long long)count << (log_n - 1);
    for (int st = 0; st < log_n; st++) {
        k_fft_pass<<<grid_for(total), 256, 0, s>>>(a, b, t.tw, log_n, st, sign, count);
        count_launches(1);
        double2* tmp = a; a = b; b = tmp;
    }
    return a;
}

constexpr int ENC_CHUNK = 64;  // messages per FFT batch (2 x 64 x N x 16 B of scratch)

}  // namespace

extern "C" int helr_encode(helr_ctx* c, const double* re, const double* im, int64_t slot_stride, int count,
                           double scale, int64_t* coef, void* stream) {
    clear_stale_error("helr_encode");
    if (count < 0 || slot_stride < c->n / 2) { set_error("encode: bad count or slot stride"); return HELR_EINVAL; }
    if (!(scale > 0.0)) { set_error("encode: scale must be positive"); return HELR_EINVAL; }
    if (count == 0) return HELR_OK;
    cudaStream_t s = (cudaStream_t)stream;
    EncTables t;
    int r = enc_tables(c, t, s);
    if (r) return r;
    const int n = c->n;
    const int ch = count < ENC_CHUNK ? count : ENC_CHUNK;
    double2* buf = nullptr;
    int* bad = nullptr;
    if (!cuda_ok(cudaMallocAsync(&buf, sizeof(double2) * 2 * (size_t)ch * n, s), "cudaMallocAsync(encode)"))
        return HELR_ENOMEM;
    if (!cuda_ok(cudaMallocAsync(&bad, sizeof(int), s), "cudaMallocAsync(encode)")) return HELR_ENOMEM;
    cudaMemsetAsync(bad, 0, sizeof(int), s);
    for (int b0 = 0; b0 < count; b0 += ch) {
        const int nb = count - b0 < ch ? count - b0 : ch;
        double2* a = buf;
        double2* b = buf + (size_t)ch * n;
        cudaMemsetAsync(a, 0, sizeof(double2) * (size_t)nb * n, s);
        k_enc_scatter<<<grid_for((long long)nb * n / 2), 256, 0, s>>>(re + (size_t)b0 * slot_stride,
                                                                       im ? im + (size_t)b0 * slot_stride : nullptr,
                                                                       slot_stride, a, t, n, nb);
        count_launches(1);
        double2* res = fft_run(a, b, t, c->log_n, -1, nb, s);
        k_enc_round<<<grid_for((long long)nb * n), 256, 0, s>>>(res, (long long*)coef + (size_t)b0 * n, c->log_n,
                                                                scale / (double)n, nb, bad);
        count_launches(1);
    }
    int hbad = 0;
    cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(buf, s);
    cudaFreeAsync(bad, s);
    if (!cuda_ok(cudaStreamSynchronize(s), "encode")) return HELR_ECUDA;
    if (hbad) { set_error("encoded coefficient exceeds 2**62; lower the scale or the values"); return HELR_EINVAL; }
    return HELR_OK;
}

extern "C" int helr_decode(helr_ctx* c, const int64_t* coef, int count, double scale, double* re, double* im,
                           int64_t slot_stride, void* stream) {
    clear_stale_error("helr_decode");
    if (count < 0 || slot_stride < c->n / 2) { set_error("decode: bad count or slot stride"); return HELR_EINVAL; }
    if (!(scale > 0.0)) { set_error("decode: scale must be positive"); return HELR_EINVAL; }
    if (count == 0) return HELR_OK;
    cudaStream_t s = (cudaStream_t)stream;
    EncTables t;
    int r = enc_tables(c, t, s);
    if (r) return r;
    const int n = c->n;
    const int ch = count < ENC_CHUNK ? count : ENC_CHUNK;
    double2* buf = nullptr;
    if (!cuda_ok(cudaMallocAsync(&buf, sizeof(double2) * 2 * (size_t)ch * n, s), "cudaMallocAsync(decode)"))
        return HELR_ENOMEM;
    for (int b0 = 0; b0 < count; b0 += ch) {
        const int nb = count - b0 < ch ? count - b0 : ch;
        double2* a = buf;
        double2* b = buf + (size_t)ch * n;
        k_dec_twist<<<grid_for((long long)nb * n), 256, 0, s>>>((const long long*)coef + (size_t)b0 * n, a, c->log_n,
                                                               nb);
        count_launches(1);
        double2* res = fft_run(a, b, t, c->log_n, +1, nb, s);
        k_dec_gather<<<grid_for((long long)nb * n / 2), 256, 0, s>>>(res, re + (size_t)b0 * slot_stride,
                                                                      im ? im + (size_t)b0 * slot_stride : nullptr,
                                                                      slot_stride, t, n, 1.0 / scale, nb);
        count_launches(1);
    }
    cudaFreeAsync(buf, s);
    if (!cuda_ok(cudaGetLastError(), "decode")) return HELR_ECUDA;
    return HELR_OK;
}
