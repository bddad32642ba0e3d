// metrics.cu — training-harness metrics on the device (SURVEY.md §8(f) row 4:
// the per-iteration metrics of train_encrypted, enctrain.py:417-436, built
// from optim.py:123-126 log_likelihood, optim.py:200-206 predict / accuracy
// and optim.py:209-229 auroc).
//
//   scores s_i = X_i . w   (X row-major n x d, the bias column included)
//   log_likelihood = -mean_i logaddexp(0, -y_i s_i)
//   accuracy       = mean_i [sign(s_i) == y_i]   (s_i >= 0 -> +1)
//   auroc          = (sum of positive midranks - n_pos (n_pos + 1) / 2) / (n_pos n_neg)
//
// The midrank sum uses a bitonic sort of the scores (padded to a power of
// two with +inf) and, per element, a binary search for its tie group; the
// midranks are half-integers, so their sum is exact in fp64 and the AUROC is
// the reference's value for the same scores.  Sums are reduced per block and
// then in one block in a fixed order (deterministic).
#include <cmath>

#include "../../include/helr_ckks.h"
#include "ctx.cuh"

namespace {

constexpr int MT = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) t += sh[i];
    return t;  // valid in thread 0
}

// one warp per row: s_i, and the per-block partial sums of the log-likelihood
// terms and of the correct predictions
__global__ void k_scores(const double* __restrict__ X, const double* __restrict__ y, const double* __restrict__ w,
                         int n, int d, double* __restrict__ s, double* __restrict__ part) {
    __shared__ double sh[MT / 32];
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    double ll = 0.0, ok = 0.0, np = 0.0;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        const double* xi = X + (size_t)i * d;
        double acc = 0.0;
        for (int j = lane; j < d; j += 32) acc = fma(xi[j], w[j], acc);
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            s[i] = acc;
            const double u = -y[i] * acc;  // logaddexp(0, u) = max(0, u) + log1p(exp(-|u|))
            ll += fmax(0.0, u) + log1p(exp(-fabs(u)));
            ok += ((acc >= 0.0 ? 1.0 : -1.0) == y[i]) ? 1.0 : 0.0;
            np += y[i] > 0.0 ? 1.0 : 0.0;
        }
    }
    const double a = block_sum(ll, sh);
    const double b = block_sum(ok, sh);
    const double e = block_sum(np, sh);
    if (threadIdx.x == 0) {
        part[3 * blockIdx.x] = a;
        part[3 * blockIdx.x + 1] = b;
        part[3 * blockIdx.x + 2] = e;
    }
}

__global__ void k_pad(const double* s, double* key, int n, int npad) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npad; i += gridDim.x * blockDim.x)
        key[i] = i < n ? s[i] : INFINITY;
}

// one bitonic compare-exchange step (k: sequence size, j: distance), ascending
__global__ void k_bitonic(double* key, int npad, int k, int j) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npad; i += gridDim.x * blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
            const double a = key[i], b = key[l];
            const bool up = (i & k) == 0;
            if ((a > b) == up) { key[i] = b; key[l] = a; }
        }
    }
}

// per positive element: its midrank among the sorted scores (lower / upper
// bound of its tie group), summed per block
__global__ void k_midranks(const double* __restrict__ s, const double* __restrict__ y,
                           const double* __restrict__ sorted, int n, double* __restrict__ part) {
    __shared__ double sh[MT / 32];
    double acc = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (!(y[i] > 0.0)) continue;
        const double v = s[i];
        int lo = 0, hi = n;  // first index with sorted >= v
        while (lo < hi) { const int m = (lo + hi) >> 1; if (sorted[m] < v) lo = m + 1; else hi = m; }
        const int first = lo;
        hi = n;  // first index with sorted > v
        while (lo < hi) { const int m = (lo + hi) >> 1; if (sorted[m] <= v) lo = m + 1; else hi = m; }
        acc += 0.5 * (double)(first + lo - 1) + 1.0;
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// fixed-order final sums: out[c] = sum_b part[b * stride + c]
__global__ void k_final(const double* part, int nb, int stride, int comps, double* out) {
    __shared__ double sh[MT / 32];
    for (int c = 0; c < comps; c++) {
        double v = 0.0;
        for (int b = threadIdx.x; b < nb; b += blockDim.x) v += part[(size_t)b * stride + c];
        const double t = block_sum(v, sh);
        if (threadIdx.x == 0) out[c] = t;
    }
}

}  // namespace

// out[0] = log_likelihood, out[1] = accuracy, out[2] = auroc (NaN when only one
// class is present, where the reference raises), out[3] = n_pos (host array).
// X: n x d row-major (bias column included), y in {-1, +1}, w: d; device
// pointers; scratch: helr_metrics_scratch(n) doubles.
extern "C" size_t helr_metrics_scratch(int n) {
    size_t npad = 1;
    while (npad < (size_t)n) npad <<= 1;
    return (size_t)n + npad + 5 * 1184 + 8;
}

extern "C" int helr_metrics(helr_ctx* c, const double* X, const double* y, const double* w, int n, int d,
                            double* scratch, double* out, void* stream) {
    clear_stale_error("helr_metrics");
    (void)c;
    if (n < 1 || d < 1) { set_error("metrics: empty data"); return HELR_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    int npad = 1;
    while (npad < n) npad <<= 1;
    const int nb = 1184;  // 8 blocks per SM
    double* sc = scratch;                 // [n] scores
    double* key = sc + n;                 // [npad] sorted scores
    double* part = key + npad;            // [3 * nb] partials
    double* part2 = part + 3 * nb;        // [nb]
    double* tmp = part2 + 2 * nb;         // [8]
    k_scores<<<nb, MT, 0, s>>>(X, y, w, n, d, sc, part);
    k_pad<<<nb, MT, 0, s>>>(sc, key, n, npad);
    for (int k = 2; k <= npad; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) k_bitonic<<<nb, MT, 0, s>>>(key, npad, k, j);
    k_midranks<<<nb, MT, 0, s>>>(sc, y, key, n, part2);
    k_final<<<1, MT, 0, s>>>(part, nb, 3, 3, tmp);
    k_final<<<1, MT, 0, s>>>(part2, nb, 1, 1, tmp + 3);
    double h[4];
    cudaMemcpyAsync(h, tmp, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (!cuda_ok(cudaStreamSynchronize(s), "metrics")) return HELR_ECUDA;
    const double npos = h[2], nneg = (double)n - h[2];
    out[0] = -h[0] / n;
    out[1] = h[1] / n;
    out[2] = (npos > 0.0 && nneg > 0.0) ? (h[3] - npos * (npos + 1.0) / 2.0) / (npos * nneg) : NAN;
    out[3] = npos;
    return HELR_OK;
}
