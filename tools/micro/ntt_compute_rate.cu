// fp64 butterfly throughput of the NTT register stages alone (no global
// memory): 16 doubles per thread, 4 radix-2 stages per iteration with the
// exact 6-instruction twiddle product, twiddles from shared memory.
// Reports fp64 warp-instructions per clock per SM sub-partition (pipe peak 0.5)
// for 1..4 resident 256-thread CTAs per SM (64 registers), and the dependent
// DFMA latency.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ntt_compute_rate ntt_compute_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr double MAGIC = 6755399441055744.0;
struct DblC { double q, qinv; };
__device__ __forceinline__ double mulmod_d(double a, double w, const DblC& c) {
    const double p = __dmul_rn(a, w);
    const double e = __fma_rn(a, w, -p);
    const double h = __dsub_rn(__fma_rn(p, c.qinv, MAGIC), MAGIC);
    return __dadd_rn(__fma_rn(-h, c.q, p), e);
}
template <int H>
__device__ __forceinline__ void stage(double (&x)[16], const double* W, int tb0, const DblC& c) {
#pragma unroll
    for (int j = 0; j < (16 >> (H + 1)); j++) {
        const double w = W[tb0 + j];
#pragma unroll
        for (int t = 0; t < (1 << H); t++) {
            const int i = (j << (H + 1)) + t;
            const double u = x[i], v = mulmod_d(x[i + (1 << H)], w, c);
            x[i] = u + v;
            x[i + (1 << H)] = u - v;
        }
    }
}
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k(double* out, int iters, double q) {
    __shared__ double tw[256];
    tw[threadIdx.x] = 1000.0 + threadIdx.x * 3.0;
    __syncthreads();
    DblC c{q, 1.0 / q};
    double x[16];
    for (int i = 0; i < 16; i++) x[i] = threadIdx.x * 17.0 + i;
    const int s = threadIdx.x & 15;
    for (int it = 0; it < iters; it++) {
        stage<3>(x, tw, 1, c);
        stage<2>(x, tw, 2, c);
        stage<1>(x, tw, 4, c);
        stage<0>(x, tw, 8, c);
        stage<3>(x, tw, 16 + s, c);
        stage<2>(x, tw, 32 + 2 * s, c);
        stage<1>(x, tw, 64 + 4 * s, c);
        stage<0>(x, tw, 128 + 8 * s, c);
    }
    double a = 0;
    for (int i = 0; i < 16; i++) a += x[i];
    out[blockIdx.x * 256 + threadIdx.x] = a;
}
__global__ void lat(double* out, int iters, long long* cyc) {
    double d = threadIdx.x;
    const long long t0 = clock64();
    for (int i = 0; i < iters; i++) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d) : "d"(0.999999));
    const long long t1 = clock64();
    out[threadIdx.x] = d;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int MINB>
void run(int sms, double clk_hz, int ctas_per_sm) {
    double* out;
    cudaMalloc(&out, 8 * 256 * sms * 8);
    const int iters = 2000, blocks = sms * ctas_per_sm;
    k<MINB><<<blocks, 256>>>(out, 10, 1099511480321.0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MINB><<<blocks, 256>>>(out, iters, 1099511480321.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double wi = (double)blocks * 8 * iters * 64 * 8;  // warps x iters x butterflies x 8 fp64
    printf("MINB %d, %d CTAs/SM (%d warps/SMSP): %.3f fp64 warp-instr/clk/SMSP\n", MINB, ctas_per_sm, ctas_per_sm * 2,
           wi / (ms * 1e-3 * clk_hz) / sms / 4);
    cudaFree(out);
}
int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    int khz; cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double hz = khz * 1e3;
    printf("%s, %d SMs, %.0f MHz\n", p.name, p.multiProcessorCount, hz / 1e6);
    double* out; long long* cyc;
    cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8);
    lat<<<1, 32>>>(out, 4096, cyc);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dependent DFMA latency: %.1f cycles\n", h / 4096.0);
    for (int c = 1; c <= 4; c++) run<4>(p.multiProcessorCount, hz, c);
    for (int c = 1; c <= 3; c++) run<3>(p.multiProcessorCount, hz, c);
    for (int c = 1; c <= 2; c++) run<2>(p.multiProcessorCount, hz, c);
    return 0;
}
