// Integer/FP multiply issue rates on sm_100a: warp-instructions per clock per
// SM for IMAD (lo), IMAD.HI, IMAD.WIDE, 64-bit mul.lo/mul.hi, DFMA, FFMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imad_rate imad_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 2048
#define CH 8

template <int OP>
__global__ void k(uint64_t* out, uint32_t seed) {
    uint32_t a[CH];
    uint64_t w[CH];
    double d[CH];
    float f[CH];
    for (int c = 0; c < CH; c++) {
        a[c] = seed * (threadIdx.x + 7 * c + 1);
        w[c] = (uint64_t)a[c] * 0x9E3779B97F4A7C15ull;
        d[c] = 1.0 + a[c] * 1e-12;
        f[c] = 1.0f + a[c] * 1e-9f;
    }
    const uint32_t m = seed | 1;
    const uint64_t m64 = 0x9E3779B97F4A7C15ull ^ seed;
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int c = 0; c < CH; c++) {
            if (OP == 0) asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(a[c]) : "r"(m));
            if (OP == 1) asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(a[c]) : "r"(m));
            if (OP == 2) {
                uint64_t r;
                asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"((uint32_t)w[c]), "r"(m), "l"(w[c]));
                w[c] = r;
            }
            if (OP == 3) asm volatile("mul.lo.u64 %0, %0, %1;" : "+l"(w[c]) : "l"(m64));
            if (OP == 4) asm volatile("mul.hi.u64 %0, %0, %1;" : "+l"(w[c]) : "l"(m64));
            if (OP == 5) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[c]) : "d"(0.999999));
            if (OP == 6) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f[c]) : "f"(0.999f));
            if (OP == 7) {  // u64 -> f64 -> u64 round trip (I2F.F64.U64 + F2I.U64.F64)
                double t;
                asm volatile("cvt.rn.f64.u64 %0, %1;" : "=d"(t) : "l"(w[c]));
                asm volatile("cvt.rzi.u64.f64 %0, %1;" : "=l"(w[c]) : "d"(t));
            }
            if (OP == 8) asm volatile("cvt.rmi.f64.f64 %0, %0;" : "+d"(d[c]));  // floor
            if (OP == 9) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(d[c]) : "d"(1.0000001));
            if (OP == 10) {  // 32-bit -> f64 (I2F.F64.U32)
                double t;
                asm volatile("cvt.rn.f64.u32 %0, %1;" : "=d"(t) : "r"(a[c]));
                d[c] += t;
            }
        }
    }
    uint64_t s = 0;
    for (int c = 0; c < CH; c++) s += a[c] + w[c] + (uint64_t)d[c] + (uint64_t)f[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
void run(const char* name, int sms, int clk_khz) {
    uint64_t* out;
    const int blocks = sms * 8, threads = 256;
    cudaMalloc(&out, sizeof(uint64_t) * blocks * threads);
    k<OP><<<blocks, threads>>>(out, 3);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<OP><<<blocks, threads>>>(out, 5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_instr = (double)blocks * threads / 32 * ITERS * CH;
    const double clocks = ms * 1e-3 * clk_khz * 1e3;
    printf("%-14s %.3f ms  %.3f warp-instr/clk/SM (%.3f per SMSP)\n", name, ms, warp_instr / clocks / sms,
           warp_instr / clocks / sms / 4);
    cudaFree(out);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, clk);
    run<0>("IMAD lo32", p.multiProcessorCount, clk);
    run<1>("IMAD.HI", p.multiProcessorCount, clk);
    run<2>("IMAD.WIDE", p.multiProcessorCount, clk);
    run<3>("mul.lo.u64", p.multiProcessorCount, clk);
    run<4>("mul.hi.u64", p.multiProcessorCount, clk);
    run<5>("DFMA", p.multiProcessorCount, clk);
    run<6>("FFMA", p.multiProcessorCount, clk);
    run<7>("cvt u64>f64>u64", p.multiProcessorCount, clk);
    run<8>("floor f64", p.multiProcessorCount, clk);
    run<9>("DMUL", p.multiProcessorCount, clk);
    run<10>("cvt u32>f64 +DADD", p.multiProcessorCount, clk);
    return 0;
}
