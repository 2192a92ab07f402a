// int_peak.cu — integer-throughput microbenchmark for the B200 roofline
// ("measure with a VIMNMX/VIADDMNMX/ISETP
// microbenchmark"). Each kernel runs NCH independent dependency chains of one
// instruction form per thread, 8 warps x 4 blocks per SM (enough to hide the
// 4-cycle ALU / FMA latency), and reports thread-ops per SM clock measured
// with clock64() inside each block (independent of the clock frequency).
//
// Forms (the SASS the X-drop cell uses; `cuobjdump -sass` of this binary
// confirms each): VIMNMX3 (3-input max, __vimax3_s32), VIADDMNMX
// (__viaddmax_s32), VIMNMX.U32 (min_u32), LOP3, IADD3, SHF (funnel shift),
// IMAD (FMA pipe), the packed .S16x2 forms VIMNMX3.S16x2 / VIADDMNMX.S16x2
// (2 lanes per op), and a 1:1 mix of VIMNMX3 and IMAD (ALU + FMA pipes
// together: the issue-slot bound).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peak int_peak.cu
//   ./int_peak  -> one JSON object on stdout
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NCH = 8;      // independent chains per thread
constexpr int ITERS = 4096; // loop trips (each: NCH ops)
constexpr int THREADS = 256;

enum Op { VMAX3, VADDMAX, VMINU32, LOP3, IADD3, SHF, IMAD, VMAX3_S16X2, VADDMAX_S16X2, MIX_VMAX3_IMAD, VADD16X2, PRMT,
          MIX_VADD16X2_VMAX3, MIX_PRMT_IMAD, IMADHI, IMADSHL, VADDMIN_U16X2, MIX_2VMAX3_IMAD, NOPS };
static const char *kName[NOPS] = {"VIMNMX3", "VIADDMNMX", "VIMNMX.U32", "LOP3", "IADD3", "SHF", "IMAD",
                                  "VIMNMX3.S16x2", "VIADDMNMX.S16x2", "VIMNMX3+IMAD (1:1)", "VIADD.16x2", "PRMT",
                                  "VIADD.16x2+VIMNMX3 (1:1)", "PRMT+IMAD (1:1)", "IMAD.HI", "IMAD.SHL",
                                  "VIADDMNMX.U16x2", "VIMNMX3+IMAD (2:1)"};
static const int kLanesPerOp[NOPS] = {1, 1, 1, 1, 1, 1, 1, 2, 2, 1, 2, 1, 1, 1, 1, 1, 2, 1};

template <int OP>
__global__ void __launch_bounds__(THREADS) k_op(uint32_t seed, uint32_t *sink, unsigned long long *cyc) {
    uint32_t a[NCH];
    const uint32_t b = seed * 3u + threadIdx.x, c = seed ^ 0x5bd1e995u, d = seed + 7u;
#pragma unroll
    for (int q = 0; q < NCH; ++q) a[q] = seed + q * 0x9e3779b9u + threadIdx.x;
    __syncthreads();
    const unsigned long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int q = 0; q < NCH; ++q) {
            if (OP == VMAX3) a[q] = (uint32_t)__vimax3_s32((int)a[q], (int)b, (int)c);
            if (OP == VADDMAX) a[q] = (uint32_t)__viaddmax_s32((int)a[q], (int)b, (int)c);
            if (OP == VMINU32) asm volatile("min.u32 %0, %0, %1;" : "+r"(a[q]) : "r"(b));
            if (OP == LOP3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[q]) : "r"(b), "r"(c));
            if (OP == IADD3) asm volatile("add.s32 %0, %0, %1;" : "+r"(a[q]) : "r"(b));
            if (OP == SHF) a[q] = __funnelshift_l(a[q], b, c & 31u);
            if (OP == IMAD) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[q]) : "r"(b), "r"(c));
            if (OP == VMAX3_S16X2) a[q] = (uint32_t)__vimax3_s16x2((int)a[q], (int)b, (int)c);
            if (OP == VADDMAX_S16X2) a[q] = (uint32_t)__viaddmax_s16x2((int)a[q], (int)b, (int)c);
            if (OP == VADD16X2) asm volatile("add.s16x2 %0, %0, %1;" : "+r"(a[q]) : "r"(b));
            if (OP == PRMT) a[q] = __byte_perm(a[q], b, 0x5432);
            if (OP == MIX_VADD16X2_VMAX3) {
                if (q & 1) asm volatile("add.s16x2 %0, %0, %1;" : "+r"(a[q]) : "r"(b));
                else a[q] = (uint32_t)__vimax3_s32((int)a[q], (int)b, (int)d);
            }
            if (OP == MIX_PRMT_IMAD) {
                if (q & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[q]) : "r"(b), "r"(c));
                else a[q] = __byte_perm(a[q], b, 0x5432);
            }
            if (OP == IMADHI) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[q]) : "r"(b), "r"(c));
            if (OP == IMADSHL) asm volatile("mul.lo.u32 %0, %0, 16;" : "+r"(a[q]));
            if (OP == VADDMIN_U16X2) a[q] = __viaddmin_u16x2(a[q], b, c);
            if (OP == MIX_2VMAX3_IMAD) {
                if (q % 3 == 2) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[q]) : "r"(b), "r"(c));
                else a[q] = (uint32_t)__vimax3_s32((int)a[q], (int)b, (int)d);
            }
            if (OP == MIX_VMAX3_IMAD) {
                if (q & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[q]) : "r"(b), "r"(c));
                else a[q] = (uint32_t)__vimax3_s32((int)a[q], (int)b, (int)d);
            }
        }
    }
    const unsigned long long t1 = clock64();
    uint32_t x = 0;
#pragma unroll
    for (int q = 0; q < NCH; ++q) x ^= a[q];
    if (x == 0x12345678u) sink[0] = x;  // keeps the chains alive
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// SASS instructions per chain step of each form
static const int kInstPerStep[NOPS] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};

template <int OP>
static double run(int sms, int blocks_per_sm, uint32_t *sink, unsigned long long *cyc) {
    const int grid = sms * blocks_per_sm;
    k_op<OP><<<grid, THREADS>>>(1u, sink, cyc);  // warm-up
    k_op<OP><<<grid, THREADS>>>(2u, sink, cyc);
    cudaDeviceSynchronize();
    unsigned long long *h = new unsigned long long[grid];
    cudaMemcpy(h, cyc, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    delete[] h;
    // all blocks of an SM are co-resident: per-SM thread-instructions / the slowest block's cycles
    const double inst = (double)blocks_per_sm * THREADS * ITERS * NCH * kInstPerStep[OP];
    return inst / (double)mx;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, dev);
    uint32_t *sink;
    unsigned long long *cyc;
    cudaMalloc(&sink, 4);
    cudaMalloc(&cyc, sizeof(unsigned long long) * sms * 8);
    const int bps = 4;  // 4 x 256 threads = 32 warps per SM
    double r[NOPS];
    r[VMAX3] = run<VMAX3>(sms, bps, sink, cyc);
    r[VADDMAX] = run<VADDMAX>(sms, bps, sink, cyc);
    r[VMINU32] = run<VMINU32>(sms, bps, sink, cyc);
    r[LOP3] = run<LOP3>(sms, bps, sink, cyc);
    r[IADD3] = run<IADD3>(sms, bps, sink, cyc);
    r[SHF] = run<SHF>(sms, bps, sink, cyc);
    r[IMAD] = run<IMAD>(sms, bps, sink, cyc);
    r[VMAX3_S16X2] = run<VMAX3_S16X2>(sms, bps, sink, cyc);
    r[VADDMAX_S16X2] = run<VADDMAX_S16X2>(sms, bps, sink, cyc);
    r[MIX_VMAX3_IMAD] = run<MIX_VMAX3_IMAD>(sms, bps, sink, cyc);
    r[VADD16X2] = run<VADD16X2>(sms, bps, sink, cyc);
    r[PRMT] = run<PRMT>(sms, bps, sink, cyc);
    r[MIX_VADD16X2_VMAX3] = run<MIX_VADD16X2_VMAX3>(sms, bps, sink, cyc);
    r[MIX_PRMT_IMAD] = run<MIX_PRMT_IMAD>(sms, bps, sink, cyc);
    r[IMADHI] = run<IMADHI>(sms, bps, sink, cyc);
    r[IMADSHL] = run<IMADSHL>(sms, bps, sink, cyc);
    r[VADDMIN_U16X2] = run<VADDMIN_U16X2>(sms, bps, sink, cyc);
    r[MIX_2VMAX3_IMAD] = run<MIX_2VMAX3_IMAD>(sms, bps, sink, cyc);
    if (cudaGetLastError() != cudaSuccess) { fprintf(stderr, "CUDA error\n"); return 1; }
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d, \"threads_per_sm\": %d, \"inst_per_clk_per_sm\": {",
           p.name, sms, clk, bps * THREADS);
    for (int o = 0; o < NOPS; ++o)
        printf("%s\"%s\": %.2f", o ? ", " : "", kName[o], r[o]);
    printf("}, \"lanes_per_op\": {");
    for (int o = 0; o < NOPS; ++o) printf("%s\"%s\": %d", o ? ", " : "", kName[o], kLanesPerOp[o]);
    printf("}}\n");
    return 0;
}
