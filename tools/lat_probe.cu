// lat_probe.cu — dependent-chain latencies (cycles) of the instructions on the
// X-drop sweep's per-antidiagonal critical path (the latency
// shape): one warp alone on the GPU runs a chain of N dependent instances and
// divides clock64() cycles by N.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_probe lat_probe.cu && ./lat_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int N = 4096;

enum Op { ALU_VIMNMX3, FMA_IMAD, ALU_TO_FMA, SHFL_IDX, SHFL_UP, CREDUX_MAX, CREDUX_MIN_MAX2, VOTE_BALLOT_FLO,
          SHFL_XOR_5, NOPS };
static const char *kName[NOPS] = {"VIMNMX3 (alu)", "IMAD (fma)", "VIMNMX3->IMAD (cross-pipe pair)",
                                  "SHFL.IDX", "SHFL.UP", "CREDUX.MAX (__reduce_max_sync)",
                                  "2 independent CREDUX then max", "VOTE.ANY ballot + FLO",
                                  "5 SHFL.BFLY butterfly (sub-warp max)"};
static const int kPerStep[NOPS] = {1, 1, 2, 1, 1, 1, 1, 1, 1};

template <int OP>
__global__ void k_lat(uint32_t seed, uint32_t *sink, unsigned long long *cyc) {
    uint32_t a = seed + threadIdx.x, b = seed * 7u + 1u;
    __syncwarp();
    const unsigned long long t0 = clock64();
#pragma unroll 16
    for (int it = 0; it < N; ++it) {
        if (OP == ALU_VIMNMX3) a = (uint32_t)__vimax3_s32((int)a, (int)b, (int)(b ^ 5u));
        if (OP == FMA_IMAD) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(b));
        if (OP == ALU_TO_FMA) {
            a = (uint32_t)__vimax3_s32((int)a, (int)b, (int)(b ^ 5u));
            asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(b));
        }
        if (OP == SHFL_IDX) a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 1) & 31);
        if (OP == SHFL_UP) a = __shfl_up_sync(0xffffffffu, a, 1);
        if (OP == CREDUX_MAX) a = (uint32_t)__reduce_max_sync(0xffffffffu, (int)a) + threadIdx.x;
        if (OP == CREDUX_MIN_MAX2) {
            const int x = __reduce_max_sync(0xffffffffu, (int)a), y = __reduce_min_sync(0xffffffffu, (int)(a ^ b));
            a = (uint32_t)max(x, y) + threadIdx.x;
        }
        if (OP == VOTE_BALLOT_FLO) a = 31u - __clz(__ballot_sync(0xffffffffu, (a >> (threadIdx.x & 7)) & 1u) | 1u) + a;
        if (OP == SHFL_XOR_5) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a = max(a, __shfl_xor_sync(0xffffffffu, a, o));
        }
    }
    const unsigned long long t1 = clock64();
    if (a == 0x12345678u) sink[0] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int OP>
static double run(uint32_t *sink, unsigned long long *cyc) {
    k_lat<OP><<<1, 32>>>(1u, sink, cyc);
    k_lat<OP><<<1, 32>>>(2u, sink, cyc);
    unsigned long long h = 0;
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    return (double)h / N;
}

int main() {
    uint32_t *sink;
    unsigned long long *cyc;
    cudaMalloc(&sink, 4);
    cudaMalloc(&cyc, 8);
    double r[NOPS];
    r[ALU_VIMNMX3] = run<ALU_VIMNMX3>(sink, cyc);
    r[FMA_IMAD] = run<FMA_IMAD>(sink, cyc);
    r[ALU_TO_FMA] = run<ALU_TO_FMA>(sink, cyc);
    r[SHFL_IDX] = run<SHFL_IDX>(sink, cyc);
    r[SHFL_UP] = run<SHFL_UP>(sink, cyc);
    r[CREDUX_MAX] = run<CREDUX_MAX>(sink, cyc);
    r[CREDUX_MIN_MAX2] = run<CREDUX_MIN_MAX2>(sink, cyc);
    r[VOTE_BALLOT_FLO] = run<VOTE_BALLOT_FLO>(sink, cyc);
    r[SHFL_XOR_5] = run<SHFL_XOR_5>(sink, cyc);
    if (cudaGetLastError() != cudaSuccess) { fprintf(stderr, "CUDA error\n"); return 1; }
    printf("{\"cycles_per_dependent_step\": {");
    for (int o = 0; o < NOPS; ++o) printf("%s\"%s\": %.1f", o ? ", " : "", kName[o], r[o]);
    printf("}, \"instructions_per_step\": {");
    for (int o = 0; o < NOPS; ++o) printf("%s\"%s\": %d", o ? ", " : "", kName[o], kPerStep[o]);
    printf("}}\n");
    return 0;
}
