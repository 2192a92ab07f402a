// logan_pack.cu — device pre-pass re-encoding a LOGAN_SEQ_U8 pool of the bytes
// 'A' 'C' 'G' 'T' as a LOGAN_SEQ_2BIT pool (include/logan_xdrop.h,
// logan_pack_2bit), so such pools take the packed first window.
//
// The sweep compares bases by equality only (Alg. 1: a
// match / mismatch score per cell pair); on a pool whose every byte is one of
// the four letters, byte equality and 2-bit code equality are the same
// relation, so the two encodings give identical results. The pass counts the
// bytes outside {A, C, G, T} inside the batch's reads (the caller keeps the u8
// pool if there are any).
//
// HBM-bound: pool_len bytes read, pool_len / 4 written (one thread packs 16
// bytes into one 32-bit word, grid-stride over the pool), then the reads'
// bytes once more (one warp per read, one atomic per warp).
#include <algorithm>
#include <cstdint>

#include <cuda_runtime.h>

#include "logan_xdrop.h"

namespace {

constexpr int PACK_NT = 256;

// 4 bytes of A/C/G/T -> 4 codes in bits 0-1 of each byte: ((c >> 1) ^ (c >> 2)) & 3
// maps 0x41 'A' -> 0, 0x43 'C' -> 1, 0x47 'G' -> 2, 0x54 'T' -> 3 (bits shifted in
// from the next byte land above bit 1 and are masked off)
__device__ __forceinline__ uint32_t codes4(uint32_t w) { return ((w >> 1) ^ (w >> 2)) & 0x03030303u; }

// four 2-bit codes (one per byte) -> one byte, base b at bits 2 (b mod 4)
__device__ __forceinline__ uint32_t pack4(uint32_t c) {
    c |= c >> 6;                                 // byte 0: c0 | c1 << 2, byte 2: c2 | c3 << 2
    return (c & 0xFu) | ((c >> 12) & 0xF0u);
}

__global__ void __launch_bounds__(PACK_NT) k_pack2bit(const uint8_t *__restrict__ u8, int64_t pool_len,
                                                       uint32_t *__restrict__ out, int64_t out_words, bool vec) {
    const int64_t stride = (int64_t)gridDim.x * PACK_NT;
    for (int64_t t = (int64_t)blockIdx.x * PACK_NT + threadIdx.x; t < out_words; t += stride) {
        const int64_t b0 = 16 * t;
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        if (b0 + 16 <= pool_len) {
            if (vec) {
                const uint4 v = __ldg(reinterpret_cast<const uint4 *>(u8 + b0));
                w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u) w[u] = __ldg(reinterpret_cast<const uint32_t *>(u8 + b0) + u);
            }
        } else if (b0 < pool_len) {  // the ragged tail: whole words are readable (header)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t nv = pool_len - (b0 + 4 * u);
                if (nv > 0) {
                    w[u] = __ldg(reinterpret_cast<const uint32_t *>(u8 + b0) + u);
                    if (nv < 4) w[u] &= (1u << (8 * nv)) - 1u;  // code bytes past the end as 'A'
                }
            }
        }
        uint32_t r = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) r |= pack4(codes4(w[u])) << (8 * u);
        // bytes past pool_len (zeroed above, or the padding words) hold code 0
        out[t] = b0 < pool_len ? r : 0u;
    }
}

// Bytes outside {A, C, G, T} inside the reads of the batch: one warp per read
// (query and target of every pair), the pairs k_expand would reject skipped
// (their result is the invalid result in either format). Only the bases inside
// reads are ever compared (positions past a read's end are sentinels), so the
// gaps of the pool (padding, unused bytes) do not matter.
__global__ void __launch_bounds__(PACK_NT) k_count_other(const uint8_t *__restrict__ u8, int64_t pool_len,
                                                          const int64_t *q_off, const int32_t *q_len,
                                                          const int64_t *t_off, const int32_t *t_len,
                                                          int64_t n_pairs, unsigned long long *n_other) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (PACK_NT / 32);
    uint32_t bad = 0;
    for (int64_t r = ((int64_t)blockIdx.x * PACK_NT + threadIdx.x) / 32; r < 2 * n_pairs; r += nwarps) {
        const int64_t p = r >> 1;
        const int64_t qo = q_off[p], ql = q_len[p], to = t_off[p], tl = t_len[p];
        if (qo < 0 || ql < 0 || qo + ql > pool_len || to < 0 || tl < 0 || to + tl > pool_len) continue;
        const int64_t off = (r & 1) ? to : qo, len = (r & 1) ? tl : ql;
        const int64_t end = off + len;
        for (int64_t wd = off / 4 + lane; 4 * wd < end; wd += 32) {
            const uint32_t x = __ldg(reinterpret_cast<const uint32_t *>(u8) + wd);
            const int64_t b = 4 * wd;
            uint32_t m = 0x01010101u;                                   // bytes of the word inside the read
            if (b < off) m &= 0x01010101u << (8 * (off - b));
            if (end - b < 4) m &= (1u << (8 * (end - b))) - 1u;
            const uint32_t ok = __vcmpeq4(x, 0x41414141u) | __vcmpeq4(x, 0x43434343u) |
                                __vcmpeq4(x, 0x47474747u) | __vcmpeq4(x, 0x54545454u);
            bad += __popc(~ok & m);
        }
    }
    bad = __reduce_add_sync(0xffffffffu, bad);
    if (lane == 0 && bad) atomicAdd(n_other, (unsigned long long)bad);
}

}  // namespace

extern "C" {

size_t logan_pack_2bit_bytes(int64_t pool_len) {
    if (pool_len < 0) return 0;
    return (size_t)(((pool_len + 15) / 16) * 4 + 16);
}

int logan_pack_2bit(const uint8_t *u8_pool, int64_t pool_len, const int64_t *q_off, const int32_t *q_len,
                    const int64_t *t_off, const int32_t *t_len, int64_t n_pairs, uint8_t *pool_2bit,
                    size_t pool_2bit_bytes, uint64_t *n_other, void *stream) {
    if (pool_len < 0 || n_pairs < 0 || !n_other || ((uintptr_t)n_other & 7) != 0) return LOGAN_EINVAL;
    if (!pool_2bit || ((uintptr_t)pool_2bit & 3) != 0) return LOGAN_EINVAL;
    if (pool_len > 0 && (!u8_pool || ((uintptr_t)u8_pool & 3) != 0)) return LOGAN_EINVAL;
    if (n_pairs > 0 && (!q_off || !q_len || !t_off || !t_len)) return LOGAN_EINVAL;
    const size_t need = logan_pack_2bit_bytes(pool_len);
    if (pool_2bit_bytes < need) return LOGAN_ENOSPC;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(n_other, 0, sizeof(uint64_t), s) != cudaSuccess) return LOGAN_ECUDA;
    const int64_t words = (int64_t)(need / 4);  // packed words plus 16 bytes of zero padding
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::min<int64_t>((words + PACK_NT - 1) / PACK_NT, (int64_t)sms * 8);
    const bool vec = ((uintptr_t)u8_pool & 15) == 0;
    k_pack2bit<<<grid, PACK_NT, 0, s>>>(u8_pool, pool_len, (uint32_t *)pool_2bit, words, vec);
    if (n_pairs > 0) {
        const int g2 = (int)std::min<int64_t>((2 * n_pairs + PACK_NT / 32 - 1) / (PACK_NT / 32), (int64_t)sms * 8);
        k_count_other<<<g2, PACK_NT, 0, s>>>(u8_pool, pool_len, q_off, q_len, t_off, t_len, n_pairs,
                                             (unsigned long long *)n_other);
    }
    return cudaGetLastError() == cudaSuccess ? LOGAN_OK : LOGAN_ECUDA;
}

}  // extern "C"
