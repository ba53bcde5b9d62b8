// common.cuh — shared device helpers for the KVComp sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "kvcomp.h"

#define KVC_CUDA_TRY(expr)                                                   \
    do {                                                                     \
        cudaError_t e_ = (expr);                                             \
        if (e_ != cudaSuccess) return kvc_fail_cuda(e_, #expr);              \
    } while (0)

int kvc_fail(int status, const char *msg);
int kvc_fail_cuda(cudaError_t e, const char *what);
int kvc_check_launch(const char *what);

// Block serialisation geometry (codec.py:229-268): "<IH" header, u16 slice
// counts, interleaved f32 (min, scale) per unit, payload, pad to 4 bytes.
__host__ __device__ __forceinline__ int kvc_header_bytes(int bs, int n_units) {
    return 6 + 2 * bs + 8 * n_units;
}

__device__ __forceinline__ float kvc_load(const __half *p) { return __half2float(*p); }
__device__ __forceinline__ float kvc_load(const float *p) { return *p; }
// exact widening loads (the quantiser's f64 arithmetic; f16/f32 -> f64 is exact)
__device__ __forceinline__ double kvc_load_d(const __half *p) { return (double)__half2float(*p); }
__device__ __forceinline__ double kvc_load_d(const float *p) { return (double)*p; }
__device__ __forceinline__ double kvc_load_d(const double *p) { return *p; }

// A sequence descriptor with the live (n_chunks, buffered) pair: when
// `live` is set the growing-cache Store keeps those two counts in device
// memory, so the descriptor itself stays unchanged across decode steps.
__device__ __forceinline__ kvc_seq_desc kvc_load_desc(const kvc_seq_desc *seqs, long i) {
    kvc_seq_desc sd = seqs[i];
    if (sd.live) {
        sd.n_chunks = sd.live[0];
        sd.buffered = sd.live[1];
    }
    return sd;
}

__device__ __forceinline__ void kvc_set_err(int *err, int code) {
    if (err) atomicCAS(err, 0, code);
}

// ---------------------------------------------------------------------------
// Generic MSB-first bit reader over global/shared bytes with an end guard.
// Used by the shape-generic kernels; the fused kernel has its own reader.
// ---------------------------------------------------------------------------
struct KvcBitReader {
    const uint8_t *p;    // next byte to load
    const uint8_t *end;  // first byte that must not be loaded
    uint64_t buf;        // left-aligned bits
    int n;               // valid bits in buf

    __device__ __forceinline__ void init(const uint8_t *base, uint64_t bitpos, const uint8_t *e) {
        p = base + (bitpos >> 3);
        end = e;
        buf = 0;
        n = 0;
        refill();
        int skip = (int)(bitpos & 7);
        buf <<= skip;
        n -= skip;
    }
    __device__ __forceinline__ void refill() {
        while (n <= 56) {
            uint64_t byte = (p < end) ? (uint64_t)(*p) : 0ull;
            ++p;
            buf |= byte << (56 - n);
            n += 8;
        }
    }
    __device__ __forceinline__ uint32_t peek32() const { return (uint32_t)(buf >> 32); }
    __device__ __forceinline__ void consume(int len) {
        buf <<= len;
        n -= len;
        if (n <= 32) refill();
    }
};

// Decode one symbol with the codebook tables (12-bit LUT, canonical tail for
// codes longer than 12 bits).  Returns symbol, sets len (0 = invalid code).
__device__ __forceinline__ int kvc_decode_symbol(const kvc_codebook_dev *cb, uint32_t win,
                                                 int &len) {
    uint32_t e = cb->lut[win >> (32 - KVC_LUT_BITS)];
    len = (int)((e >> 8) & 0xFF);
    if (len) return (int)(e & 0xFF);
    for (int l = KVC_LUT_BITS + 1; l <= cb->max_len; ++l) {
        uint32_t code = win >> (32 - l);
        uint32_t rel = code - cb->first_code[l];
        if (cb->count[l] && code >= cb->first_code[l] && rel < cb->count[l]) {
            len = l;
            return cb->sorted_symbols[cb->first_index[l] + rel];
        }
    }
    len = 0;
    return 0;
}

// Warp / block reductions.
__device__ __forceinline__ float kvc_warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float kvc_warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float kvc_warp_min(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ uint32_t kvc_warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Extent [start, end) of block `ordinal` of an arena (codec.py:328-333).
__device__ __forceinline__ void kvc_extent(const uint32_t *offsets, const kvc_arena_counters *c,
                                           long ordinal, long n_blocks, uint64_t &start,
                                           uint64_t &end) {
    start = offsets[ordinal];
    end = (ordinal + 1 < n_blocks) ? (uint64_t)offsets[ordinal + 1] : c->cursor;
}
