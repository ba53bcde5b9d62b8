// store_fused.cu — the Store: quantise -> Huffman encode -> append.
//
//   append (growing cache, kvcache.py:150-177; codebooks fixed after prefill):
//     store_kernel<true>: quantise + encode + decoupled look-back over block
//     sizes (deterministic block_index order) + write, one launch
//   prefill (kvcache.py:76-145):
//     pass A  store_kernel<false>  quantise + code histogram (K, V); with small
//             alphabets also per-block histograms, and on the hot shape the
//             codes and (min, scale) pairs for pass B
//     host    2x256 histogram -> smoothed canonical codebooks
//     scan    store_offsets_kernel: per-block sizes -> arena offsets
//     pass B  store_kernel<true>   encode (from pass A's codes) + write at the
//             precomputed offsets; without per-block histograms, the append
//             kernel with its look-back
//
// One CTA per (chunk, head) block; blockIdx.y selects K (0) or V (1).  The
// block is staged in shared memory as f32 (16-byte vector loads), per-unit
// min/max and codes are computed there, and the serialised block image
// (codec.py:229-244) is assembled in shared memory as big-endian words:
// a warp per slice, each lane emits its run of codewords at the offset given
// by a warp prefix sum of code lengths.
//
// Quantisation is bit-exact with the reference's binary64 arithmetic
// (quantizer.py:114-141): an f32 candidate t = (x-min)*RN(1/s) is within
// 4.6e-5 of the binary64 quotient (3 roundings, t <= 256), so its code is final
// unless frac(t) lies within 2^-12 of 1/2 (the only decision boundary of
// round-half-up); those values, and any non-finite/huge intermediate, take the
// binary64 path (reciprocal multiply, then __ddiv_rn near the boundary).
#include <cmath>

#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct StoreTensor {
    const void *x;              // [.., H_local, D] rows, row_stride elements apart
    int mode;                   // KVC_K_BLOCK / KVC_V_TOKEN
    double rel;
    const kvc_codebook_dev *cb; // NULL in the histogram pass
    uint8_t *arena;
    uint64_t capacity;
    uint32_t *offsets;
    kvc_arena_counters *counters;
    unsigned long long *status; // look-back words, one per block (zeroed)
    unsigned long long *acc;    // [0] ticket, [1] done, [2] payload bits, [3] payload bytes, [4] max extent
    unsigned long long *hist;   // 256 bins (histogram pass)
    int max_code;               // ceil(1/rel): codes lie in [0, max_code]
    const float *ranges;        // K_CHANNEL: [2][H_local][D] whole-context (min, max)
    // prefill fast path, hot shape: pass A writes each block's codes [64][128] u8
    // and unit (min, scale) f32 pairs here; pass B reads them instead of
    // re-staging and re-quantising the input (same HBM bytes, fewer instructions)
    uint8_t *codes_io;
    float *metas_io;
};

struct StoreParams {
    StoreTensor t[2];
    long row_stride;
    int n_chunks, H_local, H_total, head_base, D, bs;
    uint32_t chunk_base;
    int *err;
    // prefill fast path (null otherwise): pass A also writes per-block code
    // histograms blk_hist [2][nb][32] u16; pass B with nb0 != null takes block b
    // = blockIdx.x and its arena offset from offsets[nb0[t] + b] (written by
    // store_offsets_kernel): no tickets, no look-back, no counter updates.
    uint16_t *blk_hist;
    const unsigned long long *nb0;
};

// out of line: the exact path must not be inlined at every unrolled call site
// (ptxas then keeps the hot loop small: pass B 1.31 -> 1.17 ms on a config-2 slice)
__device__ __noinline__ uint8_t code_f64(float x, float lo, float scale) {
    const double s64 = (double)scale;
    const double d = __dsub_rn((double)x, (double)lo);
    double t = __dmul_rn(d, __drcp_rn(s64));
    double f = floor(t);
    double frac = __dsub_rn(t, f);
    if (fabs(frac - 0.5) < 1.0e-11 * (t + 1.0)) {
        t = __ddiv_rn(d, s64);
        f = floor(t);
        frac = __dsub_rn(t, f);
    }
    if (frac >= 0.5) f += 1.0;
    return (uint8_t)(int)f;
}

__device__ __forceinline__ uint8_t code_fast(float x, float lo, float scale, float r32) {
    if (!(scale > 0.f)) return 0;
    const float t = __fmul_rn(__fsub_rn(x, lo), r32);
    if (t < 300.f) {
        const float c = floorf(t);
        const float f = t - c;
        if (fabsf(f - 0.5f) > (1.0f / 4096.0f)) return (uint8_t)(int)(c + (f >= 0.5f ? 1.f : 0.f));
    }
    return code_f64(x, lo, scale);
}

__device__ __noinline__ float code_clamped_f64(float x, float lo, float scale) {
    const double s64 = (double)scale;
    const double d = __dsub_rn((double)x, (double)lo);
    double tt = __ddiv_rn(d, s64);
    double f = floor(tt);
    if (__dsub_rn(tt, f) >= 0.5) f += 1.0;
    return (float)fmin(fmax(f, -1.0), 1024.0);
}

// K_CHANNEL: fixed whole-context ranges, so t may fall outside [0, max_code];
// round half up then clip (quantizer.py:137-140).
__device__ __forceinline__ uint8_t code_clamped(float x, float lo, float scale, float r32,
                                                int clamp_max) {
    if (!(scale > 0.f)) return 0;
    const float t = __fmul_rn(__fsub_rn(x, lo), r32);
    float code;
    if (fabsf(t) < 300.f && fabsf(t - floorf(t) - 0.5f) > (1.0f / 4096.0f)) {
        const float c = floorf(t);
        code = c + ((t - c) >= 0.5f ? 1.f : 0.f);
    } else {
        code = code_clamped_f64(x, lo, scale);
    }
    code = fminf(fmaxf(code, 0.f), (float)clamp_max);
    return (uint8_t)(int)code;
}

// code_fast with the scale read only on the (rare) exact path
// floor and the integer conversion without the XU pipe: t + 2^23 rounded toward
// -inf holds floor(t) in its low mantissa bits (0 <= t < 2^23)
__device__ __forceinline__ uint32_t code_fast_p(float x, float lo, float r32, const float *scale_p) {
    const float t = __fmul_rn(__fsub_rn(x, lo), r32);
    if (t < 300.f) {
        const float m = __fadd_rd(t, 8388608.0f);
        const float f = t - (m - 8388608.0f);  // both exact
        if (fabsf(f - 0.5f) > (1.0f / 4096.0f))
            return (__float_as_uint(m) & 0x1FFu) + (f >= 0.5f ? 1u : 0u);
    }
    const float sc = *scale_p;
    return sc > 0.f ? code_f64(x, lo, sc) : 0u;
}

// Hot shape (head_dim 128, block 64): thread -> column pair (2j, 2j+1), rows
// q, q+4, ..., mode specialised so the unit parameters are hoisted (K: per
// column, loaded once) or broadcast (V: per row, one warp shares the row).
// Pass B stores the code pair with one 16-bit store; pass A counts them.
// Branch-free fast code; `near` flags values the f32 estimate cannot decide
// (round-half-up boundary within 2^-12, or t out of range), which must take
// code_f64.  The result is only used when !near.
// With lo = unit min and scale = RN(rel*(max-min)), t <= (1/rel)(1 + 2^-22) <= 257
// for rel >= 1/256, so v = RN(t + 1/2) < 512 and round-half-up is floor(v):
// RD(v + 2^23) holds it in the low mantissa bits.  v rounds t + 1/2 only in
// its last bit, which can move floor() only inside the flagged band.
__device__ __forceinline__ uint32_t code_fast_flag(float x, float lo, float r32, bool &near) {
    const float t = __fmul_rn(__fsub_rn(x, lo), r32);
    const float v = __fadd_rn(t, 0.5f);
    const float m = __fadd_rd(v, 8388608.0f);
    const float g = v - (m - 8388607.5f);  // frac(v) - 1/2, exact
    near = fabsf(g) >= 0.5f - (1.0f / 4096.0f);
    return __float_as_uint(m) & 0xFFu;
}

// code_fast_flag for a column pair with packed f32x2 arithmetic (same
// roundings, so the same codes): returns a | b << 8 (the low byte of each
// RD(v + 2^23); byte 2 of that float is zero), `g` = frac(v) - 1/2 per lane.
__device__ __forceinline__ uint32_t code_pair_fast(float2 x, float2 nlo, float2 r, float2 &g) {
    const float2 t = __fmul2_rn(__fadd2_rn(x, nlo), r);
    const float2 v = __fadd2_rn(t, make_float2(0.5f, 0.5f));
    const float2 m = __fadd2_rd(v, make_float2(8388608.0f, 8388608.0f));
    const float2 d = __fadd2_rn(m, make_float2(-8388607.5f, -8388607.5f));  // floor(v) + 1/2, exact
    g = __ffma2_rn(d, make_float2(-1.0f, -1.0f), v);                         // v - d, exact
    return __byte_perm(__float_as_uint(m.x), __float_as_uint(m.y), 0x2240u);
}
constexpr float kNearBand = 0.5f - (1.0f / 4096.0f);

// OUT: pass A writes the codes for pass B (codes_out); SMALL: per-warp 32-bin
// histograms (alphabet < 32) instead of the shared 256-bin one.
template <typename T, bool ENCODE, int MODE, bool OUT, bool SMALL>
__device__ __forceinline__ void quantize_hot(const T *stage, uint8_t *codes, const float *u_lo,
                                             const float *u_sc, const float *u_r, int max_code,
                                             uint32_t *whist, uint32_t *sh_hist, int tid,
                                             uint8_t *codes_out) {
    constexpr int D = 128, BS = 64;
    const int j = tid & 63, q = tid >> 6;  // column pair, row phase (0..3)
    const int c0 = 2 * j;
    float klo0 = 0.f, klo1 = 0.f, kr0 = 0.f, kr1 = 0.f;
    if (MODE != KVC_V_TOKEN) {
        klo0 = u_lo[c0]; klo1 = u_lo[c0 + 1];
        kr0 = u_r[c0]; kr1 = u_r[c0 + 1];
    }
    uint32_t *hist = SMALL ? whist : sh_hist;
    uint16_t *out16 = reinterpret_cast<uint16_t *>((ENCODE ? codes : codes_out) + c0);
#pragma unroll 4
    for (int k = 0; k < BS / 4; ++k) {
        const int r = q + 4 * k;
        float x0, x1;
        if constexpr (sizeof(T) == 2) {
            const __half2 h = *reinterpret_cast<const __half2 *>(stage + r * D + c0);
            const float2 f = __half22float2(h);
            x0 = f.x; x1 = f.y;
        } else {
            const float2 f = *reinterpret_cast<const float2 *>(stage + r * D + c0);
            x0 = f.x; x1 = f.y;
        }
        uint32_t pair;
        if (MODE == KVC_K_CHANNEL) {
            const uint32_t a = code_clamped(x0, klo0, u_sc[c0], kr0, max_code);
            const uint32_t b = code_clamped(x1, klo1, u_sc[c0 + 1], kr1, max_code);
            pair = a | (b << 8);
        } else {
            // branch-free fast codes; near-ties (~0.05 % of fp16 values) are redone
            // exactly behind one warp-uniform branch per pair (taken ~3 % of the time)
            const float lo0 = MODE == KVC_V_TOKEN ? u_lo[r] : klo0;
            const float lo1 = MODE == KVC_V_TOKEN ? lo0 : klo1;
            const float r0 = MODE == KVC_V_TOKEN ? u_r[r] : kr0;
            const float r1 = MODE == KVC_V_TOKEN ? r0 : kr1;
            float2 g;
            pair = code_pair_fast(make_float2(x0, x1), make_float2(-lo0, -lo1), make_float2(r0, r1), g);
            if (__any_sync(0xffffffffu, fmaxf(fabsf(g.x), fabsf(g.y)) >= kNearBand)) {
                const int ua = MODE == KVC_V_TOKEN ? r : c0, ub = MODE == KVC_V_TOKEN ? r : c0 + 1;
                uint32_t a = pair & 0xFFu, b = pair >> 8;
                if (fabsf(g.x) >= kNearBand) a = u_sc[ua] > 0.f ? code_f64(x0, lo0, u_sc[ua]) : 0u;
                if (fabsf(g.y) >= kNearBand) b = u_sc[ub] > 0.f ? code_f64(x1, lo1, u_sc[ub]) : 0u;
                pair = a | (b << 8);
            }
        }
        if (ENCODE || OUT) out16[r * (D / 2)] = (uint16_t)pair;
        if (!ENCODE) {
            atomicAdd(&hist[pair & 0xFFu], 1u);
            atomicAdd(&hist[pair >> 8], 1u);
        }
    }
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void img_or_byte(uint32_t *img, int j, uint32_t v) {
    atomicOr(&img[j >> 2], (v & 0xFFu) << (8 * (3 - (j & 3))));
}
__device__ __forceinline__ void img_or_bits32(uint32_t *img, uint32_t p, uint32_t v) {
    const uint32_t s = p & 31;
    atomicOr(&img[p >> 5], v >> s);
    if (s) atomicOr(&img[(p >> 5) + 1], v << (32 - s));
}

// 16-bit little-endian field at even stream byte offset j of the block image
// (img words are big-endian stream words, byte-swapped at write-out); the word
// shared by the header's end and the payload's start is OR-ed
__device__ __forceinline__ void img_u16(uint32_t *img, int j, uint32_t v, int shared_word) {
    const uint32_t sw = ((v & 0xFFu) << 8) | ((v >> 8) & 0xFFu);
    if ((j >> 2) == shared_word) atomicOr(&img[j >> 2], (j & 2) ? sw : (sw << 16));
    else reinterpret_cast<uint16_t *>(img)[(j >> 1) ^ 1] = (uint16_t)sw;
}

// Shared-memory layout (dynamic): stage f32 [bs*D] (reused as the block image),
// codes u8 [bs*D], unit lo/scale/r32 f32 [n_units], slice bits u32 [bs],
// slice offsets u32 [bs], codebook words u32[256] + lengths u8[256].
// DT / BST: compile-time head_dim / block_size (0 = runtime, generic shapes).
// Hot shape: a register cap (40) for 6 resident CTAs per SM instead of 5 hides
// more of the staging and look-back latency (config-2 slice: pass A 0.386 ->
// 0.382 ms, pass B 0.405 -> 0.400, growing-cache store 0.943 -> 0.871).  A cap
// of 7 (32 registers) was faster still for the look-back store (0.764) but
// slowed pass A and the small append events.  Generic shapes keep the default.
template <typename T, bool ENCODE, int DT, int BST>
__global__ void __launch_bounds__(kThreads, (DT == 128 && BST == 64) ? 6 : 1)
store_kernel(StoreParams P, int stage_words) {
    extern __shared__ __align__(16) uint8_t sm[];
    const StoreTensor S = P.t[blockIdx.y];  // one copy into registers
    const int D = DT ? DT : P.D, bs = BST ? BST : P.bs, nv = bs * D;
    const bool is_v = S.mode == KVC_V_TOKEN;
    const int n_units = is_v ? bs : D;
    T *stage = reinterpret_cast<T *>(sm);  // staged in the input type (fp16 halves smem)
    uint8_t *codes = sm + 4 * (size_t)stage_words;
    const int codes_bytes = nv;
    float *u_lo = reinterpret_cast<float *>(codes + ((codes_bytes + 15) & ~15));
    float *u_sc = u_lo + n_units;
    float *u_r = u_sc + n_units;
    uint32_t *s_bits = reinterpret_cast<uint32_t *>(u_r + n_units);
    uint32_t *s_off = s_bits + bs;
    uint32_t *cw = s_off + bs;
    uint8_t *cl = reinterpret_cast<uint8_t *>(cw + 256);
    __shared__ uint32_t sh_hist[256];
    __shared__ uint32_t sh_whist[kWarps][32];
    __shared__ long sh_b;
    __shared__ unsigned long long sh_excl;
    __shared__ uint32_t sh_total_bits;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long nb = (long)P.n_chunks * P.H_local;

    // logical block id in scheduling order (look-back needs predecessors running)
    const bool prescanned = ENCODE && P.nb0 != nullptr;
    if (tid == 0) sh_b = (ENCODE && !prescanned) ? (long)atomicAdd(&S.acc[0], 1ull) : (long)blockIdx.x;
    if (!ENCODE)
        for (int i = tid; i < 256; i += kThreads) sh_hist[i] = 0;
    // hot encode path (head_dim 128, block 64, codes <= 8 bits): cw holds
    // codeword << 8 | length, one shared load per code
    const bool hot_enc = ENCODE && DT == 128 && BST == 64 && S.cb->max_len <= 8;
    if (ENCODE)
        for (int i = tid; i < 256; i += kThreads) {
            const uint32_t w = S.cb->words[i], l = S.cb->lengths[i];
            // hot: codeword left-aligned, length in the low bits (l <= 8, so the
            // two fields never overlap): one funnel shift appends a code
            cw[i] = hot_enc ? (l ? ((w << (32 - l)) | l) : 0u) : w;
            cl[i] = (uint8_t)l;
        }
    __syncthreads();
    const long b = sh_b;
    const int chunk = (int)(b / P.H_local), hl = (int)(b % P.H_local);
    const uint64_t base = ENCODE ? S.counters->cursor : 0;
    const T *src = static_cast<const T *>(S.x) + (long)chunk * bs * P.row_stride + (long)hl * D;

    const bool small_alpha = S.max_code < 32;
    const bool from_codes = ENCODE && S.codes_io != nullptr;  // prescanned, hot shape
    if (from_codes) {
        const uint4 *cs = reinterpret_cast<const uint4 *>(S.codes_io + (size_t)b * 8192);
        for (int i = tid; i < 8192 / 16; i += kThreads) reinterpret_cast<uint4 *>(codes)[i] = cs[i];
        for (int i = tid; i < n_units; i += kThreads) {
            const float2 m = reinterpret_cast<const float2 *>(S.metas_io)[(size_t)b * n_units + i];
            u_lo[i] = m.x;
            u_sc[i] = m.y;
        }
        __syncthreads();
    } else {
    // ---- stage [bs, D] as f32 ------------------------------------------
    constexpr int VEC = 16 / sizeof(T);
    if (D % VEC == 0 && (P.row_stride % VEC) == 0 &&
        (reinterpret_cast<uintptr_t>(S.x) & 15) == 0) {
        const int vpr = D / VEC;
        for (int i = tid; i < bs * vpr; i += kThreads) {
            const int r = i / vpr, v = i % vpr;
            const uint4 u = *reinterpret_cast<const uint4 *>(src + (long)r * P.row_stride + v * VEC);
            *reinterpret_cast<uint4 *>(stage + r * D + v * VEC) = u;
        }
    } else {
        for (int i = tid; i < nv; i += kThreads) {
            const int r = i / D, c = i % D;
            stage[i] = src[(long)r * P.row_stride + c];
        }
    }
    __syncthreads();

    // ---- per-unit (min, scale): K per channel column, V per token row ----
    const bool is_kc = S.mode == KVC_K_CHANNEL;
    if (is_kc) {
        for (int c = tid; c < D; c += kThreads) {
            const float lo = S.ranges[(long)hl * D + c];
            const float hi = S.ranges[((long)P.H_local + hl) * D + c];
            const float sc = (float)__dmul_rn(S.rel, __dsub_rn((double)hi, (double)lo));
            u_lo[c] = lo;
            u_sc[c] = sc;
            u_r[c] = sc > 0.f ? __frcp_rn(sc) : 0.f;
        }
    } else if (DT == 128 && BST == 64 && !is_v) {
        // thread -> column pair (2j, 2j+1) over rows 16q..16q+15; quarters
        // combined through shared memory (the codes area, unused until later)
        const int j = tid & 63, q = tid >> 6;
        float lo0, lo1, hi0, hi1;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int r = 16 * q + i;
            float x0, x1;
            if constexpr (sizeof(T) == 2) {
                const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(stage + r * 128 + 2 * j));
                x0 = f.x; x1 = f.y;
            } else {
                const float2 f = *reinterpret_cast<const float2 *>(stage + r * 128 + 2 * j);
                x0 = f.x; x1 = f.y;
            }
            if (i == 0) {
                lo0 = hi0 = x0;
                lo1 = hi1 = x1;
            } else {
                lo0 = fminf(lo0, x0); hi0 = fmaxf(hi0, x0);
                lo1 = fminf(lo1, x1); hi1 = fmaxf(hi1, x1);
            }
        }
        float4 *part = reinterpret_cast<float4 *>(codes);  // [4][64] (lo0, lo1, hi0, hi1)
        part[q * 64 + j] = make_float4(lo0, lo1, hi0, hi1);
        __syncthreads();
        if (tid < 128) {
            const int jj = tid >> 1, odd = tid & 1;
            float lo = 3.4e38f, hi = -3.4e38f;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                const float4 v = part[qq * 64 + jj];
                lo = fminf(lo, odd ? v.y : v.x);
                hi = fmaxf(hi, odd ? v.w : v.z);
            }
            const float sc = (float)__dmul_rn(S.rel, __dsub_rn((double)hi, (double)lo));
            u_lo[tid] = lo;
            u_sc[tid] = sc;
            u_r[tid] = sc > 0.f ? __frcp_rn(sc) : 0.f;
        }
    } else if (DT == 128 && BST == 64 && kWarps == 8) {
        // V: warp w owns rows w, w+8, .., w+56; lane -> 4 consecutive values of
        // each.  The 8 rows' (min, max) are reduced together by a halving
        // reduce-scatter over the 16 values per lane (16 shuffles for 8 rows
        // instead of 10 per row); lane pair (2i, 2i+1) ends with slot i =
        // (row w + 8*(i>>1), min if i even else max) and computes its scale.
        float v16[16];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int r = warp + 8 * k;
            float v[4];
            if constexpr (sizeof(T) == 2) {
                const uint2 u = *reinterpret_cast<const uint2 *>(stage + r * 128 + 4 * lane);
                const float2 a = __half22float2(*reinterpret_cast<const __half2 *>(&u.x));
                const float2 b2 = __half22float2(*reinterpret_cast<const __half2 *>(&u.y));
                v[0] = a.x; v[1] = a.y; v[2] = b2.x; v[3] = b2.y;
            } else {
                const float4 u = *reinterpret_cast<const float4 *>(stage + r * 128 + 4 * lane);
                v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
            }
            v16[2 * k] = fminf(fminf(v[0], v[1]), fminf(v[2], v[3]));
            v16[2 * k + 1] = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
        }
        // slot s in [0,16): even = min, odd = max of row s >> 1.  Steps xor 16,
        // 8, 4 keep the half of the live slots selected by that lane bit and
        // combine the partner's copy (halves have even length, so slot parity =
        // index parity); then each lane holds (min, max) of row
        // k = 4*bit4 + 2*bit3 + bit2 over 8 lanes, and xor 2, 1 finish it.
#pragma unroll
        for (int o = 16, n = 8; o >= 4; o >>= 1, n >>= 1) {
            const bool hi = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (i < n) {
                    const float keep = hi ? v16[n + i] : v16[i], send = hi ? v16[i] : v16[n + i];
                    const float other = __shfl_xor_sync(0xffffffffu, send, o);
                    v16[i] = (i & 1) ? fmaxf(keep, other) : fminf(keep, other);
                }
            }
        }
        float lo = v16[0], hi = v16[1];
#pragma unroll
        for (int o = 2; o >= 1; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if ((lane & 3) == 0) {
            const int r = warp + 8 * (4 * ((lane >> 4) & 1) + 2 * ((lane >> 3) & 1) + ((lane >> 2) & 1));
            const float sc = (float)__dmul_rn(S.rel, __dsub_rn((double)hi, (double)lo));
            u_lo[r] = lo;
            u_sc[r] = sc;
            u_r[r] = sc > 0.f ? __frcp_rn(sc) : 0.f;
        }
    } else if (DT == 128 && BST == 64) {
        // V: warp per row, lane -> 4 consecutive values (one vector load)
#pragma unroll 2
        for (int r = warp; r < 64; r += kWarps) {
            float v[4];
            if constexpr (sizeof(T) == 2) {
                const uint2 u = *reinterpret_cast<const uint2 *>(stage + r * 128 + 4 * lane);
                const float2 a = __half22float2(*reinterpret_cast<const __half2 *>(&u.x));
                const float2 b = __half22float2(*reinterpret_cast<const __half2 *>(&u.y));
                v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
            } else {
                const float4 u = *reinterpret_cast<const float4 *>(stage + r * 128 + 4 * lane);
                v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
            }
            float lo = fminf(fminf(v[0], v[1]), fminf(v[2], v[3]));
            float hi = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
            lo = kvc_warp_min(lo);
            hi = kvc_warp_max(hi);
            if (lane == 0) {
                const float sc = (float)__dmul_rn(S.rel, __dsub_rn((double)hi, (double)lo));
                u_lo[r] = lo;
                u_sc[r] = sc;
                u_r[r] = sc > 0.f ? __frcp_rn(sc) : 0.f;
            }
        }
    } else if (!is_v) {
        for (int c = tid; c < D; c += kThreads) {
            float lo = kvc_load(&stage[c]), hi = lo;
            for (int r = 1; r < bs; ++r) {
                const float v = kvc_load(&stage[r * D + c]);
                lo = fminf(lo, v);
                hi = fmaxf(hi, v);
            }
            const float sc = (float)__dmul_rn(S.rel, __dsub_rn((double)hi, (double)lo));
            u_lo[c] = lo;
            u_sc[c] = sc;
            u_r[c] = sc > 0.f ? __frcp_rn(sc) : 0.f;
        }
    } else {
        for (int r = warp; r < bs; r += kWarps) {
            float lo = 3.4e38f, hi = -3.4e38f;
            for (int c = lane; c < D; c += 32) {
                const float v = kvc_load(&stage[r * D + c]);
                lo = fminf(lo, v);
                hi = fmaxf(hi, v);
            }
            lo = kvc_warp_min(lo);
            hi = kvc_warp_max(hi);
            if (lane == 0) {
                const float sc = (float)__dmul_rn(S.rel, __dsub_rn((double)hi, (double)lo));
                u_lo[r] = lo;
                u_sc[r] = sc;
                u_r[r] = sc > 0.f ? __frcp_rn(sc) : 0.f;
            }
        }
    }
    __syncthreads();

    // pass A, hot shape, prefill fast path: this block's codes and metas go out
    uint8_t *cout = (!ENCODE && S.codes_io) ? S.codes_io + (size_t)b * 8192 : nullptr;
    if (!ENCODE && S.metas_io && tid < n_units) {
        S.metas_io[((size_t)b * n_units + tid) * 2] = u_lo[tid];
        S.metas_io[((size_t)b * n_units + tid) * 2 + 1] = u_sc[tid];
    }

    // ---- codes (+ histogram in pass A) --------------------------------
    // Pass A: per-warp 32-bin shared histograms (small alphabets) keep atomic
    // contention inside a warp; wider alphabets use the shared 256-bin one.
    uint32_t *whist = sh_whist[warp];
    if (!ENCODE) {
        whist[lane] = 0;
        __syncwarp();
    }
    auto count = [&](bool ok, uint32_t code) {
        if (!ok) return;
        if (small_alpha) atomicAdd(&whist[code], 1u);
        else atomicAdd(&sh_hist[code], 1u);
    };
    if constexpr (DT == 128 && BST == 64) {
        // (out, small) specialised so the loop carries no per-pair branches
#define KVC_QH(M)                                                                               \
    do {                                                                                        \
        if (ENCODE)                                                                             \
            quantize_hot<T, ENCODE, M, false, false>(stage, codes, u_lo, u_sc, u_r, S.max_code, \
                                                     whist, sh_hist, tid, cout);                \
        else if (cout && small_alpha)                                                           \
            quantize_hot<T, ENCODE, M, true, true>(stage, codes, u_lo, u_sc, u_r, S.max_code,   \
                                                   whist, sh_hist, tid, cout);                  \
        else if (cout)                                                                          \
            quantize_hot<T, ENCODE, M, true, false>(stage, codes, u_lo, u_sc, u_r, S.max_code,  \
                                                    whist, sh_hist, tid, cout);                 \
        else if (small_alpha)                                                                   \
            quantize_hot<T, ENCODE, M, false, true>(stage, codes, u_lo, u_sc, u_r, S.max_code,  \
                                                    whist, sh_hist, tid, cout);                 \
        else                                                                                    \
            quantize_hot<T, ENCODE, M, false, false>(stage, codes, u_lo, u_sc, u_r, S.max_code, \
                                                     whist, sh_hist, tid, cout);                \
    } while (0)
        if (is_kc) KVC_QH(KVC_K_CHANNEL);
        else if (is_v) KVC_QH(KVC_V_TOKEN);
        else KVC_QH(KVC_K_BLOCK);
#undef KVC_QH
    } else if (D <= kThreads) {
        // thread -> fixed column c (one division per thread, none per element)
        const int rstep = kThreads / D;
        const int c = tid % D, r0 = tid / D;
        const bool col_ok = r0 < rstep;
        const int iters = (bs + rstep - 1) / rstep;
        for (int k = 0; k < iters; ++k) {
            const int r = r0 + k * rstep;
            const bool ok = col_ok && r < bs;
            uint32_t code = 0;
            if (ok) {
                const int u = is_v ? r : c;
                const int i = r * D + c;
                code = is_kc ? code_clamped(kvc_load(&stage[i]), u_lo[u], u_sc[u], u_r[u], S.max_code)
                             : code_fast(kvc_load(&stage[i]), u_lo[u], u_sc[u], u_r[u]);
                if (ENCODE) codes[i] = (uint8_t)code;
            }
            if (!ENCODE) count(ok, code);
        }
    } else {
        for (int i = tid; i < nv; i += kThreads) {
            const int r = i / D, c = i - r * D;
            const int u = is_v ? r : c;
            const uint32_t code =
                is_kc ? code_clamped(kvc_load(&stage[i]), u_lo[u], u_sc[u], u_r[u], S.max_code)
                      : code_fast(kvc_load(&stage[i]), u_lo[u], u_sc[u], u_r[u]);
            if (ENCODE) codes[i] = (uint8_t)code;
            else count(true, code);
        }
    }
    __syncthreads();
    }  // !from_codes
    if (!ENCODE) {
        if (small_alpha) {
            if (tid < 32) {
                uint32_t v = 0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) v += sh_whist[w][tid];
                if (v) atomicAdd(&S.hist[tid], (unsigned long long)v);
                if (P.blk_hist) P.blk_hist[((size_t)blockIdx.y * nb + b) * 32 + tid] = (uint16_t)v;
            }
        } else {
            for (int i = tid; i < 256; i += kThreads)
                if (sh_hist[i]) atomicAdd(&S.hist[i], (unsigned long long)sh_hist[i]);
        }
        return;
    }

    bool bad = false;
    uint32_t total_bits, pbytes, size;
    const int hdr = kvc_header_bytes(bs, n_units);
    const uint32_t block_index = (P.chunk_base + (uint32_t)chunk) * (uint32_t)P.H_total +
                                 (uint32_t)(P.head_base + hl);
    uint32_t *img = reinterpret_cast<uint32_t *>(sm);
    if (hot_enc) {
        // hot shape, codes <= 8 bits: warp w owns rows w, w+8, ..; lane l the 4
        // codes 4l..4l+3 of a row (one 32-bit load), their codewords packed into
        // one <= 32-bit run kept in registers between the counts and the emission
        constexpr int RW = 64 / kWarps;
        static_assert(RW % 2 == 0, "rows are scanned in pairs");
        uint32_t run[RW], ex[RW], nn[RW];
#pragma unroll
        for (int i = 0; i < RW; ++i) {
            const int r = warp + kWarps * i;
            const uint32_t w4 = *reinterpret_cast<const uint32_t *>(codes + r * 128 + 4 * lane);
            uint32_t rn = 0, nsum = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                // entry = codeword << (32 - l) | l (0 = symbol absent)
                const uint32_t e = cw[__byte_perm(w4, 0u, 0x4440u | k)];
                bad |= (e == 0);
                rn = __funnelshift_l(e, rn, e);  // (rn << l) | codeword
                nsum += e;                       // low 6 bits: sum of the 4 lengths
            }
            run[i] = rn;
            nn[i] = nsum & 63u;
        }
        // two rows per scan: a row's lane-run totals are <= 1024 bits, so the
        // 16-bit halves never carry into each other
#pragma unroll
        for (int i = 0; i < RW; i += 2) {
            const uint32_t inc2 = kvc_warp_incl_scan(nn[i] | (nn[i + 1] << 16), lane);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t n = nn[i + h], inc = h ? (inc2 >> 16) : (inc2 & 0xFFFFu);
                ex[i + h] = (inc - n) | (n << 24);
                if (lane == 31) {
                    s_bits[warp + kWarps * (i + h)] = inc;
                    bad |= inc > 0xFFFFu;
                }
            }
        }
        if (bad) kvc_set_err(P.err, KVC_ERR_CODEC);
        __syncthreads();
        if (warp == 0) {
            const uint32_t v0 = s_bits[lane], v1 = s_bits[lane + 32];
            const uint32_t i0 = kvc_warp_incl_scan(v0, lane);
            const uint32_t t0 = __shfl_sync(0xffffffffu, i0, 31);
            const uint32_t i1 = kvc_warp_incl_scan(v1, lane);
            s_off[lane] = i0 - v0;
            s_off[lane + 32] = t0 + i1 - v1;
            if (lane == 31) sh_total_bits = t0 + i1;
        }
        __syncthreads();
        total_bits = sh_total_bits;
        pbytes = (total_bits + 7) / 8;
        size = (hdr + pbytes + 3) & ~3u;
        for (int i = tid; i < (int)(size >> 4) + 1; i += kThreads)
            reinterpret_cast<uint4 *>(img)[i] = make_uint4(0u, 0u, 0u, 0u);
        __syncthreads();
        // header: 16-bit little-endian fields at even offsets (plain stores; the
        // word shared with the payload start takes an OR)
        const int shw = (hdr & 3) ? (hdr >> 2) : -1;
        if (tid == 0) img_u16(img, 0, block_index & 0xFFFFu, shw);
        if (tid == 1) img_u16(img, 2, block_index >> 16, shw);
        if (tid == 2) img_u16(img, 4, 64u, shw);
        if (tid < 64) img_u16(img, 6 + 2 * tid, s_bits[tid], shw);
        if (tid < n_units) {
            const int j0 = 6 + 2 * 64 + 8 * tid;
            const uint32_t lo = __float_as_uint(u_lo[tid]), sc = __float_as_uint(u_sc[tid]);
            img_u16(img, j0, lo & 0xFFFFu, shw);
            img_u16(img, j0 + 2, lo >> 16, shw);
            img_u16(img, j0 + 4, sc & 0xFFFFu, shw);
            img_u16(img, j0 + 6, sc >> 16, shw);
        }
#pragma unroll
        for (int i = 0; i < RW; ++i) {
            const uint32_t n = ex[i] >> 24;
            if (!n) continue;
            const int r = warp + kWarps * i;
            const uint32_t p = (uint32_t)hdr * 8 + s_off[r] + (ex[i] & 0xFFFFFFu);
            const uint32_t left = run[i] << (32 - n), sft = p & 31;
            atomicOr(&img[p >> 5], left >> sft);
            if (sft + n > 32) atomicOr(&img[(p >> 5) + 1], left << (32 - sft));
        }
    } else {
        // ---- slice bit counts: warp per slice, lane per run of codes --------
        const int cpl = (D + 31) / 32;
        for (int r = warp; r < bs; r += kWarps) {
            uint32_t bits = 0;
            for (int k = 0; k < cpl; ++k) {
                const int c = lane * cpl + k;
                if (c < D) {
                    const uint32_t l = cl[codes[r * D + c]];
                    bad |= (l == 0);
                    bits += l;
                }
            }
            bits = kvc_warp_incl_scan(bits, lane);
            if (lane == 31) {
                s_bits[r] = bits;
                bad |= bits > 0xFFFFu;
            }
        }
        if (bad) kvc_set_err(P.err, KVC_ERR_CODEC);
        __syncthreads();
        if (warp == 0) {
            uint32_t carry = 0;
            for (int r0 = 0; r0 < bs; r0 += 32) {
                const int r = r0 + lane;
                const uint32_t v = r < bs ? s_bits[r] : 0;
                const uint32_t inc = kvc_warp_incl_scan(v, lane);
                if (r < bs) s_off[r] = carry + inc - v;
                carry += __shfl_sync(0xffffffffu, inc, 31);
            }
            if (lane == 0) sh_total_bits = carry;
        }
        __syncthreads();
        total_bits = sh_total_bits;
        pbytes = (total_bits + 7) / 8;
        size = (hdr + pbytes + 3) & ~3u;

        // ---- block image in shared memory (reuses the staging area) --------
        for (int i = tid; i < (int)(size >> 2); i += kThreads) img[i] = 0;
        __syncthreads();
        if (tid < 4) img_or_byte(img, tid, block_index >> (8 * tid));
        if (tid < 2) img_or_byte(img, 4 + tid, (uint32_t)bs >> (8 * tid));
        for (int r = tid; r < bs; r += kThreads) {
            img_or_byte(img, 6 + 2 * r, s_bits[r]);
            img_or_byte(img, 7 + 2 * r, s_bits[r] >> 8);
        }
        for (int i = tid; i < 2 * n_units; i += kThreads) {
            const uint32_t w = __float_as_uint((i & 1) ? u_sc[i >> 1] : u_lo[i >> 1]);
            const int j0 = 6 + 2 * bs + 4 * i;
    #pragma unroll
            for (int k = 0; k < 4; ++k) img_or_byte(img, j0 + k, w >> (8 * k));
        }
        for (int r = warp; r < bs; r += kWarps) {
            // lane's run of codes starts at the warp-exclusive prefix of lengths
            uint32_t lbits = 0;
            for (int k = 0; k < cpl; ++k) {
                const int c = lane * cpl + k;
                if (c < D) lbits += cl[codes[r * D + c]];
            }
            const uint32_t incl = kvc_warp_incl_scan(lbits, lane);
            uint32_t p = (uint32_t)hdr * 8 + s_off[r] + incl - lbits;
            uint64_t accb = 0;
            int nacc = 0;
            for (int k = 0; k < cpl; ++k) {
                const int c = lane * cpl + k;
                if (c >= D) break;
                const uint32_t s = codes[r * D + c];
                const int l = cl[s];
                accb |= (uint64_t)cw[s] << (64 - nacc - l);
                nacc += l;
                if (nacc >= 32) {
                    img_or_bits32(img, p, (uint32_t)(accb >> 32));
                    p += 32;
                    accb <<= 32;
                    nacc -= 32;
                }
            }
            if (nacc) img_or_bits32(img, p, (uint32_t)(accb >> 32));
        }
    }

    if (prescanned) {
        if (bad) atomicCAS(&S.counters->err, 0, (int)KVC_ERR_CODEC);
        __syncthreads();
        const uint64_t off = S.offsets[P.nb0[blockIdx.y] + b];
        if (off + size <= S.capacity && off + size <= 0xFFFFFFFFull) {
            uint32_t *dst = reinterpret_cast<uint32_t *>(S.arena + off);
            for (int i = tid; i < (int)(size >> 2); i += kThreads) dst[i] = __byte_perm(img[i], 0, 0x0123);
        }
        return;
    }

    // ---- decoupled look-back over block sizes (block_index order) ------
    // warp 0 inspects 32 predecessors per step: waits until all have
    // published, adds aggregates back to the nearest inclusive prefix.
    if (warp == 0) {
        const unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kMask = (1ull << 62) - 1;
        if (lane == 0) {
            if (b == 0) st_release(&S.status[0], kInc | size);
            else st_release(&S.status[b], kAgg | size);
        }
        unsigned long long excl = 0;
        long hi = b - 1;  // window [hi-31, hi]
        while (hi >= 0) {
            const long q = hi - lane;
            unsigned long long w = 0;
            if (q >= 0) {
                do { w = ld_acquire(&S.status[q]); } while ((w >> 62) == 0);
            } else {
                w = kInc;  // before block 0: inclusive 0
            }
            const uint32_t inc_mask = __ballot_sync(0xffffffffu, (w >> 62) == 2);
            const int first_inc = inc_mask ? __ffs(inc_mask) - 1 : 32;  // nearest inclusive
            unsigned long long part = (lane <= first_inc) ? (w & kMask) : 0ull;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            excl += part;
            if (inc_mask) break;
            hi -= 32;
        }
        if (lane == 0) {
            if (b != 0) st_release(&S.status[b], kInc | (excl + size));
            sh_excl = excl;
        }
    }
    __syncthreads();

    // ---- coalesced write-out at cursor + exclusive offset --------------
    const uint64_t off = base + sh_excl;
    const bool fits = off + size <= S.capacity && off + size <= 0xFFFFFFFFull;
    if (fits) {
        uint32_t *dst = reinterpret_cast<uint32_t *>(S.arena + off);
        for (int i = tid; i < (int)(size >> 2); i += kThreads) dst[i] = __byte_perm(img[i], 0, 0x0123);
    }
    if (tid == 0) {
        S.offsets[S.counters->n_blocks + b] = (uint32_t)off;
        atomicAdd(&S.acc[2], (unsigned long long)total_bits);
        atomicAdd(&S.acc[3], (unsigned long long)pbytes);
        atomicMax(&S.acc[4], (unsigned long long)size);
        __threadfence();
        if (atomicAdd(&S.acc[1], 1ull) == (unsigned long long)(nb - 1)) {
            __threadfence();
            const unsigned long long total = atomicAdd(&S.status[nb - 1], 0ull) & ((1ull << 62) - 1);
            kvc_arena_counters *ct = S.counters;
            if (*P.err) {
                if (!ct->err) ct->err = *P.err;
            } else if (ct->cursor + total > S.capacity || ct->cursor + total > 0xFFFFFFFFull) {
                if (!ct->err) ct->err = KVC_ERR_ARENA_FULL;
            } else {
                ct->cursor += total;
                ct->n_blocks += (uint64_t)nb;
                ct->payload_bits += atomicAdd(&S.acc[2], 0ull);
                ct->payload_bytes += atomicAdd(&S.acc[3], 0ull);
                const uint32_t mx = (uint32_t)atomicAdd(&S.acc[4], 0ull);
                if (mx > ct->max_extent) ct->max_extent = mx;
            }
        }
    }
}

size_t smem_bytes(int bs, int D, int max_len, int elem = 4) {
    const int nv0 = bs * D;
    const int nv = nv0;
    const int n_units = bs > D ? bs : D;
    const size_t img = (size_t)kvc_header_bytes(bs, n_units) + ((size_t)nv * max_len + 7) / 8 + 16;
    size_t stage = (size_t)elem * nv;
    stage = (stage + 15) & ~size_t(15);
    if (img > stage) stage = (img + 15) & ~size_t(15);
    return stage + ((nv + 15) & ~15) + 12 * (size_t)n_units + 8 * (size_t)bs + 256 * 5 + 64;
}

inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

extern "C" int kvc_store_supported(int bs, int D, int max_len) {
    return bs >= 1 && D >= 1 && bs <= 1024 && D <= 2048 && smem_bytes(bs, D, max_len) <= 200 * 1024;
}

extern "C" size_t kvc_store_workspace_bytes(int n_chunks, int H, int D, int bs) {
    (void)D;
    (void)bs;
    const size_t nb = (size_t)(n_chunks > 0 ? n_chunks : 1) * H;
    return 2 * (a256(8 * nb) + 256) + 256;
}

static int launch_store(const StoreParams &P, int x_dtype, bool encode, int max_len,
                        cudaStream_t s) {
    // quantizer.py:60-66: rel_quant_scale in [1/255, 1] (codes fit u8; the fast
    // quantiser relies on t <= 1/rel < 256)
    for (int t = 0; t < 2; ++t)
        if (!(P.t[t].rel >= 1.0 / 255.0 - 1e-15 && P.t[t].rel <= 1.0))
            return kvc_fail(KVC_ERR_CONFIG, "rel_quant_scale outside [1/255, 1]");
    const int nb = P.n_chunks * P.H_local;
    const int nv = P.bs * P.D;
    size_t sm = smem_bytes(P.bs, P.D, encode ? max_len : 1, x_dtype == KVC_F16 ? 2 : 4);
    const int cb = nv;
    int stage_words = (int)((sm - ((cb + 15) & ~15) - 12 * (size_t)(P.bs > P.D ? P.bs : P.D) -
                             8 * (size_t)P.bs - 256 * 5 - 64) / 4);
    if (sm > 200 * 1024) return kvc_fail(KVC_ERR_CONFIG, "block too large for the fused store");
    dim3 grid(nb, 2);
#define KVC_STORE_LAUNCH2(T, E, DT, BST)                                                       \
    do {                                                                                       \
        KVC_CUDA_TRY(cudaFuncSetAttribute(store_kernel<T, E, DT, BST>,                         \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                                          200 * 1024));                                        \
        store_kernel<T, E, DT, BST><<<grid, kThreads, sm, s>>>(P, stage_words);                \
    } while (0)
#define KVC_STORE_LAUNCH(T, E)                                                                 \
    do {                                                                                       \
        if (P.D == 128 && P.bs == 64) KVC_STORE_LAUNCH2(T, E, 128, 64);                        \
        else KVC_STORE_LAUNCH2(T, E, 0, 0);                                                    \
    } while (0)
    if (x_dtype == KVC_F16) {
        if (encode) KVC_STORE_LAUNCH(__half, true);
        else KVC_STORE_LAUNCH(__half, false);
    } else if (x_dtype == KVC_F32) {
        if (encode) KVC_STORE_LAUNCH(float, true);
        else KVC_STORE_LAUNCH(float, false);
    } else {
        return kvc_fail(KVC_ERR_TENSOR, "unsupported dtype");
    }
#undef KVC_STORE_LAUNCH
#undef KVC_STORE_LAUNCH2
    return kvc_check_launch("store_kernel");
}

// Pass A of prefill: quantise K and V, accumulate their 256-bin histograms
// (hist_dev: 512 x u64, K then V; codebook.py:75-80 over all heads).
extern "C" int kvc_store_hist(const void *k_dev, const void *v_dev, int x_dtype, long row_stride,
                              int n_chunks, int H, int D, int bs, int k_mode, double rel_k,
                              double rel_v, const float *k_ranges_dev, uint64_t *hist_dev,
                              void *stream) {
    if (k_mode != KVC_K_BLOCK && k_mode != KVC_K_CHANNEL) return kvc_fail(KVC_ERR_CONFIG, "bad K mode");
    if (k_mode == KVC_K_CHANNEL && !k_ranges_dev)
        return kvc_fail(KVC_ERR_CONFIG, "K_CHANNEL quantization requires whole-context channel_ranges");
    if (n_chunks == 0) return KVC_OK;
    if (!kvc_store_supported(bs, D, 1)) return kvc_fail(KVC_ERR_CONFIG, "shape not supported");
    StoreParams P{};
    P.t[0].x = k_dev;
    P.t[0].mode = k_mode;
    P.t[0].ranges = k_ranges_dev;
    P.t[0].rel = rel_k;
    P.t[0].hist = reinterpret_cast<unsigned long long *>(hist_dev);
    P.t[0].max_code = (int)ceil(1.0 / rel_k);
    P.t[1].max_code = (int)ceil(1.0 / rel_v);
    P.t[1].x = v_dev;
    P.t[1].mode = KVC_V_TOKEN;
    P.t[1].rel = rel_v;
    P.t[1].hist = reinterpret_cast<unsigned long long *>(hist_dev) + 256;
    P.row_stride = row_stride;
    P.n_chunks = n_chunks;
    P.H_local = H;
    P.H_total = H;
    P.D = D;
    P.bs = bs;
    return launch_store(P, x_dtype, false, 1, static_cast<cudaStream_t>(stream));
}

// Pass B (prefill) / append event: quantise + encode + append K and V blocks
// (kvcache.py:217-239) in one launch.
extern "C" int kvc_store_append(const void *k_dev, const void *v_dev, int x_dtype, long row_stride,
                                int n_chunks, int H_local, int H_total, int head_base, int D,
                                int bs, int k_mode, double rel_k, double rel_v,
                                const float *k_ranges_dev, uint32_t chunk_base,
                                const kvc_codebook_dev *k_cb_dev, int k_max_len,
                                const kvc_codebook_dev *v_cb_dev, int v_max_len,
                                uint8_t *k_arena_dev, uint64_t k_capacity, uint32_t *k_offsets_dev,
                                kvc_arena_counters *k_counters_dev, uint8_t *v_arena_dev,
                                uint64_t v_capacity, uint32_t *v_offsets_dev,
                                kvc_arena_counters *v_counters_dev, void *workspace_dev,
                                size_t workspace_bytes, void *stream) {
    if (n_chunks == 0) return KVC_OK;
    if (k_mode != KVC_K_BLOCK && k_mode != KVC_K_CHANNEL) return kvc_fail(KVC_ERR_CONFIG, "bad K mode");
    if (k_mode == KVC_K_CHANNEL && !k_ranges_dev)
        return kvc_fail(KVC_ERR_CONFIG, "K_CHANNEL quantization requires whole-context channel_ranges");
    const int max_len = k_max_len > v_max_len ? k_max_len : v_max_len;
    if (!kvc_store_supported(bs, D, max_len)) return kvc_fail(KVC_ERR_CONFIG, "shape not supported");
    if (workspace_bytes < kvc_store_workspace_bytes(n_chunks, H_local, D, bs))
        return kvc_fail(KVC_ERR_CONFIG, "store workspace too small");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t nb = (size_t)n_chunks * H_local;
    char *w = static_cast<char *>(workspace_dev);
    const size_t per = a256(8 * nb) + 256;
    KVC_CUDA_TRY(cudaMemsetAsync(w, 0, 2 * per + 256, s));
    StoreParams P{};
    for (int t = 0; t < 2; ++t) {
        StoreTensor &T = P.t[t];
        T.x = t ? v_dev : k_dev;
        T.mode = t ? KVC_V_TOKEN : k_mode;
        T.rel = t ? rel_v : rel_k;
        T.max_code = (int)ceil(1.0 / T.rel);
        T.ranges = t ? nullptr : k_ranges_dev;
        T.cb = t ? v_cb_dev : k_cb_dev;
        T.arena = t ? v_arena_dev : k_arena_dev;
        T.capacity = t ? v_capacity : k_capacity;
        T.offsets = t ? v_offsets_dev : k_offsets_dev;
        T.counters = t ? v_counters_dev : k_counters_dev;
        T.status = reinterpret_cast<unsigned long long *>(w + t * per);
        T.acc = reinterpret_cast<unsigned long long *>(w + t * per + a256(8 * nb));
    }
    P.row_stride = row_stride;
    P.n_chunks = n_chunks;
    P.H_local = H_local;
    P.H_total = H_total;
    P.head_base = head_base;
    P.D = D;
    P.bs = bs;
    P.chunk_base = chunk_base;
    P.err = reinterpret_cast<int *>(w + 2 * per);
    return launch_store(P, x_dtype, true, max_len, s);
}

// ---------------------------------------------------------------------------
// Prefill fast path: block sizes from pass A's per-block histograms and the
// code lengths (size = header + ceil(bits/8), padded to 4: codec.py:229-244),
// exclusive scan in block_index order -> arena offsets (codec.py:308-326),
// counters update.  One 1024-thread CTA per tensor (blockIdx.y).
// ---------------------------------------------------------------------------
namespace {
// Arena offsets for the prefill fast path, all CTAs at once: CTA (c, t) takes
// blocks [1024c, 1024c + 1024) of tensor t, sizes them from pass A's block
// histograms and the code lengths, scans them locally, and gets the prefix of
// the CTAs before it by a decoupled look-back over per-CTA status words (the
// config-2 slice's 20 CTAs).  The last CTA to finish (ticket) writes the arena
// counters.  ws per tensor: [0] bits, [1] bytes, [2] max extent, [3] bad,
// [4] ticket, [5..7] pad, [8..8+NC) status (flag << 62 | value); zeroed by the
// launcher.  Replaces a single-CTA loop over the blocks (52 us -> a few us).
__global__ void __launch_bounds__(1024)
store_offsets_kernel(StoreParams P, unsigned long long *nb0, unsigned long long *ws_all, int NC) {
    const int t = blockIdx.y, c = blockIdx.x;
    const StoreTensor S = P.t[t];
    const long nb = (long)P.n_chunks * P.H_local;
    const uint16_t *bh = P.blk_hist + (size_t)t * nb * 32;
    const int n_units = S.mode == KVC_V_TOKEN ? P.bs : P.D;
    const uint32_t hdr = kvc_header_bytes(P.bs, n_units);
    unsigned long long *ws = ws_all + (size_t)t * (8 + NC);
    unsigned long long *status = ws + 8;
    __shared__ uint32_t len[32];
    __shared__ unsigned long long wsum[32];
    __shared__ unsigned long long s_prefix;
    __shared__ unsigned long long r_bits[32], r_bytes[32];
    __shared__ uint32_t r_mx[32];
    __shared__ int r_bad;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid < 32) len[tid] = S.cb->lengths[tid];
    if (tid == 0) r_bad = 0;
    const uint64_t cursor = S.counters->cursor, n0 = S.counters->n_blocks;
    __syncthreads();
    const long b = (long)c * 1024 + tid;
    uint32_t size = 0, bits = 0, by = 0;
    bool bad = false;
    if (b < nb) {
        const uint4 *h4 = reinterpret_cast<const uint4 *>(bh + (size_t)b * 32);
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
            const uint4 u = h4[qq];
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int s0 = 8 * qq + 2 * k;
                const uint32_t c0 = w[k] & 0xFFFFu, c1 = w[k] >> 16;
                bad |= (c0 && !len[s0]) || (c1 && !len[s0 + 1]);
                bits += c0 * len[s0] + c1 * len[s0 + 1];
            }
        }
        by = (bits + 7) / 8;
        size = (hdr + by + 3) & ~3u;
    }
    unsigned long long v = size;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) wsum[warp] = v;
    unsigned long long pbits = bits, pbytes = by;
    uint32_t mx = size;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        pbits += __shfl_xor_sync(0xffffffffu, pbits, o);
        pbytes += __shfl_xor_sync(0xffffffffu, pbytes, o);
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
        r_bits[warp] = pbits;
        r_bytes[warp] = pbytes;
        r_mx[warp] = mx;
    }
    if (bad) r_bad = 1;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        wsum[lane] = w;
        const unsigned long long total = __shfl_sync(0xffffffffu, w, 31);  // this CTA's sum
        // decoupled look-back (thread 0): publish the aggregate, then walk back
        if (lane == 0) {
            const unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kMask = (1ull << 62) - 1;
            if (c == 0) {
                st_release(&status[0], kInc | total);
                s_prefix = 0;
            } else {
                st_release(&status[c], kAgg | total);
                unsigned long long pre = 0;
                for (int q = c - 1; q >= 0; --q) {
                    unsigned long long sw;
                    do { sw = ld_acquire(&status[q]); } while ((sw >> 62) == 0);
                    pre += sw & kMask;
                    if ((sw >> 62) == 2) break;
                }
                st_release(&status[c], kInc | (pre + total));
                s_prefix = pre;
            }
        }
    }
    __syncthreads();
    const unsigned long long excl = s_prefix + (warp ? wsum[warp - 1] : 0ull) + v - size;
    if (b < nb) S.offsets[n0 + b] = (uint32_t)(cursor + excl);
    if (tid == 0) {
        unsigned long long tb = 0, ty = 0;
        uint32_t m = 0;
        for (int w = 0; w < 32; ++w) {
            tb += r_bits[w];
            ty += r_bytes[w];
            m = max(m, r_mx[w]);
        }
        atomicAdd(&ws[0], tb);
        atomicAdd(&ws[1], ty);
        atomicMax(&ws[2], (unsigned long long)m);
        if (r_bad) atomicOr(&ws[3], 1ull);
        __threadfence();
        if (atomicAdd(&ws[4], 1ull) == (unsigned long long)(NC - 1)) {
            __threadfence();
            // last CTA: every status is inclusive by now; its own holds the total
            const unsigned long long total = ld_acquire(&status[NC - 1]) & ((1ull << 62) - 1);
            const unsigned long long bits_all = atomicAdd(&ws[0], 0ull);
            const unsigned long long bytes_all = atomicAdd(&ws[1], 0ull);
            const unsigned long long mx_all = atomicAdd(&ws[2], 0ull);
            const bool bad_all = atomicAdd(&ws[3], 0ull) != 0;
            nb0[t] = n0;
            kvc_arena_counters *ct = S.counters;
            if (bad_all) {
                if (!ct->err) ct->err = KVC_ERR_CODEC;
            } else if (cursor + total > S.capacity || cursor + total > 0xFFFFFFFFull) {
                if (!ct->err) ct->err = KVC_ERR_ARENA_FULL;
            } else {
                ct->cursor = cursor + total;
                ct->n_blocks = n0 + (uint64_t)nb;
                ct->payload_bits += bits_all;
                ct->payload_bytes += bytes_all;
                if ((uint32_t)mx_all > ct->max_extent) ct->max_extent = (uint32_t)mx_all;
            }
        }
    }
}
}  // namespace

extern "C" int kvc_store_prefill_supported(int bs, int D, double rel_k, double rel_v) {
    return kvc_store_supported(bs, D, 1) && ceil(1.0 / rel_k) < 32 && ceil(1.0 / rel_v) < 32;
}

extern "C" size_t kvc_store_blk_hist_bytes(int n_chunks, int H) {
    return (size_t)2 * (size_t)(n_chunks > 0 ? n_chunks : 1) * H * 32 * sizeof(uint16_t);
}

// codes_dev (optional, hot shape head_dim 128 / block 64 only): [2][nb][64*128] u8
// codes, then f32 (min, scale) pairs [nb][128] for K and [nb][64] for V
extern "C" size_t kvc_store_codes_bytes(int n_chunks, int H) {
    const size_t nb = (size_t)(n_chunks > 0 ? n_chunks : 1) * H;
    return nb * (2 * 8192 + 8 * (128 + 64));
}

static void codes_layout(StoreParams &P, uint8_t *codes_dev, long nb) {
    if (!codes_dev || P.D != 128 || P.bs != 64) return;
    P.t[0].codes_io = codes_dev;
    P.t[1].codes_io = codes_dev + (size_t)nb * 8192;
    float *m = reinterpret_cast<float *>(codes_dev + (size_t)nb * 2 * 8192);
    P.t[0].metas_io = m;
    P.t[1].metas_io = m + (size_t)nb * 128 * 2;
}

extern "C" int kvc_store_hist_blocks(const void *k_dev, const void *v_dev, int x_dtype,
                                     long row_stride, int n_chunks, int H, int D, int bs,
                                     int k_mode, double rel_k, double rel_v,
                                     const float *k_ranges_dev, uint64_t *hist_dev,
                                     uint16_t *blk_hist_dev, uint8_t *codes_dev, void *stream) {
    if (k_mode != KVC_K_BLOCK && k_mode != KVC_K_CHANNEL) return kvc_fail(KVC_ERR_CONFIG, "bad K mode");
    if (k_mode == KVC_K_CHANNEL && !k_ranges_dev)
        return kvc_fail(KVC_ERR_CONFIG, "K_CHANNEL quantization requires whole-context channel_ranges");
    if (!kvc_store_prefill_supported(bs, D, rel_k, rel_v) || !blk_hist_dev)
        return kvc_fail(KVC_ERR_CONFIG, "shape / alphabet not covered by the prefill fast path");
    if (n_chunks == 0) return KVC_OK;
    StoreParams P{};
    P.t[0].x = k_dev;
    P.t[0].mode = k_mode;
    P.t[0].ranges = k_ranges_dev;
    P.t[0].rel = rel_k;
    P.t[0].hist = reinterpret_cast<unsigned long long *>(hist_dev);
    P.t[0].max_code = (int)ceil(1.0 / rel_k);
    P.t[1].max_code = (int)ceil(1.0 / rel_v);
    P.t[1].x = v_dev;
    P.t[1].mode = KVC_V_TOKEN;
    P.t[1].rel = rel_v;
    P.t[1].hist = reinterpret_cast<unsigned long long *>(hist_dev) + 256;
    P.row_stride = row_stride;
    P.n_chunks = n_chunks;
    P.H_local = H;
    P.H_total = H;
    P.D = D;
    P.bs = bs;
    P.blk_hist = blk_hist_dev;
    codes_layout(P, codes_dev, (long)n_chunks * H);
    return launch_store(P, x_dtype, false, 1, static_cast<cudaStream_t>(stream));
}

extern "C" int kvc_store_prefill(const void *k_dev, const void *v_dev, int x_dtype, long row_stride,
                                 int n_chunks, int H_local, int H_total, int head_base, int D,
                                 int bs, int k_mode, double rel_k, double rel_v,
                                 const float *k_ranges_dev, uint32_t chunk_base,
                                 const kvc_codebook_dev *k_cb_dev, int k_max_len,
                                 const kvc_codebook_dev *v_cb_dev, int v_max_len,
                                 uint8_t *k_arena_dev, uint64_t k_capacity, uint32_t *k_offsets_dev,
                                 kvc_arena_counters *k_counters_dev, uint8_t *v_arena_dev,
                                 uint64_t v_capacity, uint32_t *v_offsets_dev,
                                 kvc_arena_counters *v_counters_dev, const uint16_t *blk_hist_dev,
                                 const uint8_t *codes_dev, void *workspace_dev,
                                 size_t workspace_bytes, void *stream) {
    if (n_chunks == 0) return KVC_OK;
    if (k_mode != KVC_K_BLOCK && k_mode != KVC_K_CHANNEL) return kvc_fail(KVC_ERR_CONFIG, "bad K mode");
    if (k_mode == KVC_K_CHANNEL && !k_ranges_dev)
        return kvc_fail(KVC_ERR_CONFIG, "K_CHANNEL quantization requires whole-context channel_ranges");
    const int max_len = k_max_len > v_max_len ? k_max_len : v_max_len;
    if (!kvc_store_prefill_supported(bs, D, rel_k, rel_v) || !kvc_store_supported(bs, D, max_len) ||
        !blk_hist_dev)
        return kvc_fail(KVC_ERR_CONFIG, "shape / alphabet not covered by the prefill fast path");
    if (workspace_bytes < 64) return kvc_fail(KVC_ERR_CONFIG, "store workspace too small");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    StoreParams P{};
    for (int t = 0; t < 2; ++t) {
        StoreTensor &T = P.t[t];
        T.x = t ? v_dev : k_dev;
        T.mode = t ? KVC_V_TOKEN : k_mode;
        T.rel = t ? rel_v : rel_k;
        T.max_code = (int)ceil(1.0 / T.rel);
        T.ranges = t ? nullptr : k_ranges_dev;
        T.cb = t ? v_cb_dev : k_cb_dev;
        T.arena = t ? v_arena_dev : k_arena_dev;
        T.capacity = t ? v_capacity : k_capacity;
        T.offsets = t ? v_offsets_dev : k_offsets_dev;
        T.counters = t ? v_counters_dev : k_counters_dev;
    }
    P.row_stride = row_stride;
    P.n_chunks = n_chunks;
    P.H_local = H_local;
    P.H_total = H_total;
    P.head_base = head_base;
    P.D = D;
    P.bs = bs;
    P.chunk_base = chunk_base;
    P.blk_hist = const_cast<uint16_t *>(blk_hist_dev);
    unsigned long long *nb0 = static_cast<unsigned long long *>(workspace_dev);  // [2]
    P.err = reinterpret_cast<int *>(nb0 + 2);
    const long nbl = (long)n_chunks * H_local;
    const int NC = (int)((nbl + 1023) / 1024);
    // offsets-kernel scratch at +256: per tensor 8 accumulators + NC status words
    unsigned long long *ows = reinterpret_cast<unsigned long long *>(static_cast<char *>(workspace_dev) + 256);
    const size_t scratch = 256 + (size_t)2 * (8 + NC) * 8;
    if (workspace_bytes < scratch) return kvc_fail(KVC_ERR_CONFIG, "store workspace too small");
    KVC_CUDA_TRY(cudaMemsetAsync(workspace_dev, 0, scratch, s));
    store_offsets_kernel<<<dim3(NC, 2), 1024, 0, s>>>(P, nb0, ows, NC);
    int st = kvc_check_launch("store_offsets_kernel");
    if (st) return st;
    P.nb0 = nb0;
    codes_layout(P, const_cast<uint8_t *>(codes_dev), (long)n_chunks * H_local);
    return launch_store(P, x_dtype, true, max_len, s);
}
