// store.cu — Store path: error-bounded quantisation + warp-aggregated
// histogram, then block-parallel canonical-Huffman encode with a
// deterministic prefix sum over block sizes and append to the arena.
//
// Reference behaviour (bit-exact):
//   quantize_block / _quantize_grid   quantizer.py:114-141, :162-209
//   build_histogram                   codebook.py:75-80
//   compress_block / _codeword_bits   codec.py:77-138
//   _serialize_block                  codec.py:229-244
//   CompressedArena.append            codec.py:308-326 (we scan instead of
//                                     taking an atomic cursor, so offsets come
//                                     out in block_index order as the oracle's)
#include <cub/cub.cuh>

#include "common.cuh"

namespace {

constexpr int kQuantThreads = 128;
constexpr int kEncThreads = 256;

// ---------------------------------------------------------------------------
// Quantisation.  f64 arithmetic, identical IEEE ops to numpy:
//   scale = f32(rel * (f64(max) - f64(min)))
//   t     = (f64(x) - f64(min)) / f64(scale);  code = floor(t) + (frac >= .5)
// Fast path: t' = d * RN(1/s) and only when t' is within a few ulps of a
// half-integer (the only decision boundaries of round-half-up) recompute with
// the correctly rounded division.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint8_t quant_code(double x, float vmin, double s64, double r64) {
    if (!(s64 > 0.0)) return 0;
    double d = __dsub_rn(x, (double)vmin);
    double t = __dmul_rn(d, r64);
    double f = floor(t);
    double frac = __dsub_rn(t, f);
    // |t' - t| <= ~2 ulp(t); widen to 8 ulp of a value up to 256 (2^-44).
    // Integers are not decision boundaries (code = m for t in [m-.5, m+.5)).
    if (fabs(frac - 0.5) < 1.0e-11 * (t + 1.0)) {
        t = __ddiv_rn(d, s64);
        f = floor(t);
        frac = __dsub_rn(t, f);
    }
    if (frac >= 0.5) f += 1.0;
    return (uint8_t)(int)f;
}

// Aggregated histogram update: one smem atomic per distinct code in the warp.
__device__ __forceinline__ void hist_add(uint32_t *sh_hist, uint32_t code, bool valid) {
    uint32_t active = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    uint32_t peers = __match_any_sync(active, code);
    int leader = __ffs(peers) - 1;
    if ((threadIdx.x & 31) == leader) atomicAdd(&sh_hist[code], (uint32_t)__popc(peers));
}

// K_CHANNEL (quantizer.py:191-197): whole-context ranges, codes clipped to
// [0, clamp_max] (values outside the ranges appear after they were fixed).
__device__ __forceinline__ uint8_t quant_code_clip(double x, float vmin, double s64, double r64,
                                                   int clamp_max) {
    if (!(s64 > 0.0)) return 0;
    double d = __dsub_rn((double)x, (double)vmin);
    double t = __dmul_rn(d, r64);
    double f = floor(t);
    double frac = __dsub_rn(t, f);
    if (fabs(frac - 0.5) < 1.0e-11 * (fabs(t) + 1.0)) {
        t = __ddiv_rn(d, s64);
        f = floor(t);
        frac = __dsub_rn(t, f);
    }
    if (frac >= 0.5) f += 1.0;
    f = fmin(fmax(f, 0.0), (double)clamp_max);
    return (uint8_t)(int)f;
}

template <typename T>
__global__ void __launch_bounds__(kQuantThreads)
quantize_kernel(const T *__restrict__ x, long row_stride, int H, int D, int bs, int mode,
                double rel, const float *__restrict__ ranges, int clamp_max,
                uint8_t *__restrict__ codes, float *__restrict__ metas,
                unsigned long long *__restrict__ hist) {
    __shared__ uint32_t sh_hist[256];
    const long b = blockIdx.x;
    const int chunk = (int)(b / H), head = (int)(b % H);
    const T *blk = x + (long)chunk * bs * row_stride + (long)head * D;
    uint8_t *out = codes + b * (long)bs * D;
    const bool do_hist = hist != nullptr;
    if (do_hist)
        for (int i = threadIdx.x; i < 256; i += blockDim.x) sh_hist[i] = 0;
    __syncthreads();

    if (mode == KVC_V_TOKEN) {
        // one unit per token row: a warp per row, lanes stride over D
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
        float *m = metas + b * (long)bs * 2;
        for (int r = warp; r < bs; r += nw) {
            const T *row = blk + (long)r * row_stride;
            float lo = 3.4e38f, hi = -3.4e38f;
            for (int c = lane; c < D; c += 32) {
                float v = (float)kvc_load_d(row + c);
                lo = fminf(lo, v);
                hi = fmaxf(hi, v);
            }
            lo = kvc_warp_min(lo);
            hi = kvc_warp_max(hi);
            float scale = (float)__dmul_rn(rel, __dsub_rn((double)hi, (double)lo));
            double s64 = (double)scale;
            double r64 = s64 > 0.0 ? __drcp_rn(s64) : 0.0;
            for (int c0 = 0; c0 < D; c0 += 32) {
                int c = c0 + lane;
                bool ok = c < D;
                uint8_t code = ok ? quant_code(kvc_load_d(row + c), lo, s64, r64) : 0;
                if (ok) out[(long)r * D + c] = code;
                if (do_hist) hist_add(sh_hist, code, ok);
            }
            if (lane == 0) {
                m[2 * r] = lo;
                m[2 * r + 1] = scale;
            }
        }
    } else {
        // K_BLOCK: one unit per channel column over the block's bs tokens
        float *m = metas + b * (long)D * 2;
        for (int c0 = 0; c0 < D; c0 += blockDim.x) {
            int c = c0 + threadIdx.x;
            bool ok = c < D;
            float lo = 3.4e38f, hi = -3.4e38f;
            if (ok && ranges) {  // K_CHANNEL: ranges [2][H][D]
                lo = ranges[(long)head * D + c];
                hi = ranges[(long)(H + head) * D + c];
            } else if (ok) {
                for (int r = 0; r < bs; ++r) {
                    float v = (float)kvc_load_d(blk + (long)r * row_stride + c);
                    lo = fminf(lo, v);
                    hi = fmaxf(hi, v);
                }
            }
            float scale = ok ? (float)__dmul_rn(rel, __dsub_rn((double)hi, (double)lo)) : 0.f;
            double s64 = (double)scale;
            double r64 = s64 > 0.0 ? __drcp_rn(s64) : 0.0;
            for (int r = 0; r < bs; ++r) {
                const double xv = ok ? kvc_load_d(blk + (long)r * row_stride + c) : 0.0;
                uint8_t code = !ok ? 0
                               : ranges ? quant_code_clip(xv, lo, s64, r64, clamp_max)
                                        : quant_code(xv, lo, s64, r64);
                if (ok) out[(long)r * D + c] = code;
                if (do_hist) hist_add(sh_hist, code, ok);
            }
            if (ok) {
                m[2 * c] = lo;
                m[2 * c + 1] = scale;
            }
        }
    }
    if (do_hist) {
        __syncthreads();
        for (int i = threadIdx.x; i < 256; i += blockDim.x)
            if (sh_hist[i]) atomicAdd(&hist[i], (unsigned long long)sh_hist[i]);
    }
}

// ---------------------------------------------------------------------------
// Encode, pass 1: per-slice bit counts and serialised block sizes.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kEncThreads)
block_size_kernel(const uint8_t *__restrict__ codes, int bs, int D, int n_units,
                  const kvc_codebook_dev *__restrict__ cb, uint32_t *__restrict__ slice_bits,
                  unsigned long long *__restrict__ block_bytes, unsigned long long *pay_bytes,
                  unsigned long long *pay_bits, uint32_t *max_extent, int *err) {
    __shared__ uint8_t sh_len[256];
    __shared__ unsigned long long sh_total;
    const long b = blockIdx.x;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh_len[i] = cb->lengths[i];
    if (threadIdx.x == 0) sh_total = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const uint8_t *blk = codes + b * (long)bs * D;
    for (int r = warp; r < bs; r += nw) {
        uint32_t cnt = 0;
        bool missing = false;
        for (int c = lane; c < D; c += 32) {
            uint32_t l = sh_len[blk[(long)r * D + c]];
            missing |= (l == 0);
            cnt += l;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (__any_sync(0xffffffffu, missing) && lane == 0) kvc_set_err(err, KVC_ERR_CODEC);
        if (lane == 0) {
            if (cnt > 0xFFFFu) kvc_set_err(err, KVC_ERR_CODEC);
            slice_bits[b * bs + r] = cnt;
            atomicAdd(&sh_total, (unsigned long long)cnt);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long bits = sh_total;
        unsigned long long pbytes = (bits + 7) / 8;
        unsigned long long raw = (unsigned long long)kvc_header_bytes(bs, n_units) + pbytes;
        unsigned long long total = (raw + 3) & ~3ull;
        if (bits > 0xFFFFFFFFull) kvc_set_err(err, KVC_ERR_CODEC);
        block_bytes[b] = total;
        atomicAdd(pay_bytes, pbytes);
        atomicAdd(pay_bits, bits);
        atomicMax(max_extent, (uint32_t)total);
    }
}

// Big-endian-word image helpers: image byte j lives in word j>>2 at bits
// [8*(3-(j&3)), +8).  The stream bit p lives in word p>>5 at bit 31-(p&31).
__device__ __forceinline__ void img_or_byte(uint32_t *img, long j, uint32_t v) {
    atomicOr(&img[j >> 2], (v & 0xFFu) << (8 * (3 - (j & 3))));
}
__device__ __forceinline__ void img_or_bits32(uint32_t *img, uint64_t p, uint32_t v) {
    uint32_t s = (uint32_t)(p & 31);
    atomicOr(&img[p >> 5], v >> s);
    if (s) atomicOr(&img[(p >> 5) + 1], v << (32 - s));
}

// ---------------------------------------------------------------------------
// Encode, pass 2: compose each block image in shared memory (header, u16
// counts, metas, MSB-first payload), then coalesced u32 stores to the arena
// at cursor + exclusive-scan offset.  Capacity is checked before any write.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kEncThreads)
block_write_kernel(const uint8_t *__restrict__ codes, const float *__restrict__ metas, int nb,
                   int H_local, int H_total, int head_base, uint32_t chunk_base, int bs, int D,
                   int n_units, const kvc_codebook_dev *__restrict__ cb,
                   const uint32_t *__restrict__ slice_bits,
                   const unsigned long long *__restrict__ block_bytes,
                   const unsigned long long *__restrict__ rel_off, uint8_t *__restrict__ arena,
                   uint64_t capacity, uint32_t *__restrict__ offsets,
                   const kvc_arena_counters *__restrict__ counters, const int *err) {
    extern __shared__ uint32_t img[];
    __shared__ uint32_t sh_words[256];
    __shared__ uint8_t sh_len[256];
    __shared__ uint32_t sh_off[1024 + 32];
    const long b = blockIdx.x;
    if (*err) return;
    const uint64_t cursor = counters->cursor;
    const unsigned long long total = rel_off[nb - 1] + block_bytes[nb - 1];
    if (cursor + total > capacity || cursor + total > 0xFFFFFFFFull) return;  // commit flags it
    const unsigned long long size = block_bytes[b];
    const int words = (int)(size >> 2);
    for (int i = threadIdx.x; i < words; i += blockDim.x) img[i] = 0;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        sh_words[i] = cb->words[i];
        sh_len[i] = cb->lengths[i];
    }
    // exclusive scan of slice bit counts (bs <= 1024 on this path)
    const uint32_t *sb = slice_bits + b * bs;
    if (threadIdx.x < 32) {
        uint32_t carry = 0;
        for (int r0 = 0; r0 < bs; r0 += 32) {
            int r = r0 + threadIdx.x;
            uint32_t v = r < bs ? sb[r] : 0;
            uint32_t inc = kvc_warp_incl_scan(v, threadIdx.x);
            if (r < bs) sh_off[r] = carry + inc - v;
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
    __syncthreads();
    // header: block_index u32, n_slices u16, counts u16[bs], (min, scale) f32 pairs
    const int chunk = (int)(b / H_local), hl = (int)(b % H_local);
    const uint32_t block_index = (chunk_base + (uint32_t)chunk) * (uint32_t)H_total +
                                 (uint32_t)(head_base + hl);
    if (threadIdx.x < 4) img_or_byte(img, threadIdx.x, block_index >> (8 * threadIdx.x));
    if (threadIdx.x < 2) img_or_byte(img, 4 + threadIdx.x, (uint32_t)bs >> (8 * threadIdx.x));
    for (int r = threadIdx.x; r < bs; r += blockDim.x) {
        img_or_byte(img, 6 + 2 * r, sb[r]);
        img_or_byte(img, 7 + 2 * r, sb[r] >> 8);
    }
    const uint32_t *mw = reinterpret_cast<const uint32_t *>(metas + b * (long)n_units * 2);
    const long meta0 = 6 + 2L * bs;
    for (int i = threadIdx.x; i < 2 * n_units; i += blockDim.x) {
        uint32_t w = mw[i];
        for (int k = 0; k < 4; ++k) img_or_byte(img, meta0 + 4L * i + k, w >> (8 * k));
    }
    // payload: thread per slice, 64-bit accumulator flushed 32 bits at a time
    const uint64_t pay_bit0 = (uint64_t)kvc_header_bytes(bs, n_units) * 8;
    const uint8_t *blk = codes + b * (long)bs * D;
    for (int r = threadIdx.x; r < bs; r += blockDim.x) {
        uint64_t p = pay_bit0 + sh_off[r];
        uint64_t acc = 0;
        int nacc = 0;
        const uint8_t *row = blk + (long)r * D;
        for (int c = 0; c < D; ++c) {
            uint32_t s = row[c];
            int l = sh_len[s];
            uint64_t w = sh_words[s];
            // l <= 32, nacc < 32  => fits in 64 bits
            acc |= w << (64 - nacc - l);
            nacc += l;
            if (nacc >= 32) {
                img_or_bits32(img, p, (uint32_t)(acc >> 32));
                p += 32;
                acc <<= 32;
                nacc -= 32;
            }
        }
        if (nacc) img_or_bits32(img, p, (uint32_t)(acc >> 32));
    }
    __syncthreads();
    // coalesced write-out (blocks start 4-byte aligned)
    const uint64_t off = cursor + rel_off[b];
    uint32_t *dst = reinterpret_cast<uint32_t *>(arena + off);
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = __byte_perm(img[i], 0, 0x0123);
    if (threadIdx.x == 0) offsets[counters->n_blocks + b] = (uint32_t)off;
}

__global__ void commit_kernel(int nb, const unsigned long long *block_bytes,
                              const unsigned long long *rel_off, uint64_t capacity,
                              const unsigned long long *pay_bytes,
                              const unsigned long long *pay_bits, const uint32_t *max_extent,
                              kvc_arena_counters *counters, const int *err) {
    if (*err) {
        if (!counters->err) counters->err = *err;
        return;
    }
    unsigned long long total = rel_off[nb - 1] + block_bytes[nb - 1];
    if (counters->cursor + total > capacity || counters->cursor + total > 0xFFFFFFFFull) {
        if (!counters->err) counters->err = KVC_ERR_ARENA_FULL;
        return;
    }
    counters->cursor += total;
    counters->n_blocks += (uint64_t)nb;
    counters->payload_bits += *pay_bits;
    counters->payload_bytes += *pay_bytes;
    if (*max_extent > counters->max_extent) counters->max_extent = *max_extent;
}

struct EncodeWs {
    uint32_t *slice_bits;
    unsigned long long *block_bytes;
    unsigned long long *rel_off;
    unsigned long long *scalars;  // pay_bytes, pay_bits
    uint32_t *max_extent;
    int *err;
    void *cub_tmp;
    size_t cub_bytes;
};

size_t cub_scan_bytes(int nb) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (unsigned long long *)nullptr,
                                  (unsigned long long *)nullptr, nb);
    return bytes;
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

EncodeWs carve(void *ws, int nb, int bs) {
    EncodeWs w;
    char *p = static_cast<char *>(ws);
    w.slice_bits = reinterpret_cast<uint32_t *>(p);
    p += align256(sizeof(uint32_t) * (size_t)nb * bs);
    w.block_bytes = reinterpret_cast<unsigned long long *>(p);
    p += align256(sizeof(unsigned long long) * (size_t)nb);
    w.rel_off = reinterpret_cast<unsigned long long *>(p);
    p += align256(sizeof(unsigned long long) * (size_t)nb);
    w.scalars = reinterpret_cast<unsigned long long *>(p);
    w.max_extent = reinterpret_cast<uint32_t *>(p + 16);
    w.err = reinterpret_cast<int *>(p + 20);
    p += 256;
    w.cub_tmp = p;
    w.cub_bytes = cub_scan_bytes(nb);
    return w;
}

}  // namespace

extern "C" size_t kvc_encode_workspace_bytes(int nb, int bs) {
    if (nb < 1) nb = 1;
    return align256(sizeof(uint32_t) * (size_t)nb * bs) + 2 * align256(8 * (size_t)nb) + 256 +
           align256(cub_scan_bytes(nb)) + 256;
}

extern "C" int kvc_quantize(const void *x_dev, int x_dtype, long row_stride, int n_chunks, int H,
                            int D, int bs, int mode, double rel, const float *k_ranges_dev,
                            uint8_t *codes_dev, float *metas_dev, uint64_t *hist_dev,
                            void *stream) {
    if (n_chunks < 0 || H < 1 || D < 1 || bs < 1) return kvc_fail(KVC_ERR_CONFIG, "bad shape");
    if (mode != KVC_K_BLOCK && mode != KVC_V_TOKEN && mode != KVC_K_CHANNEL)
        return kvc_fail(KVC_ERR_CONFIG, "unknown quantisation mode");
    if (mode == KVC_K_CHANNEL && k_ranges_dev == nullptr)
        return kvc_fail(KVC_ERR_CONFIG, "K_CHANNEL quantization requires whole-context channel_ranges");
    if (mode != KVC_K_CHANNEL) k_ranges_dev = nullptr;
    if (!(rel >= 1.0 / 255.0 && rel <= 1.0)) return kvc_fail(KVC_ERR_CONFIG, "rel outside [1/255, 1]");
    const int clamp_max = (int)ceil(1.0 / rel);
    long nb = (long)n_chunks * H;
    if (nb == 0) return KVC_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto *hist = reinterpret_cast<unsigned long long *>(hist_dev);
    if (x_dtype == KVC_F16)
        quantize_kernel<__half><<<(unsigned)nb, kQuantThreads, 0, s>>>(
            static_cast<const __half *>(x_dev), row_stride, H, D, bs, mode, rel, k_ranges_dev,
            clamp_max, codes_dev, metas_dev, hist);
    else if (x_dtype == KVC_F32)
        quantize_kernel<float><<<(unsigned)nb, kQuantThreads, 0, s>>>(
            static_cast<const float *>(x_dev), row_stride, H, D, bs, mode, rel, k_ranges_dev,
            clamp_max, codes_dev, metas_dev, hist);
    else if (x_dtype == KVC_F64)  // quantize_unit on float64 values (quantizer.py:144-160)
        quantize_kernel<double><<<(unsigned)nb, kQuantThreads, 0, s>>>(
            static_cast<const double *>(x_dev), row_stride, H, D, bs, mode, rel, k_ranges_dev,
            clamp_max, codes_dev, metas_dev, hist);
    else
        return kvc_fail(KVC_ERR_TENSOR, "unsupported dtype");
    return kvc_check_launch("quantize_kernel");
}

extern "C" int kvc_encode_append(const uint8_t *codes_dev, const float *metas_dev, int n_chunks,
                                 int H_local, int H_total, int head_base, uint32_t chunk_base,
                                 int bs, int D, int n_units, int max_len,
                                 const kvc_codebook_dev *cb_dev, uint8_t *arena_dev,
                                 uint64_t capacity, uint32_t *offsets_dev,
                                 kvc_arena_counters *counters_dev, void *workspace_dev,
                                 void *stream) {
    const int nb = n_chunks * H_local;
    if (nb == 0) return KVC_OK;
    if (bs > 1024) return kvc_fail(KVC_ERR_CONFIG, "block_size > 1024 unsupported by the encoder");
    if (max_len < 1 || max_len > 32) return kvc_fail(KVC_ERR_CODEBOOK, "bad max code length");
    const size_t img_bytes =
        (size_t)kvc_header_bytes(bs, n_units) + ((size_t)bs * D * max_len + 7) / 8 + 16;
    if (img_bytes > 200 * 1024)
        return kvc_fail(KVC_ERR_CONFIG, "block image exceeds shared memory (bs*D*max_len too large)");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    EncodeWs w = carve(workspace_dev, nb, bs);
    KVC_CUDA_TRY(cudaMemsetAsync(w.scalars, 0, 32, s));
    block_size_kernel<<<nb, kEncThreads, 0, s>>>(codes_dev, bs, D, n_units, cb_dev, w.slice_bits,
                                                 w.block_bytes, &w.scalars[0], &w.scalars[1],
                                                 w.max_extent, w.err);
    int st = kvc_check_launch("block_size_kernel");
    if (st) return st;
    size_t tmp = w.cub_bytes;
    KVC_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.cub_tmp, tmp, w.block_bytes, w.rel_off, nb, s));
    static bool attr_set = false;
    if (!attr_set) {
        KVC_CUDA_TRY(cudaFuncSetAttribute(block_write_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr_set = true;
    }
    block_write_kernel<<<nb, kEncThreads, img_bytes, s>>>(
        codes_dev, metas_dev, nb, H_local, H_total, head_base, chunk_base, bs, D, n_units, cb_dev,
        w.slice_bits, w.block_bytes, w.rel_off, arena_dev, capacity, offsets_dev, counters_dev,
        w.err);
    st = kvc_check_launch("block_write_kernel");
    if (st) return st;
    commit_kernel<<<1, 1, 0, s>>>(nb, w.block_bytes, w.rel_off, capacity, &w.scalars[0],
                                  &w.scalars[1], w.max_extent, counters_dev, w.err);
    return kvc_check_launch("commit_kernel");
}
