// fetch_generic.cu — shape-generic Fetch kernels (any head_dim / block_size /
// code length).  They serve the reference's drop-in functions one-to-one:
//   fused_k_scores   attention.py:59-109   -> kvc_k_scores
//   softmax_rows     attention.py:168-173  -> kvc_softmax_rows
//   fused_v_output   attention.py:112-165  -> kvc_v_output
//   fetch_dequantized kvcache.py:182-212   -> kvc_dequantize
// Decoding happens inside the dot products: a thread per slice walks its
// bitstream with the codebook LUT (canonical tail for codes > 12 bits); the
// decompressed codes live only in registers / one shared-memory tile.
// Corrupt streams (codec.py:169-172, :218-223, :253-267) set *err = CodecError.
#include "common.cuh"

namespace {

constexpr int kThreads = 128;
constexpr int kMaxDPerThread = 16;  // D <= 2048

struct BlockView {
    const uint8_t *base;   // block start
    const uint8_t *end;    // extent end
    const uint8_t *payload;
    int ok;
};

__device__ __forceinline__ uint32_t ld_u16(const uint8_t *p) { return p[0] | (p[1] << 8); }
__device__ __forceinline__ float ld_f32(const uint8_t *p) {
    uint32_t u = p[0] | (p[1] << 8) | (p[2] << 16) | ((uint32_t)p[3] << 24);
    return __uint_as_float(u);
}

// Parse and validate one extent (codec.py:247-268); fills shared slice offsets.
__device__ int parse_block(const uint8_t *arena, uint64_t start, uint64_t end, int bs, int n_units,
                           uint32_t *sh_off, uint32_t *sh_cnt, uint32_t *sh_tot) {
    const uint8_t *blk = arena + start;
    long len = (long)(end - start);
    int ok = (len >= 6 && (len & 3) == 0);
    if (ok) ok = (int)ld_u16(blk + 4) == bs;
    long pay_off = 6 + 2L * bs + 8L * n_units;
    if (ok) ok = pay_off <= len;
    if (ok) {
        for (int r = threadIdx.x; r < bs; r += blockDim.x) sh_cnt[r] = ld_u16(blk + 6 + 2 * r);
    }
    __syncthreads();
    if (threadIdx.x == 0 && ok) {
        uint32_t acc = 0;
        for (int r = 0; r < bs; ++r) {
            sh_off[r] = acc;
            acc += sh_cnt[r];
        }
        *sh_tot = acc;
        long pbytes = ((long)acc + 7) / 8;
        long pad = len - pay_off - pbytes;
        if (pad < 0 || pad > 3) ok = 0;
    }
    return ok;
}

// Decode slice r (bit_count bits at bit_off of payload) into D codes; calls
// sink(c, code) per symbol.  Returns false on a corrupt slice.
template <typename Sink>
__device__ __forceinline__ bool decode_slice(const kvc_codebook_dev *cb, const uint8_t *payload,
                                             const uint8_t *end, uint32_t bit_off,
                                             uint32_t bit_count, int D, Sink sink) {
    KvcBitReader br;
    br.init(payload, bit_off, end + 8);
    uint32_t used = 0;
    bool good = true;
    for (int c = 0; c < D; ++c) {
        int len;
        int sym = kvc_decode_symbol(cb, br.peek32(), len);
        if (!len) { good = false; len = 1; }
        used += (uint32_t)len;
        br.consume(len);
        sink(c, sym);
    }
    return good && used == bit_count;
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
k_scores_kernel(const kvc_seq_desc *__restrict__ seqs, int H, int D, int bs,
                const float *__restrict__ q, float *__restrict__ scores, long ctx_stride,
                int *err) {
    extern __shared__ float sh_f[];  // folded[D]
    __shared__ uint32_t sh_off[1024], sh_cnt[1024], sh_tot;
    __shared__ float sh_base;
    const int h = blockIdx.y, sidx = blockIdx.z;
    const kvc_seq_desc sd = kvc_load_desc(seqs, sidx);
    const float *qh = q + ((long)sidx * H + h) * D;
    float *out = scores + ((long)sidx * H + h) * ctx_stride;
    const float inv = (float)(1.0 / sqrt((double)D));
    const long n_blocks = (long)sd.n_chunks * H;
    for (int chunk = blockIdx.x; chunk < sd.n_chunks; chunk += gridDim.x) {
        long ord = (long)chunk * H + h;
        uint64_t start, end;
        kvc_extent(sd.k_offsets, sd.k_counters, ord, (long)sd.k_counters->n_blocks, start, end);
        __syncthreads();
        int ok = parse_block(sd.k_arena, start, end, bs, D, sh_off, sh_cnt, &sh_tot);
        ok = __syncthreads_and(ok);
        if (!ok) {
            if (threadIdx.x == 0) kvc_set_err(err, KVC_ERR_CODEC);
            continue;
        }
        const uint8_t *meta = sd.k_arena + start + 6 + 2 * bs;
        float part = 0.f;
        for (int c = threadIdx.x; c < D; c += blockDim.x) {
            float mn = ld_f32(meta + 8 * c), sc = ld_f32(meta + 8 * c + 4);
            sh_f[c] = sc * qh[c];
            part += mn * qh[c];
        }
        part = kvc_warp_sum(part);
        if (threadIdx.x == 0) sh_base = 0.f;
        __syncthreads();
        if ((threadIdx.x & 31) == 0) atomicAdd(&sh_base, part);
        __syncthreads();
        const uint8_t *payload = meta + 8 * D;
        const uint8_t *pend = sd.k_arena + end;
        for (int r = threadIdx.x; r < bs; r += blockDim.x) {
            float acc = 0.f;
            bool good = decode_slice(sd.k_cb, payload, pend, sh_off[r], sh_cnt[r], D,
                                     [&](int c, int sym) { acc = fmaf((float)sym, sh_f[c], acc); });
            if (!good) kvc_set_err(err, KVC_ERR_CODEC);
            out[(long)chunk * bs + r] = (acc + sh_base) * inv;
        }
    }
    // buffered tokens: exact dot products (attention.py:103-107)
    if (blockIdx.x == 0) {
        const long t0 = (long)sd.n_chunks * bs;
        for (int t = threadIdx.x; t < sd.buffered; t += blockDim.x) {
            const float *kv = sd.k_buffer + ((long)t * H + h) * D;
            float acc = 0.f;
            for (int c = 0; c < D; ++c) acc = fmaf(kv[c], qh[c], acc);
            out[t0 + t] = acc * inv;
        }
    }
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
v_output_kernel(const kvc_seq_desc *__restrict__ seqs, int H, int D, int bs,
                const float *__restrict__ w, long ctx_stride, float *__restrict__ partial,
                int tile_rows, int *err) {
    extern __shared__ uint8_t sh_tile[];  // [tile_rows][D] codes
    __shared__ uint32_t sh_off[1024], sh_cnt[1024], sh_tot;
    __shared__ float sh_a[1024];
    __shared__ float sh_wm;
    const int h = blockIdx.y, sidx = blockIdx.z;
    const kvc_seq_desc sd = kvc_load_desc(seqs, sidx);
    const float *wh = w + ((long)sidx * H + h) * ctx_stride;
    float acc[kMaxDPerThread];
#pragma unroll
    for (int k = 0; k < kMaxDPerThread; ++k) acc[k] = 0.f;
    float wm_total = 0.f;
    for (int chunk = blockIdx.x; chunk < sd.n_chunks; chunk += gridDim.x) {
        long ord = (long)chunk * H + h;
        uint64_t start, end;
        kvc_extent(sd.v_offsets, sd.v_counters, ord, (long)sd.v_counters->n_blocks, start, end);
        __syncthreads();
        int ok = parse_block(sd.v_arena, start, end, bs, bs, sh_off, sh_cnt, &sh_tot);
        ok = __syncthreads_and(ok);
        if (!ok) {
            if (threadIdx.x == 0) kvc_set_err(err, KVC_ERR_CODEC);
            continue;
        }
        const uint8_t *meta = sd.v_arena + start + 6 + 2 * bs;
        if (threadIdx.x == 0) sh_wm = 0.f;
        __syncthreads();
        float wmp = 0.f;
        for (int r = threadIdx.x; r < bs; r += blockDim.x) {
            float wr = wh[(long)chunk * bs + r];
            sh_a[r] = wr * ld_f32(meta + 8 * r + 4);
            wmp += wr * ld_f32(meta + 8 * r);
        }
        wmp = kvc_warp_sum(wmp);
        if ((threadIdx.x & 31) == 0) atomicAdd(&sh_wm, wmp);
        const uint8_t *payload = meta + 8 * bs;
        const uint8_t *pend = sd.v_arena + end;
        for (int r0 = 0; r0 < bs; r0 += tile_rows) {
            int rows = min(tile_rows, bs - r0);
            __syncthreads();
            for (int rr = threadIdx.x; rr < rows; rr += blockDim.x) {
                int r = r0 + rr;
                uint8_t *row = sh_tile + (long)rr * D;
                bool good = decode_slice(sd.v_cb, payload, pend, sh_off[r], sh_cnt[r], D,
                                         [&](int c, int sym) { row[c] = (uint8_t)sym; });
                if (!good) kvc_set_err(err, KVC_ERR_CODEC);
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < kMaxDPerThread; ++k) {
                int c = threadIdx.x + k * blockDim.x;
                if (c < D) {
                    float a = acc[k];
                    for (int rr = 0; rr < rows; ++rr)
                        a = fmaf(sh_a[r0 + rr], (float)sh_tile[(long)rr * D + c], a);
                    acc[k] = a;
                }
            }
        }
        __syncthreads();
        wm_total += sh_wm;
    }
    float *dst = partial + (((long)blockIdx.x * gridDim.z + sidx) * H + h) * D;
#pragma unroll
    for (int k = 0; k < kMaxDPerThread; ++k) {
        int c = threadIdx.x + k * blockDim.x;
        if (c < D) dst[c] = acc[k] + wm_total;
    }
}

// Sum split partials in split order, then add buffered tokens (attention.py:160-164).
__global__ void v_combine_kernel(const kvc_seq_desc *__restrict__ seqs, int H, int D, int splits,
                                 const float *__restrict__ partial, const float *__restrict__ w,
                                 long ctx_stride, int bs, float *__restrict__ out) {
    const int h = blockIdx.y, sidx = blockIdx.z;
    const kvc_seq_desc sd = kvc_load_desc(seqs, sidx);
    const float *wh = w + ((long)sidx * H + h) * ctx_stride;
    const long t0 = (long)sd.n_chunks * bs;
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
        float a = 0.f;
        for (int s = 0; s < splits; ++s) a += partial[(((long)s * gridDim.z + sidx) * H + h) * D + c];
        for (int t = 0; t < sd.buffered; ++t)
            a = fmaf(wh[t0 + t], sd.v_buffer[((long)t * H + h) * D + c], a);
        out[((long)sidx * H + h) * D + c] = a;
    }
}

__global__ void softmax_kernel(float *x, long n_cols, long row_stride) {
    float *row = x + (long)blockIdx.x * row_stride;
    __shared__ float sh[32];
    float m = -INFINITY;
    for (long j = threadIdx.x; j < n_cols; j += blockDim.x) m = fmaxf(m, row[j]);
    m = kvc_warp_max(m);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : -INFINITY;
        v = kvc_warp_max(v);
        if (threadIdx.x == 0) sh[0] = v;
    }
    __syncthreads();
    m = sh[0];
    __syncthreads();
    float s = 0.f;
    for (long j = threadIdx.x; j < n_cols; j += blockDim.x) {
        float e = expf(row[j] - m);
        row[j] = e;
        s += e;
    }
    s = kvc_warp_sum(s);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.f;
        v = kvc_warp_sum(v);
        if (threadIdx.x == 0) sh[0] = v;
    }
    __syncthreads();
    s = sh[0];
    for (long j = threadIdx.x; j < n_cols; j += blockDim.x) row[j] = row[j] / s;
}

// f64 dequantisation: f32(min64 + code64 * scale64), two roundings like numpy.
__global__ void __launch_bounds__(kThreads)
dequant_kernel(const kvc_seq_desc *__restrict__ seq, int H, int D, int bs, int which,
               float *__restrict__ out, int *err) {
    __shared__ uint32_t sh_off[1024], sh_cnt[1024], sh_tot;
    const long ord = blockIdx.x;
    const bool is_v = which == 1;
    const uint8_t *arena = is_v ? seq->v_arena : seq->k_arena;
    const uint32_t *offs = is_v ? seq->v_offsets : seq->k_offsets;
    const kvc_arena_counters *cnt = is_v ? seq->v_counters : seq->k_counters;
    const kvc_codebook_dev *cb = is_v ? seq->v_cb : seq->k_cb;
    const int n_units = is_v ? bs : D;
    uint64_t start, end;
    kvc_extent(offs, cnt, ord, (long)cnt->n_blocks, start, end);
    int ok = parse_block(arena, start, end, bs, n_units, sh_off, sh_cnt, &sh_tot);
    ok = __syncthreads_and(ok);
    if (!ok) {
        if (threadIdx.x == 0) kvc_set_err(err, KVC_ERR_CODEC);
        return;
    }
    const uint8_t *blk = arena + start;
    const uint32_t bi = blk[0] | (blk[1] << 8) | (blk[2] << 16) | ((uint32_t)blk[3] << 24);
    const int head = (int)(bi % (uint32_t)H);
    const long t0 = (long)(bi / (uint32_t)H) * bs;
    const uint8_t *meta = blk + 6 + 2 * bs;
    const uint8_t *payload = meta + 8 * n_units;
    for (int r = threadIdx.x; r < bs; r += blockDim.x) {
        float *row = out + ((t0 + r) * H + head) * (long)D;
        bool good = decode_slice(cb, payload, arena + end, sh_off[r], sh_cnt[r], D,
                                 [&](int c, int sym) {
                                     int u = is_v ? r : c;
                                     double mn = (double)ld_f32(meta + 8 * u);
                                     double sc = (double)ld_f32(meta + 8 * u + 4);
                                     row[c] = (float)__dadd_rn(mn, __dmul_rn((double)sym, sc));
                                 });
        if (!good) kvc_set_err(err, KVC_ERR_CODEC);
    }
}

// decompress_block (codec.py:356-391) for a list of arena ordinals: parse and
// validate each extent, decode its slices with the codebook LUT (canonical
// tail for long codes) into codes [bs, D] u8, copy the (min, scale) pairs and
// the header's block_index.  One CTA per block.
__global__ void __launch_bounds__(kThreads)
decode_blocks_kernel(const uint8_t *__restrict__ arena, const uint32_t *__restrict__ offsets,
                     const kvc_arena_counters *__restrict__ counters,
                     const int32_t *__restrict__ ordinals, int bs, int n_units, int D,
                     const kvc_codebook_dev *__restrict__ cb, uint8_t *__restrict__ codes,
                     float *__restrict__ metas, uint32_t *__restrict__ block_index, int *err) {
    __shared__ uint32_t sh_off[1024], sh_cnt[1024], sh_tot;
    const long i = blockIdx.x;
    const long nb = (long)counters->n_blocks;
    const long ord = ordinals[i];
    if (ord < 0 || ord >= nb) {
        if (threadIdx.x == 0) kvc_set_err(err, KVC_ERR_CODEC);
        return;
    }
    uint64_t start, end;
    kvc_extent(offsets, counters, ord, nb, start, end);
    int ok = parse_block(arena, start, end, bs, n_units, sh_off, sh_cnt, &sh_tot);
    ok = __syncthreads_and(ok);
    if (!ok) {
        if (threadIdx.x == 0) kvc_set_err(err, KVC_ERR_CODEC);
        return;
    }
    const uint8_t *blk = arena + start;
    if (threadIdx.x == 0)
        block_index[i] = blk[0] | (blk[1] << 8) | (blk[2] << 16) | ((uint32_t)blk[3] << 24);
    const uint8_t *meta = blk + 6 + 2 * bs;
    for (int u = threadIdx.x; u < 2 * n_units; u += blockDim.x)
        metas[i * 2 * n_units + u] = ld_f32(meta + 4 * u);
    const uint8_t *payload = meta + 8 * n_units;
    uint8_t *out = codes + i * (long)bs * D;
    for (int r = threadIdx.x; r < bs; r += blockDim.x) {
        uint8_t *row = out + (long)r * D;
        bool good = decode_slice(cb, payload, arena + end, sh_off[r], sh_cnt[r], D,
                                 [&](int c, int sym) { row[c] = (uint8_t)sym; });
        if (!good) kvc_set_err(err, KVC_ERR_CODEC);
    }
}

int max_chunks_of(const kvc_seq_desc *seqs_host, int n) { return 0; }

}  // namespace

extern "C" int kvc_k_scores(const kvc_seq_desc *seqs_dev, int n_seqs, int H, int D, int bs,
                            const float *q_dev, float *scores_dev, long ctx_stride, int *err_dev,
                            void *stream) {
    if (n_seqs < 1 || H < 1 || D < 1 || bs < 1) return kvc_fail(KVC_ERR_CONFIG, "bad shape");
    if (bs > 1024 || D > 2048) return kvc_fail(KVC_ERR_CONFIG, "shape beyond generic kernel limits");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    dim3 grid(64, H, n_seqs);
    k_scores_kernel<<<grid, kThreads, sizeof(float) * D, s>>>(seqs_dev, H, D, bs, q_dev, scores_dev,
                                                               ctx_stride, err_dev);
    return kvc_check_launch("k_scores_kernel");
}

extern "C" int kvc_softmax_rows(float *x_dev, int n_rows, long n_cols, long row_stride,
                                void *stream) {
    if (n_rows < 1 || n_cols < 1) return KVC_OK;
    softmax_kernel<<<n_rows, 256, 0, static_cast<cudaStream_t>(stream)>>>(x_dev, n_cols, row_stride);
    return kvc_check_launch("softmax_kernel");
}

extern "C" size_t kvc_v_output_workspace_bytes(int n_seqs, int H, int D) {
    return sizeof(float) * 64 * (size_t)n_seqs * H * D;
}

extern "C" int kvc_v_output(const kvc_seq_desc *seqs_dev, int n_seqs, int H, int D, int bs,
                            const float *w_dev, long ctx_stride, float *out_dev, float *ws_dev,
                            int *err_dev, void *stream) {
    if (n_seqs < 1 || H < 1 || D < 1 || bs < 1) return kvc_fail(KVC_ERR_CONFIG, "bad shape");
    if (bs > 1024 || D > 2048) return kvc_fail(KVC_ERR_CONFIG, "shape beyond generic kernel limits");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int splits = 64;
    int tile_rows = (32 * 1024) / D;
    if (tile_rows > bs) tile_rows = bs;
    if (tile_rows < 1) tile_rows = 1;
    dim3 grid(splits, H, n_seqs);
    v_output_kernel<<<grid, kThreads, (size_t)tile_rows * D, s>>>(seqs_dev, H, D, bs, w_dev,
                                                                  ctx_stride, ws_dev, tile_rows,
                                                                  err_dev);
    int st = kvc_check_launch("v_output_kernel");
    if (st) return st;
    v_combine_kernel<<<dim3(1, H, n_seqs), 128, 0, s>>>(seqs_dev, H, D, splits, ws_dev, w_dev,
                                                         ctx_stride, bs, out_dev);
    return kvc_check_launch("v_combine_kernel");
}

extern "C" int kvc_dequantize(const kvc_seq_desc *seq_dev, int H, int D, int bs, int which,
                              int n_chunks, float *out_dev, int *err_dev, void *stream) {
    if (n_chunks == 0) return KVC_OK;
    if (bs > 1024) return kvc_fail(KVC_ERR_CONFIG, "block_size > 1024 unsupported");
    dequant_kernel<<<n_chunks * H, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        seq_dev, H, D, bs, which, out_dev, err_dev);
    return kvc_check_launch("dequant_kernel");
}

extern "C" int kvc_decode_blocks(const uint8_t *arena_dev, const uint32_t *offsets_dev,
                                 const kvc_arena_counters *counters_dev,
                                 const int32_t *ordinals_dev, int n, int bs, int n_units, int D,
                                 const kvc_codebook_dev *cb_dev, uint8_t *codes_dev,
                                 float *metas_dev, uint32_t *block_index_dev, int *err_dev,
                                 void *stream) {
    if (n < 0 || bs < 1 || D < 1 || n_units < 1) return kvc_fail(KVC_ERR_CONFIG, "bad shape");
    if (bs > 1024) return kvc_fail(KVC_ERR_CONFIG, "block_size > 1024 unsupported");
    if (n == 0) return KVC_OK;
    decode_blocks_kernel<<<n, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        arena_dev, offsets_dev, counters_dev, ordinals_dev, bs, n_units, D, cb_dev, codes_dev,
        metas_dev, block_index_dev, err_dev);
    return kvc_check_launch("decode_blocks_kernel");
}
