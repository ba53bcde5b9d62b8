// fetch_fused.cu — single-pass fused Fetch for the hot shape (head_dim 128,
// block_size 64): per (sequence, KV head, context split) one CTA of NW warps;
// each warp streams its chunks' K and V block extents HBM -> shared memory
// with cp.async.bulk (TMA 1D) into a private 2-stage mbarrier ring, Huffman-
// decodes 2 slices per lane (one token each) straight into the dot products:
//   K: score_t = sum_c code_tc * (scale_c q_c) + sum_c min_c q_c   (attention.py:91-94)
//   online softmax (flash-decoding) in the log2 domain
//   V: o_c += sum_t (p_t scale_t) code_tc + sum_t p_t min_t        (attention.py:144-148)
// The decompressed KV never exists outside registers.  Split partials
// (m, l, o[128]) are merged, together with the f32 buffered tokens, by
// combine_kernel.  Also: the uncompressed fp16 decode-attention comparator.
#include <cstring>
#include <type_traits>
#include <vector>
#include <algorithm>
#include <mutex>
#include <cstdio>

#include <cstdlib>

#include "common.cuh"
#include "mma.cuh"

namespace {

constexpr int D = 128;
constexpr int BS = 64;
constexpr int NW = 4;                // warps per CTA
constexpr int kThreadsF = NW * 32;
constexpr int K_HDR = 6 + 2 * BS + 8 * D;   // 1158
constexpr int V_HDR = 6 + 2 * BS + 8 * BS;  // 646
constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + cp.async.bulk (TMA 1D)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ uint32_t lds_u16(const uint8_t *p) {
    return *reinterpret_cast<const uint16_t *>(p);
}
// f32 stored at a 2-byte aligned shared address
__device__ __forceinline__ float lds_f32_a2(const uint8_t *p) {
    const uint16_t *h = reinterpret_cast<const uint16_t *>(p);
    return __uint_as_float((uint32_t)h[0] | ((uint32_t)h[1] << 16));
}
// 32-bit MSB-first window starting at bit `pos` of a byte buffer (word aligned base)
__device__ __forceinline__ uint32_t window32(const uint32_t *w, uint32_t pos) {
    uint32_t i = pos >> 5;
    uint32_t a = __byte_perm(w[i], 0, 0x0123);
    uint32_t b = __byte_perm(w[i + 1], 0, 0x0123);
    return __funnelshift_l(b, a, pos);
}

struct Partial {
    float m;  // running max, log2 domain
    float l;  // sum of exp2
    float o[D];
};

// Shared loads on the decode path are `ld.volatile`: ptxas keeps volatile
// accesses in program order, which pins the per-step interleave of the four
// cursor chains written below (without it ptxas runs two chains far ahead of
// the other two and exposes the LDS latency).
#ifdef KVC_NONVOLATILE_LDS
#define KVC_LD_SHARED "ld.shared"
#else
#define KVC_LD_SHARED "ld.volatile.shared"
#endif
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile(KVC_LD_SHARED ".u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ float2 lds64f(uint32_t addr) {
    float2 v;
    asm volatile(KVC_LD_SHARED ".v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// One slice's bit cursor.  `base` = shared byte address of the word holding
// the slice's first bit; `p` = bit position relative to base.  Only the low
// 16 bits of p are meaningful: the cursor advances by whole LUT entries
// (consumed bits in bits 0..3, symbols in bits 16..31), so the high half
// collects garbage that is masked off where p is used.
struct Cursor {
    uint32_t win;
    uint32_t p;
    uint32_t base;
};

__device__ __forceinline__ void cursor_init(Cursor &c, uint32_t stage_addr, uint32_t bit) {
    c.base = stage_addr + ((bit >> 5) << 2);
    c.p = bit & 31u;
    c.win = 0;
}
__device__ __forceinline__ void cursor_reload(Cursor &c) {
    const uint32_t a = c.base + ((c.p >> 3) & 0x1FFCu);
    const uint32_t w0 = bswap32(lds32(a)), w1 = bswap32(lds32(a + 4));
    c.win = __funnelshift_l(w1, w0, c.p);
}
constexpr uint32_t kMagicBits = 0x4B000000u;  // float 2^23
__device__ __forceinline__ float sym_hi_byte(uint32_t e, uint32_t sel) {
    return __uint_as_float(__byte_perm(e, kMagicBits, sel));
}
// ---------------------------------------------------------------------------
// Decoder policies (selected per launch):
//   MODE 0  lane-replicated 64-entry single-symbol LUT (codes <= 6 bits):
//           entry i of lane l at word i*32+l, so every lookup is bank-
//           conflict-free; entry = float bits of the symbol | code length.
//   MODE 1  shared 4096-entry pair LUT (codes <= 6 bits): one lookup decodes
//           two symbols; entry = (l0+l1) | s0<<16 | s1<<24.
//   MODE 2  shared 4096-entry single-symbol LUT (codes <= 12 bits), float|len.
//   MODE 6  512-entry single-symbol LUT (codes <= 9 bits), float|len, in 16
//           copies: entry i of copy c at word i*16+c, lane l reads copy l&15,
//           so only lanes l and l+16 can collide (~2 wavefronts per lookup
//           instead of ~3.3 for MODE 2's random 12-bit indices).
//   MODE 7  256-entry single-symbol LUT (codes <= 8 bits) in 32 copies, one
//           per lane: every lookup is bank-conflict-free.
//   MODE 8  1024-entry single-symbol LUT (codes <= 10 bits) in 8 copies
//           (lanes l, l+8, l+16, l+24 share one).
// In every format the low 4 bits are the bits consumed and bits 4..15 are
// zero, so `win <<= e` (funnel shift masks to 5 bits) and `p += e` need no
// field extraction.
// ---------------------------------------------------------------------------
template <int MODE>
struct Dec {
    // MODE 5: single-symbol LUT over 13-bit windows (books with 13-bit codes)
    static constexpr int kLutWords = MODE == 0 ? 64 * 32 : (MODE >= 5 ? 8192 : (1 << KVC_LUT_BITS));
    // single-symbol window and symbols per 64-bit window
    static constexpr int kSymBits =
        MODE == 5 ? 13 : (MODE == 6 ? 9 : (MODE == 7 ? 8 : (MODE == 8 ? 10 : 12)));
    static constexpr int kReload =
        MODE == 5 ? 4 : (MODE == 6 ? 7 : (MODE == 7 ? 8 : (MODE == 8 ? 6 : 5)));
    static constexpr int kCopies =
        MODE == 6 ? 16 : (MODE == 7 ? 32 : (MODE == 8 ? 8 : 1));  // lane copies
    static constexpr bool kDyn = MODE >= 5;  // LUT in the dynamic shared region
    static constexpr bool kSingle = MODE == 2 || MODE >= 5;
    static constexpr bool kPair = MODE == 1 || MODE == 3 || MODE == 4;  // the 4096-entry pair LUT (TMA-loaded)
    // symbols decodable from one 32-bit window; MODE 0 uses 4 (not 5) so the
    // reload cadence divides the unrolled loop (24 of 32 bits)
    static constexpr int kSymsPerWin = MODE == 0 ? 4 : (MODE == 1 ? 4 : 2);
};

template <int MODE>
__device__ __forceinline__ uint32_t lut_addr(uint32_t win, uint32_t lut_s, uint32_t lane_s) {
    if (MODE == 0) return lane_s + ((win >> 26) << 7);   // lane_s = lut_s + 4*lane
    return lut_s + ((win >> 20) << 2);
}

// Builds the per-CTA LUT from the codebook's 12-bit decode table.
template <int MODE>
__device__ void build_lut(uint32_t *dst, const kvc_codebook_dev *cb) {
    for (int i = threadIdx.x; i < Dec<MODE>::kLutWords; i += blockDim.x) {
        uint32_t e12;
        if (MODE == 0) e12 = cb->lut[(i >> 5) << 6];
        else if (MODE == 2) e12 = cb->lut[i];
        else { dst[i] = cb->fetch_lut[i & 4095]; continue; }
        dst[i] = __float_as_uint((float)(e12 & 0xFF)) | ((e12 >> 8) & 0xF);
    }
}

// MODE 6 / 7 tables: entry i (float(sym) | len, from the 12-bit table's
// entry i << (12 - BITS): codes are <= BITS bits) in R copies, word i*R + c.
// A warp loads 32 entries and writes them out with consecutive lanes storing
// consecutive words.
template <int BITS, int R>
__device__ void build_lut_copies(uint32_t *dst, const kvc_codebook_dev *cb) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int kb = 32 * warp; kb < (1 << BITS); kb += 32 * nw) {
        const uint32_t e12 = cb->lut[(kb + lane) << (12 - BITS)];
        const uint32_t e = __float_as_uint((float)(e12 & 0xFF)) | ((e12 >> 8) & 0xF);
#pragma unroll 4
        for (int i = 0; i < R; ++i)
            dst[kb * R + 32 * i + lane] = __shfl_sync(0xffffffffu, e, i * (32 / R) + lane / R);
    }
}

// ---------------------------------------------------------------------------
// Fused fetch-attention.  Per warp, iteration i decodes K(chunk i) and
// V(chunk i-1) together (four independent cursors per lane), so the K scores
// of chunk i update the online softmax while chunk i-1's weights drive the V
// accumulation.  K and V extents have separate 2-slot TMA rings: at the end
// of iteration i, K(i+2) and V(i+1) are issued into the slots just freed.
// Iteration 0 has no V and iteration n has no K: those halves decode a stable
// dummy stream (the LUT itself) with zero weights and are discarded.
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kThreadsF, 2)
fused_attn_kernel(const kvc_seq_desc *__restrict__ seqs, int H, const float *__restrict__ q,
                  float *__restrict__ scores, long ctx_stride, Partial *__restrict__ partial,
                  int chunks_per_split, int n_splits, int stage_k, int stage_v, int *err) {
    constexpr int W = Dec<MODE>::kSymsPerWin;
    __shared__ __align__(128) uint32_t s_lut[2][Dec<MODE>::kLutWords];
    __shared__ uint64_t s_lbar[1];
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t *lutK = s_lut[0];
    uint32_t *lutV = s_lut[1];
    uint8_t *wbase = smem;
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const int per_warp = 2 * (stage_k + stage_v) + D * 4 + 64;
    uint8_t *my = wbase + warp * per_warp;
    float *qf = reinterpret_cast<float *>(my + 2 * (stage_k + stage_v));
    uint64_t *bar = reinterpret_cast<uint64_t *>(my + 2 * (stage_k + stage_v) + D * 4);
    const uint32_t my_s = smem_u32(my);
    const uint32_t kslot0 = my_s, vslot0 = my_s + 2 * stage_k;
    const uint32_t qf_s = smem_u32(qf);
    const uint32_t lutK_s = smem_u32(lutK), lutV_s = smem_u32(lutV);
    const uint32_t laneK_s = lutK_s + 4 * lane, laneV_s = lutV_s + 4 * lane;

    const int split = blockIdx.x, h = blockIdx.y, sidx = blockIdx.z;
    const kvc_seq_desc sd = kvc_load_desc(seqs, sidx);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) mbar_init(&bar[k], 1);
    }
    if (MODE == 1 && threadIdx.x == 0) mbar_init(s_lbar, 1);
    fence_mbar_init();
    __syncthreads();
    if (MODE == 1) {
        if (threadIdx.x == 0) {
            mbar_expect_tx(s_lbar, 2u * (4u << KVC_LUT_BITS));
            tma_load_1d(lutK, sd.k_cb->fetch_lut, 4u << KVC_LUT_BITS, s_lbar);
            tma_load_1d(lutV, sd.v_cb->fetch_lut, 4u << KVC_LUT_BITS, s_lbar);
        }
    } else {
        build_lut<MODE>(lutK, sd.k_cb);
        build_lut<MODE>(lutV, sd.v_cb);
    }

    const int c_begin = split * chunks_per_split;
    const int c_end = min(sd.n_chunks, c_begin + chunks_per_split);
    const int first = c_begin + warp;
    const int n = first < c_end ? (c_end - first + NW - 1) / NW : 0;
    const long nbk = (long)sd.k_counters->n_blocks, nbv = (long)sd.v_counters->n_blocks;
    const uint64_t kcur = sd.k_counters->cursor, vcur = sd.v_counters->cursor;
    const float *qh = q + ((long)sidx * H + h) * D;
    float qreg[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) qreg[k] = qh[lane + 32 * k];
    const float sm_scale = kLog2e / sqrtf((float)D);
    const float inv_sqrt = 1.0f / sqrtf((float)D);

    auto issue = [&](bool is_v, int i) {
        if (lane == 0) {
            const long ord = (long)(first + NW * i) * H + h;
            const uint32_t *offs = is_v ? sd.v_offsets : sd.k_offsets;
            const long nb = is_v ? nbv : nbk;
            const uint64_t s0 = offs[ord];
            const uint64_t e0 = (ord + 1 < nb) ? (uint64_t)offs[ord + 1] : (is_v ? vcur : kcur);
            const uint64_t a = s0 & ~15ull;
            uint32_t bytes = (uint32_t)(((e0 + 15) & ~15ull) - a);
            const int cap = is_v ? stage_v : stage_k;
            if (bytes > (uint32_t)cap) {
                kvc_set_err(err, KVC_ERR_CODEC);
                bytes = 16;
            }
            uint64_t *b = &bar[(is_v ? 2 : 0) + (i & 1)];
            uint8_t *dst = my + (is_v ? 2 * stage_k + (i & 1) * stage_v : (i & 1) * stage_k);
            mbar_expect_tx(b, bytes);
            tma_load_1d(dst, (is_v ? sd.v_arena : sd.k_arena) + a, bytes, b);
        }
    };
    if (n > 0) {
        issue(false, 0);
        issue(true, 0);
    }
    if (n > 1) issue(false, 1);

    float m = -INFINITY, lsum = 0.f, wm = 0.f;
    float2 acc[D / 2];
#pragma unroll
    for (int c = 0; c < D / 2; ++c) acc[c] = make_float2(0.f, 0.f);
    float pwA = 0.f, pwB = 0.f;  // softmax weights of the previous chunk's tokens
    bool bad = false;
    if (MODE == 1) mbar_wait(s_lbar, 0);
    else __syncthreads();

    for (int i = 0; i <= n; ++i) {
        const bool hasK = i < n, hasV = i > 0;
        Cursor cur[4];  // kA, kB, vA, vB
        uint32_t cnt[4] = {0, 0, 0, 0};
        float base = 0.f;
        float2 aA2 = make_float2(0.f, 0.f), aB2 = aA2;
        if (hasK) {
            mbar_wait(&bar[i & 1], (i >> 1) & 1);
            const long ord = (long)(first + NW * i) * H + h;
            const uint32_t kofs = sd.k_offsets[ord] & 15u;
            const uint8_t *ks = my + (i & 1) * stage_k + kofs;
            cnt[0] = lds_u16(ks + 6 + 2 * lane);
            cnt[1] = lds_u16(ks + 6 + 2 * (lane + 32));
            const uint32_t iA = kvc_warp_incl_scan(cnt[0], lane);
            const uint32_t totA = __shfl_sync(0xffffffffu, iA, 31);
            const uint32_t iB = kvc_warp_incl_scan(cnt[1], lane);
            float basep = 0.f;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = lane + 32 * k;
                const float mn = lds_f32_a2(ks + 6 + 2 * BS + 8 * c);
                const float sc = lds_f32_a2(ks + 6 + 2 * BS + 8 * c + 4);
                qf[c] = sc * qreg[k];
                basep = fmaf(mn, qreg[k], basep);
            }
            base = kvc_warp_sum(basep);
            const uint32_t bit0 = (kofs + K_HDR) * 8;
            const uint32_t slot = kslot0 + (i & 1) * stage_k;
            cursor_init(cur[0], slot, bit0 + iA - cnt[0]);
            cursor_init(cur[1], slot, bit0 + totA + iB - cnt[1]);
        } else {
            cursor_init(cur[0], lutK_s, 0);
            cursor_init(cur[1], lutK_s, 0);
        }
        if (hasV) {
            const int j = i - 1;
            mbar_wait(&bar[2 + (j & 1)], (j >> 1) & 1);
            const long ord = (long)(first + NW * j) * H + h;
            const uint32_t vofs = sd.v_offsets[ord] & 15u;
            const uint8_t *vs = my + 2 * stage_k + (j & 1) * stage_v + vofs;
            cnt[2] = lds_u16(vs + 6 + 2 * lane);
            cnt[3] = lds_u16(vs + 6 + 2 * (lane + 32));
            const uint32_t iA = kvc_warp_incl_scan(cnt[2], lane);
            const uint32_t totA = __shfl_sync(0xffffffffu, iA, 31);
            const uint32_t iB = kvc_warp_incl_scan(cnt[3], lane);
            const float aA = pwA * lds_f32_a2(vs + 6 + 2 * BS + 8 * lane + 4);
            const float aB = pwB * lds_f32_a2(vs + 6 + 2 * BS + 8 * (lane + 32) + 4);
            wm = fmaf(pwA, lds_f32_a2(vs + 6 + 2 * BS + 8 * lane), wm);
            wm = fmaf(pwB, lds_f32_a2(vs + 6 + 2 * BS + 8 * (lane + 32)), wm);
            aA2 = make_float2(aA, aA);
            aB2 = make_float2(aB, aB);
            const uint32_t bit0 = (vofs + V_HDR) * 8;
            const uint32_t slot = vslot0 + (j & 1) * stage_v;
            cursor_init(cur[2], slot, bit0 + iA - cnt[2]);
            cursor_init(cur[3], slot, bit0 + totA + iB - cnt[3]);
        } else {
            cursor_init(cur[2], lutV_s, 0);
            cursor_init(cur[3], lutV_s, 0);
        }
        uint32_t p0[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) p0[k] = cur[k].p;
        __syncwarp();

        float2 sA2 = make_float2(0.f, 0.f), sB2 = sA2;
        if (MODE == 1) {
#pragma unroll
            for (int c2 = 0; c2 < D / 2; ++c2) {
                if (c2 % 2 == 0) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) cursor_reload(cur[k]);
                }
                uint32_t e[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    e[k] = lds32(lut_addr<1>(cur[k].win, k < 2 ? lutK_s : lutV_s, 0));
                    cur[k].win = __funnelshift_l(0u, cur[k].win, e[k]);
                    cur[k].p += e[k];
                }
                const float2 magic = make_float2(-8388608.f, -8388608.f);
                float2 f[4];
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    f[k] = __fadd2_rn(make_float2(sym_hi_byte(e[k], 0x7652),
                                                  sym_hi_byte(e[k], 0x7653)), magic);
                const float2 q2 = lds64f(qf_s + 8 * c2);
                sA2 = __ffma2_rn(f[0], q2, sA2);
                sB2 = __ffma2_rn(f[1], q2, sB2);
#ifdef KVC_EXPERIMENT_VREG
                acc[c2 % KVC_EXPERIMENT_VREG] = __ffma2_rn(f[2], aA2, acc[c2 % KVC_EXPERIMENT_VREG]);
                acc[c2 % KVC_EXPERIMENT_VREG] = __ffma2_rn(f[3], aB2, acc[c2 % KVC_EXPERIMENT_VREG]);
#else
                acc[c2] = __ffma2_rn(f[2], aA2, acc[c2]);
                acc[c2] = __ffma2_rn(f[3], aB2, acc[c2]);
#endif
            }
        } else {
            uint32_t e0[4];
#pragma unroll
            for (int s = 0; s < D; ++s) {
                if (s % W == 0) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) cursor_reload(cur[k]);
                }
                uint32_t e[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    e[k] = lds32(lut_addr<MODE>(cur[k].win, k < 2 ? lutK_s : lutV_s,
                                                k < 2 ? laneK_s : laneV_s));
                    cur[k].win = __funnelshift_l(0u, cur[k].win, e[k]);
                    cur[k].p += e[k];
                }
                if (s & 1) {
                    float2 f[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        f[k] = make_float2(__uint_as_float(e0[k] & ~15u),
                                           __uint_as_float(e[k] & ~15u));
                    const float2 q2 = lds64f(qf_s + 4 * (s - 1));
                    sA2 = __ffma2_rn(f[0], q2, sA2);
                    sB2 = __ffma2_rn(f[1], q2, sB2);
                    acc[s / 2] = __ffma2_rn(f[2], aA2, acc[s / 2]);
                    acc[s / 2] = __ffma2_rn(f[3], aB2, acc[s / 2]);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) e0[k] = e[k];
                }
            }
        }
        if (hasK)
            bad |= (((cur[0].p - p0[0]) & 0xFFFFu) != cnt[0]) |
                   (((cur[1].p - p0[1]) & 0xFFFFu) != cnt[1]);
        if (hasV)
            bad |= (((cur[2].p - p0[2]) & 0xFFFFu) != cnt[2]) |
                   (((cur[3].p - p0[3]) & 0xFFFFu) != cnt[3]);
        __syncwarp();
        if (hasK && i + 2 < n) issue(false, i + 2);
        if (i + 1 < n) issue(true, i + 1);

        if (hasK) {
            const int chunk = first + NW * i;
            float sA = sA2.x + sA2.y + base, sB = sB2.x + sB2.y + base;
            if (scores) {
                float *srow = scores + ((long)sidx * H + h) * ctx_stride + (long)chunk * BS;
                srow[lane] = sA * inv_sqrt;
                srow[lane + 32] = sB * inv_sqrt;
            }
            sA *= sm_scale;
            sB *= sm_scale;
            const float bm = kvc_warp_max(fmaxf(sA, sB));
            if (bm > m) {
                const float alpha = exp2f(m - bm);
                const float2 al2 = make_float2(alpha, alpha);
#pragma unroll
                for (int c = 0; c < D / 2; ++c) acc[c] = __fmul2_rn(acc[c], al2);
                lsum *= alpha;
                wm *= alpha;
                m = bm;
            }
            pwA = exp2f(sA - m);
            pwB = exp2f(sB - m);
            lsum += pwA + pwB;
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) kvc_set_err(err, KVC_ERR_CODEC);

    // ---- warp reduce, then CTA merge through shared memory --------------
    lsum = kvc_warp_sum(lsum);
    wm = kvc_warp_sum(wm);
    __syncthreads();  // all warps done with their stages: reuse as scratch
    Partial *wp = reinterpret_cast<Partial *>(wbase) + warp;
#pragma unroll
    for (int c = 0; c < D / 2; ++c) {
        const float vx = kvc_warp_sum(acc[c].x);
        const float vy = kvc_warp_sum(acc[c].y);
        if (lane == ((2 * c) & 31)) {
            wp->o[2 * c] = vx + wm;
            wp->o[2 * c + 1] = vy + wm;
        }
    }
    if (lane == 0) {
        wp->m = m;
        wp->l = lsum;
    }
    __syncthreads();
    if (warp == 0) {
        Partial *all = reinterpret_cast<Partial *>(wbase);
        float M = -INFINITY;
        for (int w = 0; w < NW; ++w) M = fmaxf(M, all[w].m);
        float L = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
        for (int w = 0; w < NW; ++w) {
            const float sc = (all[w].m == -INFINITY) ? 0.f : exp2f(all[w].m - M);
            L += all[w].l * sc;
#pragma unroll
            for (int k = 0; k < 4; ++k) o[k] += all[w].o[lane + 32 * k] * sc;
        }
        Partial *dst = partial + ((long)sidx * H + h) * n_splits + split;
#pragma unroll
        for (int k = 0; k < 4; ++k) dst->o[lane + 32 * k] = o[k];
        if (lane == 0) {
            dst->m = M;
            dst->l = L;
        }
    }
}

// 64-bit window cursor for the pair decoder: `hi` holds the next 32 stream
// bits, `lo` the following 32.  A reload (3 shared words) refills 64 valid
// bits, enough for 4 pair steps (<= 48 bits at max_len 6), so reloads cost
// 0.75 loads per pair step instead of 1.
struct Cursor2 {
    uint32_t hi, lo;
    uint32_t p;
    uint32_t base;
};
__device__ __forceinline__ void cursor2_init(Cursor2 &c, uint32_t stage_addr, uint32_t bit) {
    c.base = stage_addr + ((bit >> 5) << 2);
    c.p = bit & 31u;
    c.hi = c.lo = 0;
}
__device__ __forceinline__ void cursor2_reload(Cursor2 &c) {
    const uint32_t a = c.base + ((c.p >> 3) & 0x1FFCu);
    const uint32_t w0 = bswap32(lds32(a)), w1 = bswap32(lds32(a + 4)), w2 = bswap32(lds32(a + 8));
    c.hi = __funnelshift_l(w1, w0, c.p);
    c.lo = __funnelshift_l(w2, w1, c.p);
}
// single-symbol step on the lane-replicated 64-entry LUT (entry = float | len)
__device__ __forceinline__ uint32_t cursor2_sym(Cursor2 &c, uint32_t lane_s) {
    const uint32_t e = lds32(lane_s + ((c.hi >> 26) << 7));
    c.hi = __funnelshift_l(c.lo, c.hi, e);
    c.lo = __funnelshift_l(0u, c.lo, e);
    c.p += e;
    return e;
}
// single-symbol step on the 4096- / 8192-entry LUT (MODE 2 / 5: entry =
// float(sym) bits | len, codes <= 12 / 13 bits): 5 / 4 steps per 64-bit window
template <int BITS = 12>
__device__ __forceinline__ float cursor2_sym12(Cursor2 &c, uint32_t lut_s) {
    const uint32_t e = lds32(lut_s + ((c.hi >> (32 - BITS)) << 2));
    c.hi = __funnelshift_l(c.lo, c.hi, e);
    c.lo = __funnelshift_l(0u, c.lo, e);
    c.p += e;
    return __uint_as_float(e & ~15u);
}
// single-symbol step on a lane-copied LUT (MODE 6 / 7): lane_s = the lane's
// copy, entry i at lane_s + i * 4R
template <int BITS, int R>
__device__ __forceinline__ float cursor2_sym_copy(Cursor2 &c, uint32_t lane_s) {
    constexpr int kShift = 2 + (R == 32 ? 5 : (R == 16 ? 4 : (R == 8 ? 3 : 0)));
    const uint32_t e = lds32(lane_s + ((c.hi >> (32 - BITS)) << kShift));
    c.hi = __funnelshift_l(c.lo, c.hi, e);
    c.lo = __funnelshift_l(0u, c.lo, e);
    c.p += e;
    return __uint_as_float(e & ~15u);
}
__device__ __forceinline__ float2 cursor2_pair(Cursor2 &c, uint32_t lut_s) {
    const uint32_t e = lds32(lut_s + ((c.hi >> 20) << 2));
    c.hi = __funnelshift_l(c.lo, c.hi, e);
    c.lo = __funnelshift_l(0u, c.lo, e);
    c.p += e;
    return __fadd2_rn(make_float2(sym_hi_byte(e, 0x7652), sym_hi_byte(e, 0x7653)),
                      make_float2(-8388608.f, -8388608.f));
}

// Pair step on the bank-swizzled table (fetch_lut_x): byte address
// ((hi >> 18) ^ (hi >> 25)) & 0x3FFC = 4 * (i ^ ((i >> 7) & 31)) for the 12-bit
// window i, so the bank is window bits 7-11 XOR bits 0-4.  With short V pairs
// bits 7-11 belong to the next pair and cluster across lanes (4.4-way
// conflicts); the XOR spreads them (3.1-way, measured on config-2 streams).
__device__ __forceinline__ float2 cursor2_pair_x(Cursor2 &c, uint32_t lut_s) {
    const uint32_t e = lds32(lut_s + (((c.hi >> 18) ^ (c.hi >> 25)) & 0x3FFCu));
    c.hi = __funnelshift_l(c.lo, c.hi, e);
    c.lo = __funnelshift_l(0u, c.lo, e);
    c.p += e;
    return __fadd2_rn(make_float2(sym_hi_byte(e, 0x7652), sym_hi_byte(e, 0x7653)),
                      make_float2(-8388608.f, -8388608.f));
}

// Pair step with the low 5 index bits replaced by the lane id (MODE 3).  The
// last 5 bits of a 12-bit window are don't-care whenever the pair is <= 7
// bits long, so entry (idx & ~31) | lane equals entry idx and the lookup of
// every such lane lands in bank `lane`: conflict-free.  A pair of >= 8 bits
// (bit 3 of the consumed-bits field; the substituted entry shares the first
// 7 bits, so it is >= 8 bits too) is re-read at its true index, predicated,
// by the few lanes that need it.  At default V scales ~8% of pairs do, so a
// lookup costs ~2.0 wavefronts instead of ~3.5.
__device__ __forceinline__ uint32_t lut_pair_sub(uint32_t hi, uint32_t lut_s, uint32_t lane4) {
    const uint32_t x = hi >> 18;
    uint32_t e = lds32(lut_s + ((x & 0x3F80u) | lane4));
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p " KVC_LD_SHARED ".u32 %0, [%2];\n\t}"
                 : "+r"(e) : "r"(e & 8u), "r"(lut_s + (x & 0x3FFCu)));
    return e;
}
__device__ __forceinline__ float2 cursor2_pair_sub(Cursor2 &c, uint32_t lut_s, uint32_t lane4) {
    const uint32_t e = lut_pair_sub(c.hi, lut_s, lane4);
    c.hi = __funnelshift_l(c.lo, c.hi, e);
    c.lo = __funnelshift_l(0u, c.lo, e);
    c.p += e;
    return __fadd2_rn(make_float2(sym_hi_byte(e, 0x7652), sym_hi_byte(e, 0x7653)),
                      make_float2(-8388608.f, -8388608.f));
}
__device__ __forceinline__ float4 lds128f(uint32_t addr) {
    float4 v;
    asm volatile(KVC_LD_SHARED ".v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

// Decode the 128 symbols of two slices (cursors c[0], c[1]) in lockstep and
// hand each channel pair to sink(c2, f[slice0], f[slice1]).  Fully unrolled so
// the sink can index register arrays with c2.
template <int MODE, bool FULL, typename Sink>
__device__ __forceinline__ void decode_two(Cursor *c, uint32_t lut_s, uint32_t lane_s, Sink sink) {
    const float2 magic = make_float2(-8388608.f, -8388608.f);
    if (MODE == 1) {
#pragma unroll(FULL ? 64 : 8)
        for (int c2 = 0; c2 < D / 2; ++c2) {
            if (c2 % 2 == 0) {
                cursor_reload(c[0]);
                cursor_reload(c[1]);
            }
            float2 f[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const uint32_t e = lds32(lut_addr<1>(c[k].win, lut_s, 0));
                c[k].win = __funnelshift_l(0u, c[k].win, e);
                c[k].p += e;
                f[k] = __fadd2_rn(make_float2(sym_hi_byte(e, 0x7652), sym_hi_byte(e, 0x7653)), magic);
            }
            sink(c2, f[0], f[1]);
        }
    } else {
        constexpr int W = Dec<MODE>::kSymsPerWin;
        uint32_t e0[2];
#pragma unroll(FULL ? 128 : 16)
        for (int sy = 0; sy < D; ++sy) {
            if (sy % W == 0) {
                cursor_reload(c[0]);
                cursor_reload(c[1]);
            }
            uint32_t e[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                e[k] = lds32(lut_addr<MODE>(c[k].win, lut_s, lane_s));
                c[k].win = __funnelshift_l(0u, c[k].win, e[k]);
                c[k].p += e[k];
            }
            if (sy & 1) {
                sink(sy / 2, make_float2(__uint_as_float(e0[0] & ~15u), __uint_as_float(e[0] & ~15u)),
                     make_float2(__uint_as_float(e0[1] & ~15u), __uint_as_float(e[1] & ~15u)));
            } else {
                e0[0] = e[0];
                e0[1] = e[1];
            }
        }
    }
}

// Sum 128 floats (acc[64] float2, channel 2c + {0,1}) over the 32 lanes with a
// halving reduce-scatter: at step k (xor 16, 8, .., 1) a lane keeps the half of
// its live values selected by lane bit 4-k and adds the partner's copy of it.
// Lane l ends with channels 4l .. 4l+3 in r[0], r[1].
__device__ __forceinline__ void reduce_scatter_128(float2 (&acc)[D / 2], uint32_t lane, float2 (&r)[2]) {
    float2 v[32];
    {
        const bool hi = (lane >> 4) & 1;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const float2 keep = hi ? acc[32 + i] : acc[i], send = hi ? acc[i] : acc[32 + i];
            v[i] = make_float2(keep.x + __shfl_xor_sync(0xffffffffu, send.x, 16),
                               keep.y + __shfl_xor_sync(0xffffffffu, send.y, 16));
        }
    }
#pragma unroll
    for (int o = 8, n = 16; o >= 1; o >>= 1, n >>= 1) {
        const bool hi = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (i < n) {
                const float2 keep = hi ? v[n + i] : v[i], send = hi ? v[i] : v[n + i];
                v[i] = make_float2(keep.x + __shfl_xor_sync(0xffffffffu, send.x, o),
                                   keep.y + __shfl_xor_sync(0xffffffffu, send.y, o));
            }
        }
    }
    r[0] = v[0];
    r[1] = v[1];
}

// ---------------------------------------------------------------------------
// Warp-specialized fused fetch-attention (default).  CTA = 2 warpgroups:
// warps 0-3 decode K, warps 4-7 decode V; K warp w and V warp w+4 form a pair
// that walks chunks first+4j of this CTA's context split.  Per pair: a K TMA
// ring (2 slots), a V TMA ring (2 slots) and a 2-slot score ring; the K warp
// publishes each chunk's 64 log2-scaled scores through mbarriers (sfull /
// sempty), the V warp runs the online softmax and the weighted V decode.
// setmaxnreg moves registers from the K warpgroup (2 cursors, no arrays) to
// the V warpgroup (128 f32 accumulators per lane), which lets 2 CTAs = 16
// warps share an SM; every warp runs two independent decode chains.
// ---------------------------------------------------------------------------
// Context split plan of a fused launch: split s covers chunks [begin[s],
// begin[s+1]) of every (seq, head).  Splits need not be equal: the host plans
// a few large splits followed by small tail splits so the last wave of CTAs
// is short (pick_split_plan).  The grid is 1D and split-major, so every
// (seq, head)'s large splits launch before any tail split.
constexpr int kMaxPlan = 48;
struct SplitPlan {
    int n;
    int begin[kMaxPlan + 1];
};
__device__ __forceinline__ void plan_decode(const SplitPlan &plan, int H, int &split, int &h,
                                            int &sidx) {
    const int units = gridDim.x / plan.n;  // n_seqs * H
    split = blockIdx.x / units;
    const int r = blockIdx.x - split * units;
    sidx = r / H;
    h = r - sidx * H;
}

constexpr int WS_PAIRS = 4;
constexpr int kThreadsWS = 2 * WS_PAIRS * 32;
constexpr int kRegK = 80, kRegV = 176;  // (80 + 176) * 128 threads = 32768 regs per CTA

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int MODE, int VMODE>
__global__ void __launch_bounds__(kThreadsWS, 2)
fused_attn_ws_kernel(const kvc_seq_desc *__restrict__ seqs, int H, const float *__restrict__ q,
                     float *__restrict__ scores, long ctx_stride, Partial *__restrict__ partial,
                     const SplitPlan plan, int stage_k, int stage_v, int *err) {
    // the 13-bit LUTs (MODE 5, 2 x 32 KB) exceed the static shared-memory
    // limit: they live in the dynamic region, after the pairs' staging
    // (and MODE 6's lane-private tables, 2 x 32 KB)
    constexpr bool kDynK = Dec<MODE>::kDyn, kDynV = Dec<VMODE>::kDyn;
    __shared__ __align__(128) uint32_t s_lutK_st[kDynK ? 1 : Dec<MODE>::kLutWords];
    __shared__ __align__(128) uint32_t s_lutV_st[kDynV ? 1 : Dec<VMODE>::kLutWords];
    __shared__ uint64_t s_lbar[1];
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const bool is_v = warp >= WS_PAIRS;
    const int pair = warp & (WS_PAIRS - 1);
    const int per_pair = 2 * (stage_k + stage_v) + 1024 + 64;
    uint32_t *s_lutK = kDynK ? reinterpret_cast<uint32_t *>(smem + WS_PAIRS * per_pair) : s_lutK_st;
    uint32_t *s_lutV = kDynV ? reinterpret_cast<uint32_t *>(smem + WS_PAIRS * per_pair) +
                                   (kDynK ? 8192 : 0)
                             : s_lutV_st;
    uint8_t *pb = smem + pair * per_pair;
    uint8_t *kring = pb, *vring = pb + 2 * stage_k;
    float *qf = reinterpret_cast<float *>(pb + 2 * (stage_k + stage_v));
    float *sring = qf + D;  // [2][64]
    uint64_t *bar = reinterpret_cast<uint64_t *>(pb + 2 * (stage_k + stage_v) + 1024);
    uint64_t *kfull = bar, *vfull = bar + 2, *sfull = bar + 4, *sempty = bar + 6;

    const int n_splits = plan.n;
    int split, h, sidx;
    plan_decode(plan, H, split, h, sidx);
    const kvc_seq_desc sd = kvc_load_desc(seqs, sidx);
    if (!is_v && lane == 0) {
        mbar_init(&kfull[0], 1);
        mbar_init(&kfull[1], 1);
        mbar_init(&vfull[0], 1);
        mbar_init(&vfull[1], 1);
        mbar_init(&sfull[0], 32);
        mbar_init(&sfull[1], 32);
        mbar_init(&sempty[0], 32);
        mbar_init(&sempty[1], 32);
    }
    // pair LUTs and the 13-bit LUTs come by TMA from the codebook tables
    constexpr bool kPK = Dec<MODE>::kPair || MODE == 5, kPV = Dec<VMODE>::kPair || VMODE == 5;
    constexpr bool kTma = kPK || kPV;
    if (kTma && threadIdx.x == 0) mbar_init(s_lbar, 1);
    fence_mbar_init();
    __syncthreads();
    if (kTma && threadIdx.x == 0) {
        mbar_expect_tx(s_lbar, (kPK ? 4u * Dec<MODE>::kLutWords : 0u) +
                                   (kPV ? 4u * Dec<VMODE>::kLutWords : 0u));
        if (kPK)
            tma_load_1d(s_lutK, MODE == 5 ? sd.k_cb->lut13 : sd.k_cb->fetch_lut,
                        4u * Dec<MODE>::kLutWords, s_lbar);
        if (kPV)
            tma_load_1d(s_lutV, VMODE == 5 ? sd.v_cb->lut13 : (VMODE == 1 ? sd.v_cb->fetch_lut_x : sd.v_cb->fetch_lut),
                        4u * Dec<VMODE>::kLutWords, s_lbar);
    }
    if (MODE == 6) build_lut_copies<9, 16>(s_lutK, sd.k_cb);
    else if (MODE == 7) build_lut_copies<8, 32>(s_lutK, sd.k_cb);
    else if (MODE == 8) build_lut_copies<10, 8>(s_lutK, sd.k_cb);
    else if (!kPK) build_lut<MODE>(s_lutK, sd.k_cb);
    if (VMODE == 6) build_lut_copies<9, 16>(s_lutV, sd.v_cb);
    else if (VMODE == 7) build_lut_copies<8, 32>(s_lutV, sd.v_cb);
    else if (VMODE == 8) build_lut_copies<10, 8>(s_lutV, sd.v_cb);
    else if (!kPV) build_lut<VMODE>(s_lutV, sd.v_cb);
    if (!kPK || !kPV) __syncthreads();

    const int c_begin = plan.begin[split];
    const int c_end = min(sd.n_chunks, plan.begin[split + 1]);
    const int first = c_begin + pair;
    const int n = first < c_end ? (c_end - first + WS_PAIRS - 1) / WS_PAIRS : 0;
    const float sm_scale = kLog2e / sqrtf((float)D);
    const float inv_sqrt = 1.0f / sqrtf((float)D);

    // TMA of chunk j's K or V extent into ring slot j&1 (lane 0 only).  The
    // arena counters do not change during the launch: read them once.
    const long nb_k = (long)sd.k_counters->n_blocks, nb_v = (long)sd.v_counters->n_blocks;
    const uint64_t cur_k = sd.k_counters->cursor, cur_v = sd.v_counters->cursor;
    auto issue = [&](bool v, int j) {
        const long ord = (long)(first + WS_PAIRS * j) * H + h;
        const uint32_t *offs = v ? sd.v_offsets : sd.k_offsets;
        const long nb = v ? nb_v : nb_k;
        const uint64_t s0 = offs[ord];
        const uint64_t e0 = (ord + 1 < nb) ? (uint64_t)offs[ord + 1] : (v ? cur_v : cur_k);
        const uint64_t a = s0 & ~15ull;
        uint32_t bytes = (uint32_t)(((e0 + 15) & ~15ull) - a);
        const int cap = v ? stage_v : stage_k;
        if (bytes > (uint32_t)cap) {
            kvc_set_err(err, KVC_ERR_CODEC);
            bytes = 16;
        }
        uint64_t *b = v ? &vfull[j & 1] : &kfull[j & 1];
        uint8_t *dst = v ? vring + (j & 1) * stage_v : kring + (j & 1) * stage_k;
        mbar_expect_tx(b, bytes);
        tma_load_1d(dst, (v ? sd.v_arena : sd.k_arena) + a, bytes, b);
    };
    bool bad = false;

    if (!is_v) {
        // =================== K warp: scores producer ===================
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegK));
        if (lane == 0) {
            if (n > 0) issue(false, 0);
            if (n > 1) issue(false, 1);
        }
        const float *qh = q + ((long)sidx * H + h) * D;
        float qreg[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) qreg[k] = qh[lane + 32 * k];
        const uint32_t qf_s = smem_u32(qf);
        const uint32_t lut_s = smem_u32(s_lutK);
        const uint32_t lane_s = lut_s + 4 * lane;
        if (kTma) mbar_wait(s_lbar, 0);
        // block start & 15 of the next chunk, loaded one chunk ahead
        uint32_t kofs_next = n > 0 ? sd.k_offsets[(long)first * H + h] & 15u : 0u;
        for (int j = 0; j < n; ++j) {
            const int u = j >> 1, sl = j & 1;
            const uint32_t kofs = kofs_next;
            if (j + 1 < n) kofs_next = sd.k_offsets[(long)(first + WS_PAIRS * (j + 1)) * H + h] & 15u;
            mbar_wait(&kfull[sl], u & 1);
            const uint8_t *ks = kring + sl * stage_k + kofs;
            const uint32_t cA = lds_u16(ks + 6 + 2 * lane), cB = lds_u16(ks + 6 + 2 * (lane + 32));
            const uint32_t iA = kvc_warp_incl_scan(cA, lane);
            const uint32_t totA = __shfl_sync(0xffffffffu, iA, 31);
            const uint32_t iB = kvc_warp_incl_scan(cB, lane);
            float basep = 0.f;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = lane + 32 * k;
                qf[c] = lds_f32_a2(ks + 6 + 2 * BS + 8 * c + 4) * qreg[k];
                basep = fmaf(lds_f32_a2(ks + 6 + 2 * BS + 8 * c), qreg[k], basep);
            }
            const float base = kvc_warp_sum(basep);
            __syncwarp();
            const uint32_t bit0 = (kofs + K_HDR) * 8, slot = smem_u32(kring + sl * stage_k);
            Cursor cur[2];
            cursor_init(cur[0], slot, bit0 + iA - cA);
            cursor_init(cur[1], slot, bit0 + totA + iB - cB);
            const uint32_t p0A = cur[0].p, p0B = cur[1].p;
            float2 sA2 = make_float2(0.f, 0.f), sB2 = sA2;
            if (Dec<MODE>::kPair) {
                // 64-bit windows, one reload per 5 pair steps (<= 60 bits at
                // max_len 6).
                Cursor2 c2c[2];
                cursor2_init(c2c[0], slot, bit0 + iA - cA);
                cursor2_init(c2c[1], slot, bit0 + totA + iB - cB);
                // q' for two pair steps per LDS.128 (broadcast): groups of 10
                // steps = 2 reloads + 5 q loads; 6 groups + a tail of 4.
                auto steps = [&](int c2base, auto np) {
                    float4 q4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int t = 0; t < decltype(np)::value; ++t) {
                        if (t % 5 == 0) {
                            cursor2_reload(c2c[0]);
                            cursor2_reload(c2c[1]);
                        }
                        if (t % 2 == 0) q4 = lds128f(qf_s + 8 * (c2base + t));
                        const float2 q2 = (t % 2 == 0) ? make_float2(q4.x, q4.y) : make_float2(q4.z, q4.w);
                        if (MODE == 3) {
                            sA2 = __ffma2_rn(cursor2_pair_sub(c2c[0], lut_s, 4 * lane), q2, sA2);
                            sB2 = __ffma2_rn(cursor2_pair_sub(c2c[1], lut_s, 4 * lane), q2, sB2);
                        } else {
                            sA2 = __ffma2_rn(cursor2_pair(c2c[0], lut_s), q2, sA2);
                            sB2 = __ffma2_rn(cursor2_pair(c2c[1], lut_s), q2, sB2);
                        }
                    }
                };
#pragma unroll 1
                for (int g = 0; g < 6; ++g) steps(10 * g, std::integral_constant<int, 10>());
                steps(60, std::integral_constant<int, 4>());
                cur[0].p = c2c[0].p;
                cur[1].p = c2c[1].p;
            } else if (MODE == 2 || MODE == 5) {
                // codes <= 12 (13) bits: single-symbol lookups on 64-bit windows, one
                // reload per 5 (4) symbols (was a 32-bit window reloaded every 2)
                constexpr int R = Dec<MODE>::kReload, SB = Dec<MODE>::kSymBits;
                Cursor2 c2c[2];
                cursor2_init(c2c[0], slot, bit0 + iA - cA);
                cursor2_init(c2c[1], slot, bit0 + totA + iB - cB);
                auto grp = [&](int c2base, auto np) {
                    float fa = 0.f, fb = 0.f;
#pragma unroll
                    for (int t = 0; t < 2 * decltype(np)::value; ++t) {
                        if (t % R == 0) {
                            cursor2_reload(c2c[0]);
                            cursor2_reload(c2c[1]);
                        }
                        const float xa = cursor2_sym12<SB>(c2c[0], lut_s);
                        const float xb = cursor2_sym12<SB>(c2c[1], lut_s);
                        if (t & 1) {
                            const float2 q2 = lds64f(qf_s + 8 * (c2base + t / 2));
                            sA2 = __ffma2_rn(make_float2(fa, xa), q2, sA2);
                            sB2 = __ffma2_rn(make_float2(fb, xb), q2, sB2);
                        } else {
                            fa = xa;
                            fb = xb;
                        }
                    }
                };
                if (R == 5) {  // groups of 10 symbols (2 reloads), a tail of 8
#pragma unroll 1
                    for (int g = 0; g < 12; ++g) grp(5 * g, std::integral_constant<int, 5>());
                    grp(60, std::integral_constant<int, 4>());
                } else {       // groups of 8 symbols (2 reloads)
#pragma unroll 1
                    for (int g = 0; g < 16; ++g) grp(4 * g, std::integral_constant<int, 4>());
                }
                cur[0].p = c2c[0].p;
                cur[1].p = c2c[1].p;
            } else if (MODE == 6 || MODE == 7 || MODE == 8) {
                // codes <= 9 (8) bits: lane-copied LUT, one reload per 7 (8)
                // symbols; groups of 2R symbols (2 reloads), R = 7: a tail of 2
                constexpr int R = Dec<MODE>::kReload, SB = Dec<MODE>::kSymBits,
                              CP = Dec<MODE>::kCopies;
                const uint32_t copy_s = lut_s + 4 * (lane & (CP - 1));
                Cursor2 c2c[2];
                cursor2_init(c2c[0], slot, bit0 + iA - cA);
                cursor2_init(c2c[1], slot, bit0 + totA + iB - cB);
                auto grp = [&](int c2base, auto np) {
                    float fa = 0.f, fb = 0.f;
#pragma unroll
                    for (int t = 0; t < 2 * decltype(np)::value; ++t) {
                        if (t % R == 0) {
                            cursor2_reload(c2c[0]);
                            cursor2_reload(c2c[1]);
                        }
                        const float xa = cursor2_sym_copy<SB, CP>(c2c[0], copy_s);
                        const float xb = cursor2_sym_copy<SB, CP>(c2c[1], copy_s);
                        if (t & 1) {
                            const float2 q2 = lds64f(qf_s + 8 * (c2base + t / 2));
                            sA2 = __ffma2_rn(make_float2(fa, xa), q2, sA2);
                            sB2 = __ffma2_rn(make_float2(fb, xb), q2, sB2);
                        } else {
                            fa = xa;
                            fb = xb;
                        }
                    }
                };
                constexpr int NG = D / (2 * R), TAIL = D - NG * 2 * R;
#pragma unroll 1
                for (int g = 0; g < NG; ++g) grp(R * g, std::integral_constant<int, R>());
                if (TAIL) grp(R * NG, std::integral_constant<int, (TAIL > 0 ? TAIL / 2 : 1)>());
                cur[0].p = c2c[0].p;
                cur[1].p = c2c[1].p;
            } else {
                decode_two<MODE, false>(cur, lut_s, lane_s, [&](int c2, float2 fA, float2 fB) {
                    const float2 q2 = lds64f(qf_s + 8 * c2);
                    sA2 = __ffma2_rn(fA, q2, sA2);
                    sB2 = __ffma2_rn(fB, q2, sB2);
                });
            }
            bad |= (((cur[0].p - p0A) & 0xFFFFu) != cA) | (((cur[1].p - p0B) & 0xFFFFu) != cB);
            const float sA = sA2.x + sA2.y + base, sB = sB2.x + sB2.y + base;
            if (scores) {
                float *srow = scores + ((long)sidx * H + h) * ctx_stride +
                              (long)(first + WS_PAIRS * j) * BS;
                srow[lane] = sA * inv_sqrt;
                srow[lane + 32] = sB * inv_sqrt;
            }
            mbar_wait(&sempty[sl], (u & 1) ^ 1);
            sring[sl * 64 + lane] = sA * sm_scale;
            sring[sl * 64 + lane + 32] = sB * sm_scale;
            mbar_arrive(&sfull[sl]);
            __syncwarp();
            if (lane == 0 && j + 2 < n) issue(false, j + 2);
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) kvc_set_err(err, KVC_ERR_CODEC);
        __syncthreads();
        __syncthreads();
        return;
    }

    // =================== V warp: softmax + weighted V ===================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegV));
    if (lane == 0) {
        if (n > 0) issue(true, 0);
        if (n > 1) issue(true, 1);
    }
    float m = -INFINITY, lsum = 0.f, wm = 0.f;
    float2 acc[D / 2];
#pragma unroll
    for (int c = 0; c < D / 2; ++c) acc[c] = make_float2(0.f, 0.f);
    const uint32_t lut_s = smem_u32(s_lutV);
    const uint32_t lane_s = lut_s + 4 * lane;
    if (kTma) mbar_wait(s_lbar, 0);
    uint32_t vofs_next = n > 0 ? sd.v_offsets[(long)first * H + h] & 15u : 0u;
    for (int j = 0; j < n; ++j) {
        const int u = j >> 1, sl = j & 1;
        const uint32_t vofs_cur = vofs_next;
        if (j + 1 < n) vofs_next = sd.v_offsets[(long)(first + WS_PAIRS * (j + 1)) * H + h] & 15u;
        mbar_wait(&sfull[sl], u & 1);
        const float sA = sring[sl * 64 + lane], sB = sring[sl * 64 + lane + 32];
        mbar_arrive(&sempty[sl]);
        const float bm = kvc_warp_max(fmaxf(sA, sB));
        if (bm > m) {
            const float alpha = exp2f(m - bm);
            const float2 al2 = make_float2(alpha, alpha);
#pragma unroll
            for (int c = 0; c < D / 2; ++c) acc[c] = __fmul2_rn(acc[c], al2);
            lsum *= alpha;
            wm *= alpha;
            m = bm;
        }
        const float pA = exp2f(sA - m), pB = exp2f(sB - m);
        lsum += pA + pB;
        mbar_wait(&vfull[sl], u & 1);
        const uint32_t vofs = vofs_cur;
        const uint8_t *vs = vring + sl * stage_v + vofs;
        const uint32_t cA = lds_u16(vs + 6 + 2 * lane), cB = lds_u16(vs + 6 + 2 * (lane + 32));
        const uint32_t iA = kvc_warp_incl_scan(cA, lane);
        const uint32_t totA = __shfl_sync(0xffffffffu, iA, 31);
        const uint32_t iB = kvc_warp_incl_scan(cB, lane);
        const float aA = pA * lds_f32_a2(vs + 6 + 2 * BS + 8 * lane + 4);
        const float aB = pB * lds_f32_a2(vs + 6 + 2 * BS + 8 * (lane + 32) + 4);
        wm = fmaf(pA, lds_f32_a2(vs + 6 + 2 * BS + 8 * lane), wm);
        wm = fmaf(pB, lds_f32_a2(vs + 6 + 2 * BS + 8 * (lane + 32)), wm);
        const float2 aA2 = make_float2(aA, aA), aB2 = make_float2(aB, aB);
        const uint32_t bit0 = (vofs + V_HDR) * 8, slot = smem_u32(vring + sl * stage_v);
        Cursor cur[2];
        cursor_init(cur[0], slot, bit0 + iA - cA);
        cursor_init(cur[1], slot, bit0 + totA + iB - cB);
        const uint32_t p0A = cur[0].p, p0B = cur[1].p;
        if (VMODE == 1 || VMODE == 0 || VMODE == 3 || VMODE == 4) {
            // 64-bit windows; 5 pair steps (<= 60 bits at max_len 6) per reload
            Cursor2 c2c[2];
            cursor2_init(c2c[0], slot, bit0 + iA - cA);
            cursor2_init(c2c[1], slot, bit0 + totA + iB - cB);
#pragma unroll
            for (int c2 = 0; c2 < D / 2; ++c2) {
                if (c2 % 5 == 0) {
                    cursor2_reload(c2c[0]);
                    cursor2_reload(c2c[1]);
                }
                if (VMODE == 1) {  // bank-swizzled pair table (fetch_lut_x)
                    acc[c2] = __ffma2_rn(cursor2_pair_x(c2c[0], lut_s), aA2, acc[c2]);
                    acc[c2] = __ffma2_rn(cursor2_pair_x(c2c[1], lut_s), aB2, acc[c2]);
                } else if (VMODE == 4) {  // plain pair table
                    acc[c2] = __ffma2_rn(cursor2_pair(c2c[0], lut_s), aA2, acc[c2]);
                    acc[c2] = __ffma2_rn(cursor2_pair(c2c[1], lut_s), aB2, acc[c2]);
                } else if (VMODE == 3) {
                    acc[c2] = __ffma2_rn(cursor2_pair_sub(c2c[0], lut_s, 4 * lane), aA2, acc[c2]);
                    acc[c2] = __ffma2_rn(cursor2_pair_sub(c2c[1], lut_s, 4 * lane), aB2, acc[c2]);
                } else {
                    const uint32_t a0 = cursor2_sym(c2c[0], lane_s), b0 = cursor2_sym(c2c[1], lane_s);
                    const uint32_t a1 = cursor2_sym(c2c[0], lane_s), b1 = cursor2_sym(c2c[1], lane_s);
                    acc[c2] = __ffma2_rn(make_float2(__uint_as_float(a0 & ~15u), __uint_as_float(a1 & ~15u)),
                                         aA2, acc[c2]);
                    acc[c2] = __ffma2_rn(make_float2(__uint_as_float(b0 & ~15u), __uint_as_float(b1 & ~15u)),
                                         aB2, acc[c2]);
                }
            }
            cur[0].p = c2c[0].p;
            cur[1].p = c2c[1].p;
        } else if (VMODE == 2 || VMODE == 5) {
            // codes <= 12 (13) bits: single-symbol lookups, 64-bit windows, a
            // reload per 5 (4) symbols
            constexpr int R = Dec<VMODE>::kReload, SB = Dec<VMODE>::kSymBits;
            Cursor2 c2c[2];
            cursor2_init(c2c[0], slot, bit0 + iA - cA);
            cursor2_init(c2c[1], slot, bit0 + totA + iB - cB);
            float fa = 0.f, fb = 0.f;
#pragma unroll
            for (int t = 0; t < D; ++t) {
                if (t % R == 0) {
                    cursor2_reload(c2c[0]);
                    cursor2_reload(c2c[1]);
                }
                const float xa = cursor2_sym12<SB>(c2c[0], lut_s);
                const float xb = cursor2_sym12<SB>(c2c[1], lut_s);
                if (t & 1) {
                    acc[t / 2] = __ffma2_rn(make_float2(fa, xa), aA2, acc[t / 2]);
                    acc[t / 2] = __ffma2_rn(make_float2(fb, xb), aB2, acc[t / 2]);
                } else {
                    fa = xa;
                    fb = xb;
                }
            }
            cur[0].p = c2c[0].p;
            cur[1].p = c2c[1].p;
        } else if (VMODE == 6 || VMODE == 7 || VMODE == 8) {
            // codes <= 9 (8) bits: lane-copied LUT, a reload per 7 (8) symbols
            constexpr int R = Dec<VMODE>::kReload, SB = Dec<VMODE>::kSymBits,
                          CP = Dec<VMODE>::kCopies;
            const uint32_t copy_s = lut_s + 4 * (lane & (CP - 1));
            Cursor2 c2c[2];
            cursor2_init(c2c[0], slot, bit0 + iA - cA);
            cursor2_init(c2c[1], slot, bit0 + totA + iB - cB);
            float fa = 0.f, fb = 0.f;
#pragma unroll
            for (int t = 0; t < D; ++t) {
                if (t % R == 0) {
                    cursor2_reload(c2c[0]);
                    cursor2_reload(c2c[1]);
                }
                const float xa = cursor2_sym_copy<SB, CP>(c2c[0], copy_s);
                const float xb = cursor2_sym_copy<SB, CP>(c2c[1], copy_s);
                if (t & 1) {
                    acc[t / 2] = __ffma2_rn(make_float2(fa, xa), aA2, acc[t / 2]);
                    acc[t / 2] = __ffma2_rn(make_float2(fb, xb), aB2, acc[t / 2]);
                } else {
                    fa = xa;
                    fb = xb;
                }
            }
            cur[0].p = c2c[0].p;
            cur[1].p = c2c[1].p;
        } else {
            decode_two<VMODE, true>(cur, lut_s, lane_s, [&](int c2, float2 fA, float2 fB) {
                acc[c2] = __ffma2_rn(fA, aA2, acc[c2]);
                acc[c2] = __ffma2_rn(fB, aB2, acc[c2]);
            });
        }
        bad |= (((cur[0].p - p0A) & 0xFFFFu) != cA) | (((cur[1].p - p0B) & 0xFFFFu) != cB);
        __syncwarp();
        if (lane == 0 && j + 2 < n) issue(true, j + 2);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) kvc_set_err(err, KVC_ERR_CODEC);
    lsum = kvc_warp_sum(lsum);
    wm = kvc_warp_sum(wm);
    __syncthreads();  // K warps are done: their rings are free scratch
    Partial *wp = reinterpret_cast<Partial *>(smem + pair * per_pair);
    {
        // reduce-scatter of the 128 channel sums over the warp: 5 halving steps
        // (124 shuffles instead of 640); lane l ends with channels 4l..4l+3
        float2 r[2];
        reduce_scatter_128(acc, lane, r);
        reinterpret_cast<float2 *>(wp->o)[2 * lane] = make_float2(r[0].x + wm, r[0].y + wm);
        reinterpret_cast<float2 *>(wp->o)[2 * lane + 1] = make_float2(r[1].x + wm, r[1].y + wm);
    }
    if (lane == 0) {
        wp->m = m;
        wp->l = lsum;
    }
    __syncthreads();
    if (pair == 0) {
        float M = -INFINITY;
        for (int w = 0; w < WS_PAIRS; ++w)
            M = fmaxf(M, reinterpret_cast<const Partial *>(smem + w * per_pair)->m);
        float L = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
        for (int w = 0; w < WS_PAIRS; ++w) {
            const Partial *pw = reinterpret_cast<const Partial *>(smem + w * per_pair);
            const float sc = (pw->m == -INFINITY) ? 0.f : exp2f(pw->m - M);
            L += pw->l * sc;
#pragma unroll
            for (int k = 0; k < 4; ++k) o[k] += pw->o[lane + 32 * k] * sc;
        }
        Partial *dst = partial + ((long)sidx * H + h) * n_splits + split;
#pragma unroll
        for (int k = 0; k < 4; ++k) dst->o[lane + 32 * k] = o[k];
        if (lane == 0) {
            dst->m = M;
            dst->l = L;
        }
    }
}

// G consecutive f32 from shared memory in one vector load (G = 2 or 4)
template <int G>
__device__ __forceinline__ void lds_vec(uint32_t addr, float *v) {
    if (G == 4) {
        asm volatile(KVC_LD_SHARED ".v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(addr));
    } else {
        asm volatile(KVC_LD_SHARED ".v2.f32 {%0, %1}, [%2];" : "=f"(v[0]), "=f"(v[1]) : "r"(addr));
    }
}

// ---------------------------------------------------------------------------
// Decode-once GQA fused fetch: G query heads share each KV head (Llama-3
// layout: query head h*G+g reads KV head h).  K warps decode each K slice
// once and accumulate G dot products per token (q' for every group member
// in shared memory); V warps decode each V slice once into a bank-swizzled
// u8 code tile (row stride 132 B, one STS.U16 per decoded pair) and then run a
// per-channel GEMV over the 64 tokens for all G weight vectors, lanes owning
// 4 channels each.  Same TMA rings / score ring / split partials as the G=1
// kernel; partial index = (seq * H*G + h*G + g) * n_splits + split.
// ---------------------------------------------------------------------------
// V code half-tile: 64 tokens x 64 channels, row stride 68 B (17 words, odd,
// so the 32 lanes' row stores land in 32 distinct banks)
constexpr int kTileRow = 68;
__host__ __device__ constexpr int gqa_per_pair(int stage_k, int stage_v, int G, int vslots) {
    return 2 * stage_k + vslots * stage_v + 4 * (G * D + 2 * G * BS + G * BS + 4) + BS * kTileRow + 64;
}

template <int G, int NP, int VS>
__global__ void __launch_bounds__(NP * 64, 1)
fused_attn_gqa_kernel(const kvc_seq_desc *__restrict__ seqs, int H, const float *__restrict__ q,
                      Partial *__restrict__ partial, const SplitPlan plan,
                      int stage_k, int stage_v, int *err) {
    __shared__ __align__(128) uint32_t s_lutK[1 << KVC_LUT_BITS];
    __shared__ __align__(128) uint32_t s_lutV[1 << KVC_LUT_BITS];
    __shared__ uint64_t s_lbar[1];
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const bool is_v = warp >= NP;
    const int pair = is_v ? warp - NP : warp;
    const int per_pair = gqa_per_pair(stage_k, stage_v, G, VS);
    uint8_t *pb = smem + pair * per_pair;
    uint8_t *kring = pb, *vring = pb + 2 * stage_k;
    float *qf = reinterpret_cast<float *>(pb + 2 * stage_k + VS * stage_v);  // [128][G]
    float *sring = qf + G * D;                                            // [2][G][64]
    float *sa = sring + 2 * G * BS;                                       // [64][G]
    uint8_t *tile = reinterpret_cast<uint8_t *>(sa + G * BS + 4);        // [64][68]
    // sa: weights [64][G], tokens 32..63 shifted by G floats so the two half-warps'
    // broadcast loads in the GEMV land in different banks
    uint64_t *bar = reinterpret_cast<uint64_t *>(tile + BS * kTileRow);
    uint64_t *kfull = bar, *vfull = bar + 2, *sfull = bar + 4, *sempty = bar + 6;

    const int n_splits = plan.n;
    int split, h, sidx;
    plan_decode(plan, H, split, h, sidx);
    const kvc_seq_desc sd = kvc_load_desc(seqs, sidx);
    if (!is_v && lane == 0) {
        mbar_init(&kfull[0], 1);
        mbar_init(&kfull[1], 1);
        mbar_init(&vfull[0], 1);
        mbar_init(&vfull[1], 1);
        mbar_init(&sfull[0], 32);
        mbar_init(&sfull[1], 32);
        mbar_init(&sempty[0], 32);
        mbar_init(&sempty[1], 32);
    }
    if (threadIdx.x == 0) mbar_init(s_lbar, 1);
    fence_mbar_init();
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(s_lbar, 2u * (4u << KVC_LUT_BITS));
        tma_load_1d(s_lutK, sd.k_cb->fetch_lut, 4u << KVC_LUT_BITS, s_lbar);
        tma_load_1d(s_lutV, sd.v_cb->fetch_lut_x, 4u << KVC_LUT_BITS, s_lbar);  // bank-swizzled
    }
    const int c_begin = plan.begin[split];
    const int c_end = min(sd.n_chunks, plan.begin[split + 1]);
    const int first = c_begin + pair;
    const int n = first < c_end ? (c_end - first + NP - 1) / NP : 0;
    const float sm_scale = kLog2e / sqrtf((float)D);
    const long nb_k = (long)sd.k_counters->n_blocks, nb_v = (long)sd.v_counters->n_blocks;
    const uint64_t cur_k = sd.k_counters->cursor, cur_v = sd.v_counters->cursor;
    auto issue = [&](bool v, int j) {
        const long ord = (long)(first + NP * j) * H + h;
        const uint32_t *offs = v ? sd.v_offsets : sd.k_offsets;
        const long nb = v ? nb_v : nb_k;
        const uint64_t s0 = offs[ord];
        const uint64_t e0 = (ord + 1 < nb) ? (uint64_t)offs[ord + 1] : (v ? cur_v : cur_k);
        const uint64_t a = s0 & ~15ull;
        uint32_t bytes = (uint32_t)(((e0 + 15) & ~15ull) - a);
        if (bytes > (uint32_t)(v ? stage_v : stage_k)) {
            kvc_set_err(err, KVC_ERR_CODEC);
            bytes = 16;
        }
        const int vsl = VS == 2 ? (j & 1) : 0;
        uint64_t *b = v ? &vfull[vsl] : &kfull[j & 1];
        uint8_t *dst = v ? vring + vsl * stage_v : kring + (j & 1) * stage_k;
        mbar_expect_tx(b, bytes);
        tma_load_1d(dst, (v ? sd.v_arena : sd.k_arena) + a, bytes, b);
    };
    bool bad = false;

    if (!is_v) {
        // ============ K warp: G scores per decoded token ============
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegK));
        if (lane == 0) {
            if (n > 0) issue(false, 0);
            if (n > 1) issue(false, 1);
        }
        float qreg[G][4];
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                qreg[g][k] = q[((long)sidx * H * G + (long)h * G + g) * D + lane + 32 * k];
        const uint32_t qf_s = smem_u32(qf), lut_s = smem_u32(s_lutK);
        mbar_wait(s_lbar, 0);
        uint32_t kofs_next = n > 0 ? sd.k_offsets[(long)first * H + h] & 15u : 0u;
        for (int j = 0; j < n; ++j) {
            const int u = j >> 1, sl = j & 1;
            const uint32_t kofs = kofs_next;
            if (j + 1 < n) kofs_next = sd.k_offsets[(long)(first + NP * (j + 1)) * H + h] & 15u;
            mbar_wait(&kfull[sl], u & 1);
            const uint8_t *ks = kring + sl * stage_k + kofs;
            const uint32_t cA = lds_u16(ks + 6 + 2 * lane), cB = lds_u16(ks + 6 + 2 * (lane + 32));
            const uint32_t iA = kvc_warp_incl_scan(cA, lane);
            const uint32_t totA = __shfl_sync(0xffffffffu, iA, 31);
            const uint32_t iB = kvc_warp_incl_scan(cB, lane);
            float base[G];
#pragma unroll
            for (int g = 0; g < G; ++g) base[g] = 0.f;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = lane + 32 * k;
                const float sc = lds_f32_a2(ks + 6 + 2 * BS + 8 * c + 4);
                const float mn = lds_f32_a2(ks + 6 + 2 * BS + 8 * c);
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    qf[((c >> 1) * G + g) * 2 + (c & 1)] = sc * qreg[g][k];  // [64][G][2]
                    base[g] = fmaf(mn, qreg[g][k], base[g]);
                }
            }
#pragma unroll
            for (int g = 0; g < G; ++g) base[g] = kvc_warp_sum(base[g]);
            __syncwarp();
            const uint32_t bit0 = (kofs + K_HDR) * 8, slot = smem_u32(kring + sl * stage_k);
            Cursor2 cc[2];
            cursor2_init(cc[0], slot, bit0 + iA - cA);
            cursor2_init(cc[1], slot, bit0 + totA + iB - cB);
            const uint32_t p0A = cc[0].p, p0B = cc[1].p;
            float2 sA2[G], sB2[G];
#pragma unroll
            for (int g = 0; g < G; ++g) sA2[g] = sB2[g] = make_float2(0.f, 0.f);
            // 12 groups of 5 pair steps + a tail of 4, one reload per group; q'
            // pairs (channels 2c2, 2c2+1) of every member come as float2s from
            // [64][G][2] (2 members per LDS.128), ready for FFMA2 without moves
            auto steps = [&](int c2base, auto np) {
                cursor2_reload(cc[0]);
                cursor2_reload(cc[1]);
#pragma unroll
                for (int t = 0; t < decltype(np)::value; ++t) {
                    const int c2 = c2base + t;
                    const float2 fA = cursor2_pair(cc[0], lut_s), fB = cursor2_pair(cc[1], lut_s);
#pragma unroll
                    for (int g2 = 0; g2 < G; g2 += 2) {
                        float4 q4;
                        asm volatile(KVC_LD_SHARED ".v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(q4.x), "=f"(q4.y), "=f"(q4.z), "=f"(q4.w)
                                     : "r"(qf_s + 8 * (c2 * G + g2)));
                        const float2 qa = make_float2(q4.x, q4.y), qb = make_float2(q4.z, q4.w);
                        sA2[g2] = __ffma2_rn(fA, qa, sA2[g2]);
                        sB2[g2] = __ffma2_rn(fB, qa, sB2[g2]);
                        sA2[g2 + 1] = __ffma2_rn(fA, qb, sA2[g2 + 1]);
                        sB2[g2 + 1] = __ffma2_rn(fB, qb, sB2[g2 + 1]);
                    }
                }
            };
#pragma unroll 1
            for (int g5 = 0; g5 < 12; ++g5) steps(5 * g5, std::integral_constant<int, 5>());
            steps(60, std::integral_constant<int, 4>());
            bad |= (((cc[0].p - p0A) & 0xFFFFu) != cA) | (((cc[1].p - p0B) & 0xFFFFu) != cB);
            mbar_wait(&sempty[sl], (u & 1) ^ 1);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                sring[(sl * G + g) * BS + lane] = (sA2[g].x + sA2[g].y + base[g]) * sm_scale;
                sring[(sl * G + g) * BS + lane + 32] = (sB2[g].x + sB2[g].y + base[g]) * sm_scale;
            }
            mbar_arrive(&sfull[sl]);
            __syncwarp();
            if (lane == 0 && j + 2 < n) issue(false, j + 2);
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) kvc_set_err(err, KVC_ERR_CODEC);
        __syncthreads();
        __syncthreads();
        return;
    }

    // ============ V warp: decode once into the tile, GEMV for G heads ============
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegV));
    if (lane == 0) {
        if (n > 0) issue(true, 0);
        if (VS == 2 && n > 1) issue(true, 1);
    }
    // GEMV ownership: lane (cg = l & 15, th = l >> 4) sums channels 64*half + 4cg..+3
    // over tokens 32*th..32*th+31; the two token halves are added at the end
    float m[G], lsum[G], wm[G], acc[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        m[g] = -INFINITY;
        lsum[g] = wm[g] = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[g][k] = 0.f;
    }
    const uint32_t lut_s = smem_u32(s_lutV), tile_s = smem_u32(tile), sa_s = smem_u32(sa);
    mbar_wait(s_lbar, 0);
    uint32_t vofs_next = n > 0 ? sd.v_offsets[(long)first * H + h] & 15u : 0u;
    for (int j = 0; j < n; ++j) {
        const int u = j >> 1, sl = j & 1;
        const uint32_t vofs_cur = vofs_next;
        if (j + 1 < n) vofs_next = sd.v_offsets[(long)(first + NP * (j + 1)) * H + h] & 15u;
        mbar_wait(&sfull[sl], u & 1);
        float pA[G], pB[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            pA[g] = sring[(sl * G + g) * BS + lane];
            pB[g] = sring[(sl * G + g) * BS + lane + 32];
        }
        mbar_arrive(&sempty[sl]);
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const float bm = kvc_warp_max(fmaxf(pA[g], pB[g]));
            if (bm > m[g]) {
                const float alpha = exp2f(m[g] - bm);
#pragma unroll
                for (int k = 0; k < 8; ++k) acc[g][k] *= alpha;
                lsum[g] *= alpha;
                wm[g] *= alpha;
                m[g] = bm;
            }
            pA[g] = exp2f(pA[g] - m[g]);
            pB[g] = exp2f(pB[g] - m[g]);
            lsum[g] += pA[g] + pB[g];
        }
        const int vsl = VS == 2 ? sl : 0;
        mbar_wait(&vfull[vsl], VS == 2 ? (u & 1) : (j & 1));
        const uint32_t vofs = vofs_cur;
        const uint8_t *vs = vring + vsl * stage_v + vofs;
        const uint32_t cA = lds_u16(vs + 6 + 2 * lane), cB = lds_u16(vs + 6 + 2 * (lane + 32));
        const uint32_t iA = kvc_warp_incl_scan(cA, lane);
        const uint32_t totA = __shfl_sync(0xffffffffu, iA, 31);
        const uint32_t iB = kvc_warp_incl_scan(cB, lane);
        const float scA = lds_f32_a2(vs + 6 + 2 * BS + 8 * lane + 4);
        const float scB = lds_f32_a2(vs + 6 + 2 * BS + 8 * (lane + 32) + 4);
        const float mnA = lds_f32_a2(vs + 6 + 2 * BS + 8 * lane);
        const float mnB = lds_f32_a2(vs + 6 + 2 * BS + 8 * (lane + 32));
#pragma unroll
        for (int g = 0; g < G; ++g) {
            sa[lane * G + g] = pA[g] * scA;
            sa[(lane + 32) * G + G + g] = pB[g] * scB;
            wm[g] = fmaf(pA[g], mnA, fmaf(pB[g], mnB, wm[g]));
        }
        // decode V slices A (token lane) and B (token lane+32) half by half:
        // channels 0..63 into the half-tile, GEMV, channels 64..127, GEMV
        const uint32_t bit0 = (vofs + V_HDR) * 8, slot = smem_u32(vring + vsl * stage_v);
        Cursor2 cc[2];
        cursor2_init(cc[0], slot, bit0 + iA - cA);
        cursor2_init(cc[1], slot, bit0 + totA + iB - cB);
        const uint32_t p0A = cc[0].p, p0B = cc[1].p;
        const uint32_t rowA = tile_s + lane * kTileRow, rowB = tile_s + (lane + 32) * kTileRow;
        const float2 magic = make_float2(-8388608.f, -8388608.f);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            // 32 pair steps; reload every 5 (the cadence restarts at each half);
            // two steps' symbol pairs go out as one 32-bit store per slice
            uint32_t pA = 0, pB = 0;
#pragma unroll
            for (int t = 0; t < 32; ++t) {
                if (t % 5 == 0) {
                    cursor2_reload(cc[0]);
                    cursor2_reload(cc[1]);
                }
                const uint32_t eA = lds32(lut_s + (((cc[0].hi >> 18) ^ (cc[0].hi >> 25)) & 0x3FFCu));
                cc[0].hi = __funnelshift_l(cc[0].lo, cc[0].hi, eA);
                cc[0].lo = __funnelshift_l(0u, cc[0].lo, eA);
                cc[0].p += eA;
                const uint32_t eB = lds32(lut_s + (((cc[1].hi >> 18) ^ (cc[1].hi >> 25)) & 0x3FFCu));
                cc[1].hi = __funnelshift_l(cc[1].lo, cc[1].hi, eB);
                cc[1].lo = __funnelshift_l(0u, cc[1].lo, eB);
                cc[1].p += eB;
                if (t % 2 == 0) {
                    pA = eA;
                    pB = eB;
                } else {
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(rowA + 2 * (t - 1)), "r"(__byte_perm(pA, eA, 0x7632)));
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(rowB + 2 * (t - 1)), "r"(__byte_perm(pB, eB, 0x7632)));
                }
            }
            __syncwarp();
            if (VS == 1 && half == 1 && lane == 0 && j + 1 < n) issue(true, j + 1);  // slot consumed
            // GEMV: 4 codes per 32-bit load; the upper half-warp walks its tokens
            // rotated by 16 so the two halves read disjoint banks
            {
                const uint32_t cg = lane & 15, th = lane >> 4;
#pragma unroll 4
                for (int t = 0; t < 32; ++t) {
                    const int tok = th ? 32 + ((t + 16) & 31) : t;
                    uint32_t w;
                    asm volatile(KVC_LD_SHARED ".u32 %0, [%1];" : "=r"(w) : "r"(tile_s + tok * kTileRow + 4 * cg));
                    const float2 f01 = __fadd2_rn(make_float2(sym_hi_byte(w, 0x7650), sym_hi_byte(w, 0x7651)), magic);
                    const float2 f23 = __fadd2_rn(make_float2(sym_hi_byte(w, 0x7652), sym_hi_byte(w, 0x7653)), magic);
                    float av[G];
                    lds_vec<G>(sa_s + 4 * (G * tok + (th ? G : 0)), av);
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const float2 a2 = make_float2(av[g], av[g]);
                        float2 x = make_float2(acc[g][4 * half], acc[g][4 * half + 1]);
                        float2 y = make_float2(acc[g][4 * half + 2], acc[g][4 * half + 3]);
                        x = __ffma2_rn(f01, a2, x);
                        y = __ffma2_rn(f23, a2, y);
                        acc[g][4 * half] = x.x;
                        acc[g][4 * half + 1] = x.y;
                        acc[g][4 * half + 2] = y.x;
                        acc[g][4 * half + 3] = y.y;
                    }
                }
            }
            __syncwarp();
        }
        bad |= (((cc[0].p - p0A) & 0xFFFFu) != cA) | (((cc[1].p - p0B) & 0xFFFFu) != cB);
        if (VS == 2 && lane == 0 && j + 2 < n) issue(true, j + 2);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) kvc_set_err(err, KVC_ERR_CODEC);
    __syncthreads();  // K warps done: their region is scratch
    Partial *wp = reinterpret_cast<Partial *>(smem + pair * per_pair);  // G partials per pair
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const float l = kvc_warp_sum(lsum[g]), w2 = kvc_warp_sum(wm[g]);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[g][k] += __shfl_xor_sync(0xffffffffu, acc[g][k], 16);
        if (lane < 16) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                wp[g].o[4 * lane + k] = acc[g][k] + w2;
                wp[g].o[64 + 4 * lane + k] = acc[g][4 + k] + w2;
            }
        }
        if (lane == 0) {
            wp[g].m = m[g];
            wp[g].l = l;
        }
    }
    __syncthreads();
    if (pair == 0) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float M = -INFINITY;
            for (int w = 0; w < NP; ++w)
                M = fmaxf(M, reinterpret_cast<const Partial *>(smem + w * per_pair)[g].m);
            float L = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
            for (int w = 0; w < NP; ++w) {
                const Partial *pw = reinterpret_cast<const Partial *>(smem + w * per_pair) + g;
                const float sc = (pw->m == -INFINITY) ? 0.f : exp2f(pw->m - M);
                L += pw->l * sc;
#pragma unroll
                for (int k = 0; k < 4; ++k) o[k] += pw->o[lane + 32 * k] * sc;
            }
            Partial *dst = partial + ((long)sidx * H * G + (long)h * G + g) * n_splits + split;
#pragma unroll
            for (int k = 0; k < 4; ++k) dst->o[lane + 32 * k] = o[k];
            if (lane == 0) {
                dst->m = M;
                dst->l = L;
            }
        }
    }
}


// ---------------------------------------------------------------------------
// Decode-once GQA fused fetch on tensor cores (default for groups 2 and 4).
// Same warp specialisation, TMA rings and score ring as fused_attn_gqa_kernel,
// but both dot products run on mma.sync m16n8k16 (f16 in, f32 accumulate):
//   K warp: the decoded codes of a 16-channel slab x 64 tokens go to a 1 KB u8
//     tile (one STS.128 per slice and slab), ldmatrix brings 4 codes per lane,
//     two PRMT + HSUB2 make them exact f16 A fragments (channel order
//     permuted within the slab; B follows), and S[tok][n] += codes . B with B
//     = q' in two f16 pieces (n = g: f16(q' 2^e), n = G+g: the f16
//     remainder; 2^e a per-chunk power of two): 8 slabs x 4 token m-tiles;
//   V warp: the same u8 slab tile, ldmatrix.trans, is V^T (rows = channel
//     pairs) and O^T[ch][n] += V^T . W with W = p_t scale_t in two f16 pieces
//     (per-chunk power-of-two scale): 8 channel m-tiles x 4 token k-steps.
// The FFMA dot products of the CUDA-core kernel (4 FFMA2 + 2 LDS.128 per
// pair step on the K side, a per-channel GEMV on the V side) become ~1
// instruction per pair step plus the MMAs.
// ---------------------------------------------------------------------------
constexpr int kMmRow = 16;          // u8 code tile row: one 16-channel slab
constexpr int kQbRow = 272;         // q' pieces [8][128 + 8] f16
constexpr int kWbRow = 144;         // w pieces [8][64 + 8] f16
constexpr int kRegKm = 120, kRegVm = 136;
__host__ __device__ constexpr int gqa_mma_per_pair(int stage_k, int stage_v, int G, int vslots) {
    return 2 * stage_k + vslots * stage_v + 8 * kQbRow + 8 * kWbRow + 2 * G * BS * 4 +
           2 * BS * kMmRow + 64;
}

// f16x2 of two u8 codes picked from x by a PRMT selector ([b, 0x64, b', 0x64]):
// f16(1024 + c) has the code in its low mantissa bits, minus 1024 is exact
template <uint32_t SEL>
__device__ __forceinline__ uint32_t u8x2_f16x2(uint32_t x) {
    const uint32_t y = __byte_perm(x, 0x6464u, SEL);
    uint32_t r;
    asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(y), "r"(0x64006400u));
    return r;
}
// k position of channel c (0..15) of a slab in the K MMA: ldmatrix hands lane
// (g, t) the codes 4t..4t+3, used as k = 2t, 2t+1, 2t+8, 2t+9
__host__ __device__ constexpr int slab_kpos(int c) {
    return 2 * (c >> 2) + (c & 1) + 8 * ((c >> 1) & 1);
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
                 "r"(d));
}
__device__ __forceinline__ void sts16(uint32_t addr, __half v) {
    asm volatile("st.shared.b16 [%0], %1;" ::"r"(addr), "h"(__half_as_ushort(v)));
}
__device__ __forceinline__ uint32_t lds32m(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
// power of two p with amax * p in [2^13, 2^14) (p = 1 for amax == 0)
__device__ __forceinline__ int pow2_exp(float amax) { return amax > 0.f ? 13 - ilogbf(amax) : 0; }

template <int G, int NP, int VS>
__global__ void __launch_bounds__(NP * 64, 1)
fused_attn_gqa_mma_kernel(const kvc_seq_desc *__restrict__ seqs, int H,
                          const float *__restrict__ q, Partial *__restrict__ partial,
                          const SplitPlan plan, int stage_k, int stage_v, int *err) {
    static_assert(G == 2 || G == 4, "GQA group");
    __shared__ __align__(128) uint32_t s_lutK[1 << KVC_LUT_BITS];
    __shared__ __align__(128) uint32_t s_lutV[1 << KVC_LUT_BITS];
    __shared__ uint64_t s_lbar[1];
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const bool is_v = warp >= NP;
    const int pair = is_v ? warp - NP : warp;
    const int per_pair = gqa_mma_per_pair(stage_k, stage_v, G, VS);
    uint8_t *pb = smem + pair * per_pair;
    uint8_t *kring = pb, *vring = pb + 2 * stage_k;
    uint8_t *qb = vring + VS * stage_v;                       // [8][kQbRow]
    uint8_t *wb = qb + 8 * kQbRow;                            // [8][kWbRow]
    float *sring = reinterpret_cast<float *>(wb + 8 * kWbRow);  // [2][G][64]
    uint8_t *kbuf = reinterpret_cast<uint8_t *>(sring + 2 * G * BS);  // [64][kMmRow]
    uint8_t *vbuf = kbuf + BS * kMmRow;                                 // [64][kMmRow]
    uint64_t *bar = reinterpret_cast<uint64_t *>(vbuf + BS * kMmRow);
    uint64_t *kfull = bar, *vfull = bar + 2, *sfull = bar + 4, *sempty = bar + 6;

    const int n_splits = plan.n;
    int split, h, sidx;
    plan_decode(plan, H, split, h, sidx);
    const kvc_seq_desc sd = kvc_load_desc(seqs, sidx);
    if (!is_v && lane == 0) {
        mbar_init(&kfull[0], 1);
        mbar_init(&kfull[1], 1);
        mbar_init(&vfull[0], 1);
        mbar_init(&vfull[1], 1);
        mbar_init(&sfull[0], 32);
        mbar_init(&sfull[1], 32);
        mbar_init(&sempty[0], 32);
        mbar_init(&sempty[1], 32);
    }
    if (threadIdx.x == 0) mbar_init(s_lbar, 1);
    fence_mbar_init();
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(s_lbar, 2u * (4u << KVC_LUT_BITS));
        tma_load_1d(s_lutK, sd.k_cb->fetch_lut, 4u << KVC_LUT_BITS, s_lbar);
        tma_load_1d(s_lutV, sd.v_cb->fetch_lut_x, 4u << KVC_LUT_BITS, s_lbar);  // bank-swizzled
    }
    const int c_begin = plan.begin[split];
    const int c_end = min(sd.n_chunks, plan.begin[split + 1]);
    const int first = c_begin + pair;
    const int n = first < c_end ? (c_end - first + NP - 1) / NP : 0;
    const float sm_scale = kLog2e / sqrtf((float)D);
    const long nb_k = (long)sd.k_counters->n_blocks, nb_v = (long)sd.v_counters->n_blocks;
    const uint64_t cur_k = sd.k_counters->cursor, cur_v = sd.v_counters->cursor;
    auto issue = [&](bool v, int j) {
        const long ord = (long)(first + NP * j) * H + h;
        const uint32_t *offs = v ? sd.v_offsets : sd.k_offsets;
        const long nb = v ? nb_v : nb_k;
        const uint64_t s0 = offs[ord];
        const uint64_t e0 = (ord + 1 < nb) ? (uint64_t)offs[ord + 1] : (v ? cur_v : cur_k);
        const uint64_t a = s0 & ~15ull;
        uint32_t bytes = (uint32_t)(((e0 + 15) & ~15ull) - a);
        if (bytes > (uint32_t)(v ? stage_v : stage_k)) {
            kvc_set_err(err, KVC_ERR_CODEC);
            bytes = 16;
        }
        const int vsl = VS == 2 ? (j & 1) : 0;
        uint64_t *b = v ? &vfull[vsl] : &kfull[j & 1];
        uint8_t *dst = v ? vring + vsl * stage_v : kring + (j & 1) * stage_k;
        mbar_expect_tx(b, bytes);
        tma_load_1d(dst, (v ? sd.v_arena : sd.k_arena) + a, bytes, b);
    };
    bool bad = false;
    // this lane's rows of a 64-token code tile: token lane (slice A), lane+32 (B)
    const uint32_t rowA_k = smem_u32(kbuf) + lane * kMmRow, rowB_k = rowA_k + 32 * kMmRow;
    const uint32_t rowA_v = smem_u32(vbuf) + lane * kMmRow, rowB_v = rowA_v + 32 * kMmRow;

    if (!is_v) {
        // ======== K warp: codes tile -> S = codes . q' on tensor cores ========
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegKm));
        if (lane == 0) {
            if (n > 0) issue(false, 0);
            if (n > 1) issue(false, 1);
        }
        float qreg[G][4];
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                qreg[g][k] = q[((long)sidx * H * G + (long)h * G + g) * D + lane + 32 * k];
        const uint32_t lut_s = smem_u32(s_lutK), qb_s = smem_u32(qb);
        // ldmatrix x4 over tokens 0-31 / 32-63 of the slab tile: lane t's row = token t
        const uint32_t a_ld = smem_u32(kbuf) + lane * kMmRow;
        mbar_wait(s_lbar, 0);
        uint32_t kofs_next = n > 0 ? sd.k_offsets[(long)first * H + h] & 15u : 0u;
        for (int j = 0; j < n; ++j) {
            const int u = j >> 1, sl = j & 1;
            const uint32_t kofs = kofs_next;
            if (j + 1 < n) kofs_next = sd.k_offsets[(long)(first + NP * (j + 1)) * H + h] & 15u;
            mbar_wait(&kfull[sl], u & 1);
            const uint8_t *ks = kring + sl * stage_k + kofs;
            const uint32_t cA = lds_u16(ks + 6 + 2 * lane), cB = lds_u16(ks + 6 + 2 * (lane + 32));
            const uint32_t iA = kvc_warp_incl_scan(cA, lane);
            const uint32_t totA = __shfl_sync(0xffffffffu, iA, 31);
            const uint32_t iB = kvc_warp_incl_scan(cB, lane);
            // q' = scale_c q_c per member, its power-of-two scale, the f16 pieces
            float base[G], qp[G][4], amax = 0.f;
#pragma unroll
            for (int g = 0; g < G; ++g) base[g] = 0.f;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = lane + 32 * k;
                const float sc = lds_f32_a2(ks + 6 + 2 * BS + 8 * c + 4);
                const float mn = lds_f32_a2(ks + 6 + 2 * BS + 8 * c);
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    qp[g][k] = sc * qreg[g][k];
                    amax = fmaxf(amax, fabsf(qp[g][k]));
                    base[g] = fmaf(mn, qreg[g][k], base[g]);
                }
            }
            const int e = pow2_exp(kvc_warp_max(amax));
            const float qs = ldexpf(1.f, e);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = lane + 32 * k;
                const uint32_t col = 2 * ((c & ~15) + slab_kpos(c & 15));
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    __half hi, lo;
                    split_f16(qp[g][k] * qs, hi, lo);
                    sts16(qb_s + g * kQbRow + col, hi);
                    sts16(qb_s + (G + g) * kQbRow + col, lo);
                }
            }
#pragma unroll
            for (int g = 0; g < G; ++g) base[g] = kvc_warp_sum(base[g]);
            __syncwarp();
            const uint32_t bit0 = (kofs + K_HDR) * 8, slot = smem_u32(kring + sl * stage_k);
            Cursor2 cc[2];
            cursor2_init(cc[0], slot, bit0 + iA - cA);
            cursor2_init(cc[1], slot, bit0 + totA + iB - cB);
            const uint32_t p0A = cc[0].p, p0B = cc[1].p;
            float d[4][4];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) d[mt][0] = d[mt][1] = d[mt][2] = d[mt][3] = 0.f;
            // 8 slabs of 16 channels: decode 8 pair steps of both slices (codes
            // packed 4 per register, one STS.128 per slice), then 4 MMAs over the
            // 64 tokens with f16 A fragments made from the u8 tile
            auto kstep = [&](auto ksc) {
                constexpr int kst = decltype(ksc)::value;
                uint32_t ra[4], rb[4], ta = 0, tb = 0;
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    if ((8 * kst + t) % 5 == 0) {
                        cursor2_reload(cc[0]);
                        cursor2_reload(cc[1]);
                    }
                    uint32_t eA = lds32(lut_s + ((cc[0].hi >> 20) << 2));
                    cc[0].hi = __funnelshift_l(cc[0].lo, cc[0].hi, eA);
                    cc[0].lo = __funnelshift_l(0u, cc[0].lo, eA);
                    cc[0].p += eA;
                    uint32_t eB = lds32(lut_s + ((cc[1].hi >> 20) << 2));
                    cc[1].hi = __funnelshift_l(cc[1].lo, cc[1].hi, eB);
                    cc[1].lo = __funnelshift_l(0u, cc[1].lo, eB);
                    cc[1].p += eB;
                    if (t & 1) {
                        ra[t >> 1] = __byte_perm(ta, eA, 0x7632);
                        rb[t >> 1] = __byte_perm(tb, eB, 0x7632);
                    } else {
                        ta = eA;
                        tb = eB;
                    }
                }
                sts128(rowA_k, ra[0], ra[1], ra[2], ra[3]);
                sts128(rowB_k, rb[0], rb[1], rb[2], rb[3]);
                __syncwarp();
                uint32_t b0 = 0, b1 = 0;
                if (gid < 2 * G) {
                    const uint32_t ba = qb_s + gid * kQbRow + (16 * kst + 2 * tig) * 2;
                    b0 = lds32m(ba);
                    b1 = lds32m(ba + 16);
                }
#pragma unroll
                for (int hlf = 0; hlf < 2; ++hlf) {
                    uint32_t x0, x1, x2, x3;  // tokens 32hlf + 8i + g: codes 4t..4t+3
                    ldsm_x4(a_ld + hlf * 32 * kMmRow, x0, x1, x2, x3);
                    {
                        const uint32_t a[4] = {u8x2_f16x2<0x5140>(x0), u8x2_f16x2<0x5140>(x1),
                                               u8x2_f16x2<0x5342>(x0), u8x2_f16x2<0x5342>(x1)};
                        mma_f16_16816(d[2 * hlf], a, b0, b1);
                    }
                    {
                        const uint32_t a[4] = {u8x2_f16x2<0x5140>(x2), u8x2_f16x2<0x5140>(x3),
                                               u8x2_f16x2<0x5342>(x2), u8x2_f16x2<0x5342>(x3)};
                        mma_f16_16816(d[2 * hlf + 1], a, b0, b1);
                    }
                }
                __syncwarp();
            };
            kstep(std::integral_constant<int, 0>());
            kstep(std::integral_constant<int, 1>());
            kstep(std::integral_constant<int, 2>());
            kstep(std::integral_constant<int, 3>());
            kstep(std::integral_constant<int, 4>());
            kstep(std::integral_constant<int, 5>());
            kstep(std::integral_constant<int, 6>());
            kstep(std::integral_constant<int, 7>());
            bad |= (((cc[0].p - p0A) & 0xFFFFu) != cA) | (((cc[1].p - p0B) & 0xFFFFu) != cB);
            // S[tok][n]: hi column g + lo column G + g (xor G/2 lanes away)
            const float inv_qs = ldexpf(1.f, -e);
            float sv[4][4];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    sv[mt][r] = d[mt][r] + __shfl_xor_sync(0xffffffffu, d[mt][r], G / 2);
            mbar_wait(&sempty[sl], (u & 1) ^ 1);
            if (tig < G / 2) {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int g = 2 * tig + c;
                    float bg = base[0];
#pragma unroll
                    for (int gg = 1; gg < G; ++gg) bg = g == gg ? base[gg] : bg;
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt) {
                        sring[(sl * G + g) * BS + 16 * mt + gid] = (sv[mt][c] * inv_qs + bg) * sm_scale;
                        sring[(sl * G + g) * BS + 16 * mt + gid + 8] =
                            (sv[mt][2 + c] * inv_qs + bg) * sm_scale;
                    }
                }
            }
            mbar_arrive(&sfull[sl]);
            __syncwarp();
            if (lane == 0 && j + 2 < n) issue(false, j + 2);
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) kvc_set_err(err, KVC_ERR_CODEC);
        __syncthreads();
        __syncthreads();
        return;
    }

    // ======== V warp: softmax, codes tile -> O^T += V^T . W on tensor cores ========
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegVm));
    if (lane == 0) {
        if (n > 0) issue(true, 0);
        if (VS == 2 && n > 1) issue(true, 1);
    }
    float m[G], lsum[G], wm[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        m[g] = -INFINITY;
        lsum[g] = wm[g] = 0.f;
    }
    // acc[s]: O^T rows (channels 16s + 2gid, 16s + 2gid + 1) x columns n = 2tig, 2tig+1
    float acc[8][4];
#pragma unroll
    for (int s = 0; s < 8; ++s) acc[s][0] = acc[s][1] = acc[s][2] = acc[s][3] = 0.f;
    const uint32_t lut_s = smem_u32(s_lutV), wb_s = smem_u32(wb);
    // ldmatrix x4 .trans over tokens 0-31 / 32-63 of the slab tile (row = token)
    const uint32_t a_ldv = smem_u32(vbuf) + lane * kMmRow;
    mbar_wait(s_lbar, 0);
    uint32_t vofs_next = n > 0 ? sd.v_offsets[(long)first * H + h] & 15u : 0u;
    for (int j = 0; j < n; ++j) {
        const int u = j >> 1, sl = j & 1;
        const uint32_t vofs_cur = vofs_next;
        if (j + 1 < n) vofs_next = sd.v_offsets[(long)(first + NP * (j + 1)) * H + h] & 15u;
        mbar_wait(&sfull[sl], u & 1);
        float pA[G], pB[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            pA[g] = sring[(sl * G + g) * BS + lane];
            pB[g] = sring[(sl * G + g) * BS + lane + 32];
        }
        mbar_arrive(&sempty[sl]);
        float alpha[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const float bm = kvc_warp_max(fmaxf(pA[g], pB[g]));
            alpha[g] = 1.f;
            if (bm > m[g]) {
                alpha[g] = exp2f(m[g] - bm);
                lsum[g] *= alpha[g];
                wm[g] *= alpha[g];
                m[g] = bm;
            }
            pA[g] = exp2f(pA[g] - m[g]);
            pB[g] = exp2f(pB[g] - m[g]);
            lsum[g] += pA[g] + pB[g];
        }
        {   // rescale the accumulators: column n = 2tig + c belongs to member n % G
            // (explicit selects: a select loop over g was lowered to a local array)
            const bool odd = (tig & 1) != 0;
            const float a0 = (G == 4 && odd) ? alpha[2 % G] : alpha[0];
            const float a1 = (G == 4 && odd) ? alpha[3 % G] : alpha[1 % G];
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                acc[s][0] *= a0; acc[s][1] *= a1; acc[s][2] *= a0; acc[s][3] *= a1;
            }
        }
        const int vsl = VS == 2 ? sl : 0;
        mbar_wait(&vfull[vsl], VS == 2 ? (u & 1) : (j & 1));
        const uint32_t vofs = vofs_cur;
        const uint8_t *vs = vring + vsl * stage_v + vofs;
        const uint32_t cA = lds_u16(vs + 6 + 2 * lane), cB = lds_u16(vs + 6 + 2 * (lane + 32));
        const uint32_t iA = kvc_warp_incl_scan(cA, lane);
        const uint32_t totA = __shfl_sync(0xffffffffu, iA, 31);
        const uint32_t iB = kvc_warp_incl_scan(cB, lane);
        const float scA = lds_f32_a2(vs + 6 + 2 * BS + 8 * lane + 4);
        const float scB = lds_f32_a2(vs + 6 + 2 * BS + 8 * (lane + 32) + 4);
        const float mnA = lds_f32_a2(vs + 6 + 2 * BS + 8 * lane);
        const float mnB = lds_f32_a2(vs + 6 + 2 * BS + 8 * (lane + 32));
        // W = p scale per token and member, power-of-two scaled, f16 hi / lo rows
        float amax = 0.f;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            wm[g] = fmaf(pA[g], mnA, fmaf(pB[g], mnB, wm[g]));
            pA[g] *= scA;
            pB[g] *= scB;
            amax = fmaxf(amax, fmaxf(fabsf(pA[g]), fabsf(pB[g])));
        }
        const int e = pow2_exp(kvc_warp_max(amax));
        const float ws = ldexpf(1.f, e), inv_ws = ldexpf(1.f, -e);
#pragma unroll
        for (int g = 0; g < G; ++g) {
            __half hi, lo;
            split_f16(pA[g] * ws, hi, lo);
            sts16(wb_s + g * kWbRow + 2 * lane, hi);
            sts16(wb_s + (G + g) * kWbRow + 2 * lane, lo);
            split_f16(pB[g] * ws, hi, lo);
            sts16(wb_s + g * kWbRow + 2 * (lane + 32), hi);
            sts16(wb_s + (G + g) * kWbRow + 2 * (lane + 32), lo);
        }
        __syncwarp();
        uint32_t bw0[4], bw1[4];  // B fragments of W for the 4 token k-steps
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            bw0[k] = bw1[k] = 0;
            if (gid < 2 * G) {
                const uint32_t ba = wb_s + gid * kWbRow + (16 * k + 2 * tig) * 2;
                bw0[k] = lds32m(ba);
                bw1[k] = lds32m(ba + 16);
            }
        }
        const uint32_t bit0 = (vofs + V_HDR) * 8, slot = smem_u32(vring + vsl * stage_v);
        Cursor2 cc[2];
        cursor2_init(cc[0], slot, bit0 + iA - cA);
        cursor2_init(cc[1], slot, bit0 + totA + iB - cB);
        const uint32_t p0A = cc[0].p, p0B = cc[1].p;
        auto slab = [&](auto ssc) {
            constexpr int s = decltype(ssc)::value;
            uint32_t ra[4], rb[4], ta = 0, tb = 0;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                if ((8 * s + t) % 5 == 0) {
                    cursor2_reload(cc[0]);
                    cursor2_reload(cc[1]);
                }
                const uint32_t eA = lds32(lut_s + (((cc[0].hi >> 18) ^ (cc[0].hi >> 25)) & 0x3FFCu));
                cc[0].hi = __funnelshift_l(cc[0].lo, cc[0].hi, eA);
                cc[0].lo = __funnelshift_l(0u, cc[0].lo, eA);
                cc[0].p += eA;
                const uint32_t eB = lds32(lut_s + (((cc[1].hi >> 18) ^ (cc[1].hi >> 25)) & 0x3FFCu));
                cc[1].hi = __funnelshift_l(cc[1].lo, cc[1].hi, eB);
                cc[1].lo = __funnelshift_l(0u, cc[1].lo, eB);
                cc[1].p += eB;
                if (t & 1) {
                    ra[t >> 1] = __byte_perm(ta, eA, 0x7632);
                    rb[t >> 1] = __byte_perm(tb, eB, 0x7632);
                } else {
                    ta = eA;
                    tb = eB;
                }
            }
            sts128(rowA_v, ra[0], ra[1], ra[2], ra[3]);
            sts128(rowB_v, rb[0], rb[1], rb[2], rb[3]);
            __syncwarp();
            // V^T A fragments: lane (g, t) holds codes (tok 2t, 2t+1) x (ch 2g, 2g+1)
            // per 8-token matrix; rows g / g+8 of the m-tile = channels 2g / 2g+1
            float dd[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int hlf = 0; hlf < 2; ++hlf) {
                uint32_t x0, x1, x2, x3;
                ldsm_x4_t(a_ldv + hlf * 32 * kMmRow, x0, x1, x2, x3);
                {
                    const uint32_t a[4] = {u8x2_f16x2<0x5240>(x0), u8x2_f16x2<0x5341>(x0),
                                           u8x2_f16x2<0x5240>(x1), u8x2_f16x2<0x5341>(x1)};
                    mma_f16_16816(dd, a, bw0[2 * hlf], bw1[2 * hlf]);
                }
                {
                    const uint32_t a[4] = {u8x2_f16x2<0x5240>(x2), u8x2_f16x2<0x5341>(x2),
                                           u8x2_f16x2<0x5240>(x3), u8x2_f16x2<0x5341>(x3)};
                    mma_f16_16816(dd, a, bw0[2 * hlf + 1], bw1[2 * hlf + 1]);
                }
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[s][r] = fmaf(dd[r], inv_ws, acc[s][r]);
            __syncwarp();
        };
        slab(std::integral_constant<int, 0>());
        slab(std::integral_constant<int, 1>());
        slab(std::integral_constant<int, 2>());
        slab(std::integral_constant<int, 3>());
        slab(std::integral_constant<int, 4>());
        slab(std::integral_constant<int, 5>());
        slab(std::integral_constant<int, 6>());
        slab(std::integral_constant<int, 7>());
        bad |= (((cc[0].p - p0A) & 0xFFFFu) != cA) | (((cc[1].p - p0B) & 0xFFFFu) != cB);
        __syncwarp();
        if (VS == 1 && lane == 0 && j + 1 < n) issue(true, j + 1);  // slot consumed
        if (VS == 2 && lane == 0 && j + 2 < n) issue(true, j + 2);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) kvc_set_err(err, KVC_ERR_CODEC);
    __syncthreads();  // K warps done: their region is scratch
    Partial *wp = reinterpret_cast<Partial *>(smem + pair * per_pair);  // G partials per pair
    // columns: hi n = g (lanes tig < G/2), lo n = G + g (xor G/2 lanes away)
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[s][r] += __shfl_xor_sync(0xffffffffu, acc[s][r], G / 2);
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const float l = kvc_warp_sum(lsum[g]), w2 = kvc_warp_sum(wm[g]);
        if (tig == g / 2) {
            const int c = g & 1;
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                wp[g].o[16 * s + 2 * gid] = acc[s][c] + w2;
                wp[g].o[16 * s + 2 * gid + 1] = acc[s][2 + c] + w2;
            }
        }
        if (lane == 0) {
            wp[g].m = m[g];
            wp[g].l = l;
        }
    }
    __syncthreads();
    if (pair == 0) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float M = -INFINITY;
            for (int w = 0; w < NP; ++w)
                M = fmaxf(M, reinterpret_cast<const Partial *>(smem + w * per_pair)[g].m);
            float L = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
            for (int w = 0; w < NP; ++w) {
                const Partial *pw = reinterpret_cast<const Partial *>(smem + w * per_pair) + g;
                const float sc = (pw->m == -INFINITY) ? 0.f : exp2f(pw->m - M);
                L += pw->l * sc;
#pragma unroll
                for (int k = 0; k < 4; ++k) o[k] += pw->o[lane + 32 * k] * sc;
            }
            Partial *dst = partial + ((long)sidx * H * G + (long)h * G + g) * n_splits + split;
#pragma unroll
            for (int k = 0; k < 4; ++k) dst->o[lane + 32 * k] = o[k];
            if (lane == 0) {
                dst->m = M;
                dst->l = L;
            }
        }
    }
}

// Merge split partials + the f32 buffered tokens (attention.py:103-107,
// :160-164) into out = O / L; also writes buffered scores when requested.
// Latency-shaped (it runs once per (seq, query head) per layer, between two
// long kernels; in a batch-1 decode step its time is on the critical path):
// each warp takes buffered rows w, w+4, .. and issues the K and V rows of up
// to 8 of them (float4 per lane: coalesced 512-B rows) before any use, then
// runs its own online softmax over them (scores by shuffle reduction); the
// 4 warps' (m, l, o) and the split partials merge once at the end.  At most
// 128 registers, so a large batch's thousands of these CTAs still run 4+ per SM.
__global__ void __launch_bounds__(128, 4)
combine_kernel(const kvc_seq_desc *__restrict__ seqs, int H, int bs, const float *__restrict__ q,
               const Partial *__restrict__ partial, int n_splits, float *__restrict__ out,
               float *__restrict__ scores, long ctx_stride, int group = 1) {
    static_assert(D == 128, "a float4 per lane covers one head row");
    constexpr int R = 8;  // rows per warp per pass (K and V: 16 float4 registers)
    __shared__ __align__(16) float sh_o[4][D];
    __shared__ float sh_m[4], sh_l[4];
    const int hq = blockIdx.y, sidx = blockIdx.z, h = hq / group, HQ = H * group;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const kvc_seq_desc sd = kvc_load_desc(seqs, sidx);
    const float sm_scale = kLog2e / sqrtf((float)D), inv_sqrt = 1.0f / sqrtf((float)D);
    const int nbuf = sd.buffered;
    const long t0 = (long)sd.n_chunks * bs;
    const Partial *p = partial + ((long)sidx * HQ + hq) * n_splits;
    const float4 q4 = reinterpret_cast<const float4 *>(q + ((long)sidx * HQ + hq) * D)[lane];
    float m = -INFINITY, l = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int tb = warp; tb < nbuf; tb += 4 * R) {
        float4 k4[R], v4[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int t = tb + 4 * j;
            const long row = ((long)t * H + h) * D;
            k4[j] = t < nbuf ? reinterpret_cast<const float4 *>(sd.k_buffer + row)[lane]
                             : make_float4(0.f, 0.f, 0.f, 0.f);
            v4[j] = t < nbuf ? reinterpret_cast<const float4 *>(sd.v_buffer + row)[lane]
                             : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float sc[R];
        float bm = -INFINITY;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int t = tb + 4 * j;
            float a = k4[j].x * q4.x;
            a = fmaf(k4[j].y, q4.y, a);
            a = fmaf(k4[j].z, q4.z, a);
            a = fmaf(k4[j].w, q4.w, a);
            a = kvc_warp_sum(a);  // every lane holds the row's score
            if (t < nbuf && lane == 0 && scores)
                scores[((long)sidx * HQ + hq) * ctx_stride + t0 + t] = a * inv_sqrt;
            sc[j] = t < nbuf ? a * sm_scale : -INFINITY;
            bm = fmaxf(bm, sc[j]);
        }
        if (bm > m) {  // warp-uniform
            const float alpha = exp2f(m - bm);
            l *= alpha;
            acc.x *= alpha; acc.y *= alpha; acc.z *= alpha; acc.w *= alpha;
            m = bm;
        }
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const float e = exp2f(sc[j] - m);  // 0 for rows past nbuf
            l += e;
            acc.x = fmaf(e, v4[j].x, acc.x);
            acc.y = fmaf(e, v4[j].y, acc.y);
            acc.z = fmaf(e, v4[j].z, acc.z);
            acc.w = fmaf(e, v4[j].w, acc.w);
        }
    }
    reinterpret_cast<float4 *>(sh_o[warp])[lane] = acc;
    if (lane == 0) {
        sh_m[warp] = m;
        sh_l[warp] = l;
    }
    __syncthreads();
    // merge: the 4 warps' buffered partials and the split partials
    float M = fmaxf(fmaxf(sh_m[0], sh_m[1]), fmaxf(sh_m[2], sh_m[3]));
    for (int sp = 0; sp < n_splits; ++sp) M = fmaxf(M, p[sp].m);
    const int c = tid;  // blockDim == D
    float L = 0.f, o = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        if (sh_m[w] != -INFINITY) {
            const float sw = exp2f(sh_m[w] - M);
            L += sh_l[w] * sw;
            o += sh_o[w][c] * sw;
        }
    }
    for (int sp = 0; sp < n_splits; ++sp) {
        const float ms = p[sp].m;
        if (ms != -INFINITY) {
            const float sw = exp2f(ms - M);
            L += p[sp].l * sw;
            o += p[sp].o[c] * sw;
        }
    }
    out[((long)sidx * HQ + hq) * D + c] = o / L;
}

// ---------------------------------------------------------------------------
// Uncompressed fp16 decode attention (comparator): K/V [S, H, ctx, D] f16.
// A half-warp covers one token row (16 lanes x 16 B); 8 rows in flight per
// warp per iteration; online softmax; split-K partials -> combine.
// ---------------------------------------------------------------------------
constexpr int kDenseNW = 4;
// G query heads share each KV head (GQA); K/V rows are read once for all G.
template <int G>
__global__ void __launch_bounds__(kDenseNW * 32)
dense_attn_kernel(const __half *__restrict__ K, const __half *__restrict__ V, int H, long ctx,
                  const float *__restrict__ q, Partial *__restrict__ partial, long tok_per_split,
                  int n_splits) {
    const int split = blockIdx.x, h = blockIdx.y, sidx = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane & 15, half = lane >> 4;
    const long base = ((long)sidx * H + h) * ctx * D;
    const __half *Kh = K + base, *Vh = V + base;
    const float sm_scale = kLog2e / sqrtf((float)D);
    float qv[G][8];
#pragma unroll
    for (int j = 0; j < G; ++j) {
        const float *qh = q + ((long)sidx * H * G + (long)h * G + j) * D;
#pragma unroll
        for (int i = 0; i < 8; ++i) qv[j][i] = qh[g * 8 + i] * sm_scale;
    }
    const long t_begin = (long)split * tok_per_split;
    const long t_end = min(ctx, t_begin + tok_per_split);
    float m[G], l[G], o[G][8];
#pragma unroll
    for (int j = 0; j < G; ++j) {
        m[j] = -INFINITY;
        l[j] = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) o[j][i] = 0.f;
    }
    constexpr int R = G > 2 ? 4 : 8;  // rows per half-warp per iteration
    for (long t0 = t_begin + (long)warp * 2 * R; t0 < t_end; t0 += (long)kDenseNW * 2 * R) {
        uint4 kr[R], vr[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            long t = t0 + 2 * r + half;
            if (t < t_end) {
                kr[r] = __ldg(reinterpret_cast<const uint4 *>(Kh + t * D) + g);
                vr[r] = __ldg(reinterpret_cast<const uint4 *>(Vh + t * D) + g);
            } else {
                kr[r] = make_uint4(0, 0, 0, 0);
                vr[r] = make_uint4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int j = 0; j < G; ++j) {
            float s[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const __half2 *k2 = reinterpret_cast<const __half2 *>(&kr[r]);
                float a = 0.f;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    float2 f = __half22float2(k2[i]);
                    a = fmaf(f.x, qv[j][2 * i], a);
                    a = fmaf(f.y, qv[j][2 * i + 1], a);
                }
#pragma unroll
                for (int o2 = 8; o2 > 0; o2 >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o2);
                s[r] = (t0 + 2 * r + half < t_end) ? a : -INFINITY;
            }
            float bm = -INFINITY;
#pragma unroll
            for (int r = 0; r < R; ++r) bm = fmaxf(bm, s[r]);
            bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 16));
            if (bm > m[j]) {
                float alpha = exp2f(m[j] - bm);
                l[j] *= alpha;
#pragma unroll
                for (int i = 0; i < 8; ++i) o[j][i] *= alpha;
                m[j] = bm;
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float pr = exp2f(s[r] - m[j]);
                l[j] += pr;
                const __half2 *v2 = reinterpret_cast<const __half2 *>(&vr[r]);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    float2 f = __half22float2(v2[i]);
                    o[j][2 * i] = fmaf(pr, f.x, o[j][2 * i]);
                    o[j][2 * i + 1] = fmaf(pr, f.y, o[j][2 * i + 1]);
                }
            }
        }
    }
    // merge the two half-warps (same m), then warps via smem
    __shared__ float sh_o[kDenseNW][D], sh_m[kDenseNW], sh_l[kDenseNW];
#pragma unroll
    for (int j = 0; j < G; ++j) {
        float lj = l[j] + __shfl_xor_sync(0xffffffffu, l[j], 16);
        float oj[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) oj[i] = o[j][i] + __shfl_xor_sync(0xffffffffu, o[j][i], 16);
        __syncthreads();
        if (half == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) sh_o[warp][g * 8 + i] = oj[i];
        }
        if (lane == 0) {
            sh_m[warp] = m[j];
            sh_l[warp] = lj;
        }
        __syncthreads();
        if (threadIdx.x < D) {
            float M = -INFINITY;
            for (int w = 0; w < kDenseNW; ++w) M = fmaxf(M, sh_m[w]);
            float L = 0.f, O = 0.f;
            for (int w = 0; w < kDenseNW; ++w) {
                float sc = sh_m[w] == -INFINITY ? 0.f : exp2f(sh_m[w] - M);
                L += sh_l[w] * sc;
                O += sh_o[w][threadIdx.x] * sc;
            }
            Partial *dst = partial + ((long)sidx * H * G + (long)h * G + j) * n_splits + split;
            dst->o[threadIdx.x] = O;
            if (threadIdx.x == 0) {
                dst->m = M;
                dst->l = L;
            }
        }
    }
}


// ---------------------------------------------------------------------------
// Uncompressed fp16 GQA decode attention on tensor cores (comparator, G > 1):
// flash-decoding with mma.sync m16n8k16.  Per warp, 32-token tiles of K and V
// stream HBM -> shared memory with cp.async (3 stages, rows padded to 272 B
// so ldmatrix is conflict-free).  S = Q.K^T with Q as the A operand: rows
// 0..G-1 hold f16(q'), rows G..2G-1 the f16 remainder q' - f16(q') (q'
// scaled by a power of two into f16 range), so one MMA computes both halves
// of a 22-bit-accurate product; O = P.V with P split the same way (P as A,
// from the S accumulators; V^T fragments by ldmatrix.trans).  Online softmax
// in the log2 domain; split partials -> dense_combine_kernel.
// ---------------------------------------------------------------------------
constexpr int kDmNW = 4, kDmTile = 32, kDmStages = 3, kDmRow = 272;
constexpr int kDmTileBytes = kDmTile * kDmRow;
constexpr size_t kDmSmem = (size_t)kDmNW * kDmStages * 2 * kDmTileBytes;

template <int G>
__global__ void __launch_bounds__(kDmNW * 32, 1)
dense_attn_mma_kernel(const __half *__restrict__ K, const __half *__restrict__ V, int H, long ctx,
                      const float *__restrict__ q, Partial *__restrict__ partial,
                      long tok_per_split, int n_splits) {
    static_assert(G == 2 || G == 4 || G == 8, "GQA group");
    extern __shared__ __align__(128) uint8_t smem[];
    const int split = blockIdx.x, h = blockIdx.y, sidx = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const long base = ((long)sidx * H + h) * ctx * D;
    const __half *Kh = K + base, *Vh = V + base;
    const uint32_t wbuf = smem_u32(smem) + warp * kDmStages * 2 * kDmTileBytes;
    const long t_begin = (long)split * tok_per_split;
    const long t_end = min(ctx, t_begin + tok_per_split);
    const long first = t_begin + (long)warp * kDmTile, stride = (long)kDmNW * kDmTile;
    const int n_tiles = first < t_end ? (int)((t_end - first + stride - 1) / stride) : 0;

    // q' = q * log2e / sqrt(D), scaled by qs = 2^e so max |q' qs| < 2^14
    const float *qg = q + ((long)sidx * H * G + (long)h * G) * D;
    const float sm_scale = kLog2e / sqrtf((float)D);
    float amax = 0.f;
    for (int i = lane; i < G * D; i += 32) amax = fmaxf(amax, fabsf(qg[i]) * sm_scale);
    amax = kvc_warp_max(amax);
    const int e = amax > 0.f ? 14 - ilogbf(amax) - 1 : 0;
    const float qs = ldexpf(1.f, e), inv_qs = ldexpf(1.f, -e);
    // A fragments of Q for the 8 k-steps: row r -> member r % G, hi if r < G
    uint32_t aq[8][4];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int row = gid + ((r & 1) ? 8 : 0);
            const int col = 16 * ks + 2 * tig + ((r & 2) ? 8 : 0);
            uint32_t v = 0;
            if (row < 2 * G) {
                const float *qm = qg + (row % G) * D + col;
                __half h0, l0, h1, l1;
                split_f16(qm[0] * sm_scale * qs, h0, l0);
                split_f16(qm[1] * sm_scale * qs, h1, l1);
                v = row < G ? pack_half2(h0, h1) : pack_half2(l0, l1);
            }
            aq[ks][r] = v;
        }
    }
    auto load_tile = [&](int i) {
        if (i < n_tiles) {
            const long t0 = first + (long)i * stride;
            const uint32_t slot = wbuf + (i % kDmStages) * 2 * kDmTileBytes;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int c = lane + 32 * j, row = c >> 4, c16 = c & 15;
                const long t = t0 + row;
                const bool ok = t < t_end;
                const long tt = ok ? t : t_begin;
                cp_async16(slot + row * kDmRow + c16 * 16, Kh + tt * D + c16 * 8, ok ? 16u : 0u);
                cp_async16(slot + kDmTileBytes + row * kDmRow + c16 * 16, Vh + tt * D + c16 * 8,
                           ok ? 16u : 0u);
            }
        }
        cp_async_commit();
    };
#pragma unroll
    for (int i = 0; i < kDmStages - 1; ++i) load_tile(i);

    float m_run = -INFINITY, l_run = 0.f;
    float o[16][4];
#pragma unroll
    for (int n = 0; n < 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    const bool row_live = gid < 2 * G;
    for (int i = 0; i < n_tiles; ++i) {
        cp_async_wait<kDmStages - 2>();
        __syncwarp();
        const long t0 = first + (long)i * stride;
        const uint32_t sk = wbuf + (i % kDmStages) * 2 * kDmTileBytes, sv = sk + kDmTileBytes;
        // ---- S = Q K^T: 4 n-tiles of 8 tokens
        float sc[4][4];
#pragma unroll
        for (int n = 0; n < 4; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
            for (int np = 0; np < 2; ++np) {
                const int mi = lane >> 3;
                const int tok = 16 * np + (mi >> 1) * 8 + (lane & 7);
                const int ch = 16 * ks + (mi & 1) * 8;
                uint32_t b0, b1, b2, b3;
                ldsm_x4(sk + tok * kDmRow + ch * 2, b0, b1, b2, b3);
                mma_f16_16816(sc[2 * np], aq[ks], b0, b1);
                mma_f16_16816(sc[2 * np + 1], aq[ks], b2, b3);
            }
        }
        // ---- full scores of this thread's member: hi rows + lo rows
        float s[4][2];
#pragma unroll
        for (int n = 0; n < 4; ++n) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                float v = sc[n][c];
                if (G == 8) v += sc[n][2 + c];
                else v += __shfl_xor_sync(0xffffffffu, v, 4 * G);
                const long t = t0 + 8 * n + 2 * tig + c;
                s[n][c] = (t < t_end && row_live) ? v * inv_qs : -INFINITY;
            }
        }
        float mx = -INFINITY;
#pragma unroll
        for (int n = 0; n < 4; ++n) mx = fmaxf(mx, fmaxf(s[n][0], s[n][1]));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float m_new = fmaxf(m_run, mx);
        if (m_new > m_run) {
            const float alpha = exp2f(m_run - m_new);
            l_run *= alpha;
#pragma unroll
            for (int n = 0; n < 16; ++n) {
                o[n][0] *= alpha; o[n][1] *= alpha; o[n][2] *= alpha; o[n][3] *= alpha;
            }
            m_run = m_new;
        }
        // ---- P as the A operand (x 2^12, hi rows / lo rows)
        uint32_t ap[2][4];
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                const int n = 2 * kk + hf;
                __half h0, l0, h1, l1;
                float p0 = row_live ? exp2f(s[n][0] - m_run) : 0.f;
                float p1 = row_live ? exp2f(s[n][1] - m_run) : 0.f;
                l_run += p0 + p1;
                split_f16(p0 * 4096.f, h0, l0);
                split_f16(p1 * 4096.f, h1, l1);
                const uint32_t hv = pack_half2(h0, h1), lv = pack_half2(l0, l1);
                ap[kk][2 * hf] = gid < G ? hv : (row_live ? lv : 0u);
                ap[kk][2 * hf + 1] = G == 8 ? lv : 0u;  // rows gid+8: lo rows when G = 8
            }
        }
        // ---- O += P V: 16 n-tiles of 8 channels, 2 k-steps of 16 tokens
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
            const uint32_t a[4] = {ap[kk][0], ap[kk][1], ap[kk][2], ap[kk][3]};
#pragma unroll
            for (int np = 0; np < 8; ++np) {
                const int mi = lane >> 3;
                const int tok = 16 * kk + (mi & 1) * 8 + (lane & 7);
                const int ch = 16 * np + (mi >> 1) * 8;
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(sv + tok * kDmRow + ch * 2, b0, b1, b2, b3);
                mma_f16_16816(o[2 * np], a, b0, b1);
                mma_f16_16816(o[2 * np + 1], a, b2, b3);
            }
        }
        __syncwarp();
        load_tile(i + kDmStages - 1);
    }
    cp_async_wait<0>();
    // ---- per-warp result of member gid (< G): hi + lo rows, x 2^-12
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
    __syncthreads();  // all warps done with their tile buffers: reuse as scratch
    float *sh_o = reinterpret_cast<float *>(smem);               // [NW][G][D]
    float *sh_ml = sh_o + kDmNW * G * D;                          // [NW][G][2]
#pragma unroll
    for (int n = 0; n < 16; ++n) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            float v = o[n][c];
            if (G == 8) v += o[n][2 + c];
            else v += __shfl_xor_sync(0xffffffffu, v, 4 * G);
            if (gid < G) sh_o[(warp * G + gid) * D + 8 * n + 2 * tig + c] = v * (1.f / 4096.f);
        }
    }
    if (gid < G && tig == 0) {
        sh_ml[(warp * G + gid) * 2] = m_run;
        sh_ml[(warp * G + gid) * 2 + 1] = l_run;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
        const int g = idx / D, c = idx % D;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kDmNW; ++w) M = fmaxf(M, sh_ml[(w * G + g) * 2]);
        float L = 0.f, O = 0.f;
#pragma unroll
        for (int w = 0; w < kDmNW; ++w) {
            const float mw = sh_ml[(w * G + g) * 2];
            const float sc = mw == -INFINITY ? 0.f : exp2f(mw - M);
            L += sh_ml[(w * G + g) * 2 + 1] * sc;
            O += sh_o[(w * G + g) * D + c] * sc;
        }
        Partial *dst = partial + ((long)sidx * H * G + (long)h * G + g) * n_splits + split;
        dst->o[c] = O;
        if (c == 0) {
            dst->m = M;
            dst->l = L;
        }
    }
}

__global__ void dense_combine_kernel(int H, const Partial *__restrict__ partial, int n_splits,
                                     float *__restrict__ out) {
    const int h = blockIdx.y, sidx = blockIdx.z;
    const Partial *p = partial + ((long)sidx * H + h) * n_splits;
    float M = -INFINITY;
    for (int s = 0; s < n_splits; ++s) M = fmaxf(M, p[s].m);
    float L = 0.f;
    for (int s = 0; s < n_splits; ++s)
        if (p[s].m != -INFINITY) L += p[s].l * exp2f(p[s].m - M);
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
        float o = 0.f;
        for (int s = 0; s < n_splits; ++s)
            if (p[s].m != -INFINITY) o += p[s].o[c] * exp2f(p[s].m - M);
        out[((long)sidx * H + h) * D + c] = o / L;
    }
}

int g_num_sms = 0;
int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

// Chunks per CTA split.  Candidates are multiples of the pair count; the
// model charges each CTA a start/drain cost of ~5 chunk-times and counts
// the idle part of the last wave (resident CTAs = ctas_per_sm x SMs), and picks
// the split with the lowest estimated time.
int pick_chunks_per_split(int max_chunks, long n_heads_total, int ctas_per_sm = 2, int pairs = NW) {
    const long slots = (long)num_sms() * ctas_per_sm;
    long best_cps = 4 * pairs;
    double best = 1e30;
    for (long cps = 4 * pairs; cps <= 4096; cps += pairs) {
        const long splits = (max_chunks + cps - 1) / cps;
        const long ctas = splits * n_heads_total;
        // chunk-times per pair, plus ~5 for the CTA's start (LUT TMA, first ring
        // fills) and drain (partial merge) — fitted to a cps sweep on config 2
        // (64: 1.057, 104: 1.054, 128: 1.040, 172: 1.077 ms/layer)
        const double per_cta = (double)cps / pairs + 5.0;
        const double waves = ceil((double)ctas / (double)slots);
        const double t = waves * per_cta;
        if (t < best - 1e-9) {
            best = t;
            best_cps = cps;
        }
        if (splits == 1) break;
    }
    return (int)best_cps;
}

// Launch-time model of a split plan: list-schedule the CTAs in launch order
// (split-major) onto num_sms * ctas_per_sm slots, a CTA costing its chunks per
// pair + the ~5 chunk-time start/drain of pick_chunks_per_split.  Returns the
// makespan in chunk-times.
double plan_makespan(const int *parts, int n_parts, long units, long slots, int pairs,
                     double start) {
    // identical CTAs per split: g = gcd(units, slots) independent copies of a
    // (units/g, slots/g) schedule have the same makespan, at 1/g the cost
    long a = units, b = slots;
    while (b) {
        const long t = a % b;
        a = b;
        b = t;
    }
    if (a > 1) {
        units /= a;
        slots /= a;
    }
    std::vector<double> heap((size_t)slots, 0.0);  // min-heap of slot free times
    auto greater = [](double a, double b) { return a > b; };
    double end = 0.0;
    for (int s = 0; s < n_parts; ++s) {
        const double cost = (double)parts[s] / pairs + start;
        for (long u = 0; u < units; ++u) {
            std::pop_heap(heap.begin(), heap.end(), greater);
            const double t = heap.back() + cost;
            heap.back() = t;
            std::push_heap(heap.begin(), heap.end(), greater);
            end = t > end ? t : end;
        }
    }
    return end;
}

// Split plan for a fused launch.  Candidates: the uniform split of
// pick_chunks_per_split, and "k large splits of b chunks + 1 or 2 tail
// splits", whose short last CTAs fill the final wave instead of leaving SMs
// idle behind a partial wave of full-length CTAs (config 2: 1280 uniform CTAs
// are 4.3 waves of 296 slots).  The best modelled makespan wins; plans are
// cached per shape.  KVC_FUSED_PLAN="144:144:144:80" overrides (experiments);
// KVC_PLAN_VERBOSE=1 prints each planned shape to stderr.
SplitPlan pick_split_plan(int max_chunks, long units, int ctas_per_sm, int pairs, int max_splits,
                          int uniform_cps, double start) {
    SplitPlan plan{};
    auto set_parts = [&](const std::vector<int> &parts) {
        if (parts.size() > (size_t)kMaxPlan) {  // unreachable: every candidate is bounded above
            fprintf(stderr, "[kvc] split plan of %zu parts exceeds %d\n", parts.size(), kMaxPlan);
            abort();
        }
        plan.n = (int)parts.size();
        plan.begin[0] = 0;
        for (int i = 0; i < plan.n; ++i) plan.begin[i + 1] = plan.begin[i] + parts[i];
    };
    if (const char *env = getenv("KVC_FUSED_PLAN")) {
        std::vector<int> parts;
        for (const char *c = env; *c;) {
            const int v = atoi(c);
            if (v > 0) parts.push_back(v);
            while (*c && *c != ',' && *c != ':') ++c;
            if (*c) ++c;
        }
        long tot = 0;
        for (int v : parts) tot += v;
        if (!parts.empty() && (int)parts.size() <= kMaxPlan && (int)parts.size() <= max_splits &&
            tot >= max_chunks) {
            set_parts(parts);
            return plan;
        }
    }
    if (max_splits > kMaxPlan) max_splits = kMaxPlan;
    if (max_splits < 1) max_splits = 1;
    int ucps = uniform_cps > 0 ? uniform_cps : max_chunks;
    // the plan is a fixed-size kernel parameter: never more than max_splits
    // uniform splits (few heads x long contexts would otherwise ask for more)
    if (ucps > 0 && (max_chunks + ucps - 1) / ucps > max_splits) {
        const int need = (max_chunks + max_splits - 1) / max_splits;
        ucps = (need + pairs - 1) / pairs * pairs;
    }
    std::vector<int> best;
    for (int c0 = 0; c0 < max_chunks; c0 += ucps) best.push_back(std::min(ucps, max_chunks - c0));
    if (best.empty()) best.push_back(1);
    const bool uniform_forced = getenv("KVC_FUSED_CPS") != nullptr || getenv("KVC_GQA_CPS") != nullptr;
    if (!uniform_forced && max_chunks > 0 && (long)best.size() <= max_splits) {
        struct Key {
            int mc;
            long units;
            int cps_sm, pairs, ms, ucps;
            double start;
        };
        static std::mutex mu;
        static std::vector<std::pair<Key, std::vector<int>>> cache;
        std::lock_guard<std::mutex> lock(mu);
        for (auto &e : cache)
            if (e.first.mc == max_chunks && e.first.units == units && e.first.cps_sm == ctas_per_sm &&
                e.first.pairs == pairs && e.first.ms == max_splits && e.first.ucps == ucps &&
                e.first.start == start) {
                set_parts(e.second);
                return plan;
            }
        const long slots = (long)num_sms() * ctas_per_sm;
        double best_t = plan_makespan(best.data(), (int)best.size(), units, slots, pairs, start);
        std::vector<int> cand;
        auto consider = [&]() {
            if ((int)cand.size() > max_splits) return;
            const double t = plan_makespan(cand.data(), (int)cand.size(), units, slots, pairs, start);
            if (t < best_t * (1.0 - 1e-3)) {
                best_t = t;
                best = cand;
            }
        };
        for (int b = 4 * pairs; b < max_chunks; b += pairs) {
            const int k = max_chunks / b;
            for (int kk = k; kk >= 1 && kk >= k - 1; --kk) {
                const int r = max_chunks - kk * b;
                if (r <= 0 || r >= 2 * b) continue;
                cand.assign(kk, b);
                cand.push_back(r);
                consider();
                for (int t = pairs; t < r; t *= 2) {  // two tails: r - t, t
                    cand.assign(kk, b);
                    cand.push_back(r - t);
                    cand.push_back(t);
                    consider();
                }
                if (r >= 3) {  // three near-equal tails
                    const int t3 = r / 3;
                    cand.assign(kk, b);
                    cand.push_back(r - 2 * t3);
                    cand.push_back(t3);
                    cand.push_back(t3);
                    consider();
                }
            }
        }
        if (getenv("KVC_PLAN_VERBOSE")) {
            fprintf(stderr, "[kvc] split plan chunks=%d units=%ld slots=%ld pairs=%d:", max_chunks,
                    units, slots, pairs);
            for (int v : best) fprintf(stderr, " %d", v);
            fprintf(stderr, " (model %.1f chunk-times)\n", best_t);
        }
        if (cache.size() > 64) cache.clear();
        cache.push_back({Key{max_chunks, units, ctas_per_sm, pairs, max_splits, ucps, start}, best});
    }
    set_parts(best);
    return plan;
}

}  // namespace

extern "C" size_t kvc_attention_workspace_bytes(int n_seqs, int H, int group, int D_, int max_chunks) {
    // partials: n_seqs * H * group * max_splits; max splits bounded by chunks / (4*NW)
    long splits = (max_chunks + 4 * NW - 1) / (4 * NW) + 1;
    long nh = (long)n_seqs * H * (group > 0 ? group : 1);
    // (the shape-generic fallback sizes its own scratch: kvc_v_output_workspace_bytes)
    (void)D_;
    return sizeof(Partial) * (size_t)nh * (size_t)splits;
}

extern "C" int kvc_v_output(const kvc_seq_desc *, int, int, int, int, const float *, long, float *,
                            float *, int *, void *);
extern "C" size_t kvc_v_output_workspace_bytes(int n_seqs, int H, int D);

extern "C" int kvc_attention(const kvc_seq_desc *seqs_dev, const kvc_seq_desc *seqs_host,
                             int n_seqs, int H, int D_, int bs, int group, const float *q_dev,
                             float *out_dev, float *scores_dev, long ctx_stride,
                             void *workspace_dev, size_t workspace_bytes, int *err_dev,
                             void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n_seqs < 1 || H < 1) return kvc_fail(KVC_ERR_CONFIG, "bad shape");
    if (group != 1 && group != 2 && group != 4)
        return kvc_fail(KVC_ERR_CONFIG, "fused GQA supports group 2 or 4");
    int max_chunks = 0, max_len = 0, max_len_k = 0, max_len_v = 0, stage_k = 0, stage_v = 0;
    for (int i = 0; i < n_seqs; ++i) {
        max_chunks = seqs_host[i].n_chunks > max_chunks ? seqs_host[i].n_chunks : max_chunks;
        max_len_k = std::max(max_len_k, (int)seqs_host[i].k_max_len);
        max_len_v = std::max(max_len_v, (int)seqs_host[i].v_max_len);
        max_len = std::max(max_len_k, max_len_v);
        stage_k = seqs_host[i].stage_bytes_k > stage_k ? seqs_host[i].stage_bytes_k : stage_k;
        stage_v = seqs_host[i].stage_bytes_v > stage_v ? seqs_host[i].stage_bytes_v : stage_v;
    }
    const bool fused_ok = D_ == D && bs == BS && max_len <= 13 && max_len >= 1;
    if (!fused_ok) return kvc_fail(KVC_ERR_CONFIG, "shape not covered by the fused kernel");
    stage_k = (stage_k + 15) & ~15;
    stage_v = (stage_v + 15) & ~15;
    const int cps = pick_chunks_per_split(max_chunks > 0 ? max_chunks : 1, (long)n_seqs * H);
    const int n_splits = max_chunks > 0 ? (max_chunks + cps - 1) / cps : 1;
    if (sizeof(Partial) * (size_t)n_seqs * H * n_splits > workspace_bytes)
        return kvc_fail(KVC_ERR_CONFIG, "attention workspace too small");
    Partial *part = static_cast<Partial *>(workspace_dev);
    // decoder: pair LUT12 when every code is <= 6 bits (measured fastest, see
    // profiles/), else single-symbol LUT12; env KVC_FUSED_MODE=0|1 overrides.
    // Longer codes: single-symbol decoders, chosen per side (K, V) from the
    // batch's longest code on that side: <= 9 bits the lane-private 9-bit LUT
    // (MODE 6; KVC_FUSED_LUT9=0 selects MODE 2 instead), <= 12 the shared
    // 12-bit LUT (MODE 2), 13 the 13-bit LUT (MODE 5).
    int mode = max_len <= 6 ? 1 : (max_len <= 9 ? 6 : (max_len <= 12 ? 2 : 5));
    if (max_len <= 6) {
        const char *env = getenv("KVC_FUSED_MODE");
        if (env && (env[0] == '0' || env[0] == '1')) mode = env[0] - '0';
    }
    const char *lut9env = getenv("KVC_FUSED_LUT9");
    const bool lut9 = !(lut9env && lut9env[0] == '0');
    auto side_mode = [&](int ml) {
        if (ml > 12) return 5;
        if (!lut9 || ml > 10) return 2;
        return ml <= 8 ? 7 : (ml == 9 ? 6 : 8);
    };
    int kside = mode, vside = mode;
    if (mode != 0 && mode != 1) {
        kside = side_mode(max_len_k);
        vside = side_mode(max_len_v);
        // experiments: KVC_FUSED_KSIDE / KVC_FUSED_VSIDE = 7|6|8|2|5 force a side's
        // decoder when it covers that side's longest code
        auto force = [](const char *name, int ml, int cur) {
            const char *e = getenv(name);
            if (!e) return cur;
            const int m = e[0] - '0';
            const int cap = m == 7 ? 8 : (m == 6 ? 9 : (m == 8 ? 10 : (m == 2 ? 12 : (m == 5 ? 13 : 0))));
            return ml <= cap ? m : cur;
        };
        kside = force("KVC_FUSED_KSIDE", max_len_k, kside);
        vside = force("KVC_FUSED_VSIDE", max_len_v, vside);
        // K on the 16-copy table beside a V side on the shared 12/13-bit tables
        // measured 8-40 % slower than K on the shared table too (config 5 at
        // (0.01, 0.02) and (0.02, 0.05)); every other pairing is faster
        if ((kside == 6 || kside == 8) && vside != 6 && vside != 7 && vside != 8) kside = 2;
        mode = max_len == 13 ? 5 : 2;  // (the fallback kernel's mode)
    }
    const size_t per_warp = 2 * (size_t)(stage_k + stage_v) + D * 4 + 64;
    size_t smem = NW * per_warp;  // dynamic part (LUTs are static)
    if (smem < NW * sizeof(Partial)) smem = NW * sizeof(Partial);
    auto dyn = [](int m) { return m >= 5; };  // LUT in the WS kernel's dynamic region
    const size_t dyn_lut_bytes = (dyn(kside) ? 32768 : 0) + (dyn(vside) ? 32768 : 0);
    const size_t static_lut_bytes = (dyn(kside) ? 0 : (kside == 0 ? 8192 : 16384)) +
                                    (dyn(vside) ? 0 : (vside == 0 ? 8192 : 16384));
    const size_t lut_bytes = mode == 0 ? 2 * 8192 : (mode == 5 ? 2 * 32768 : 2 * 16384);
    if (smem + lut_bytes + 256 > 227 * 1024)
        return kvc_fail(KVC_ERR_CONFIG, "block extents too large for staging");
    dim3 grid(n_splits, H, n_seqs);
    if (group > 1) {
        // decode-once GQA kernel (pair LUT: every code <= 6 bits)
        if (mode != 1 || max_chunks == 0)
            return kvc_fail(KVC_ERR_CONFIG, "fused GQA needs codes <= 6 bits and a compressed region");
        // pairs per CTA (one CTA per SM): 8 with a 1-slot V ring when the staging
        // fits, else 6 or 4 with 2-slot V rings (KVC_GQA_PAIRS=4|6 caps it)
        const size_t lim = 227 * 1024 - 2 * 16384 - 256;
        int np = 8;
        const char *npenv = getenv("KVC_GQA_PAIRS");
        if (npenv && (npenv[0] == '4' || npenv[0] == '6')) np = npenv[0] - '0';
        if (np == 8 && 8 * (size_t)gqa_per_pair(stage_k, stage_v, group, 1) > lim) np = 6;
        if (np == 6 && 6 * (size_t)gqa_per_pair(stage_k, stage_v, group, 2) > lim) np = 4;
        const int vsl = np == 8 ? 1 : 2;
        const size_t g_smem = np * (size_t)gqa_per_pair(stage_k, stage_v, group, vsl);
        if (g_smem + 2 * 16384 + 256 > 227 * 1024)
            return kvc_fail(KVC_ERR_CONFIG, "block extents too large for GQA staging");
        int g_cps = pick_chunks_per_split(max_chunks, (long)n_seqs * H, 1, np);
        if (const char *cenv = getenv("KVC_GQA_CPS")) {  // experiments: chunks per split
            const int v = atoi(cenv);
            if (v >= np && v % np == 0) g_cps = v;
        }
        const long g_max_sp = (long)(workspace_bytes / (sizeof(Partial) * (size_t)n_seqs * H * group));
        // start/drain cost per CTA in chunk-times: ~0.5 for the one-CTA-per-SM GQA
        // kernel (config 3: 448x4+86+85+85 0.558 ms vs 0.565 with 5)
        const SplitPlan g_plan = pick_split_plan(max_chunks, (long)n_seqs * H, 1, np,
                                                 (int)std::min(g_max_sp, 1L << 20), g_cps, 0.5);
        const int g_splits = g_plan.n;
        if (sizeof(Partial) * (size_t)n_seqs * H * group * g_splits > workspace_bytes)
            return kvc_fail(KVC_ERR_CONFIG, "attention workspace too small");
        dim3 g3((unsigned)(g_splits * H * n_seqs));
        // tensor-core decode-once kernel (default); KVC_GQA_IMPL=ffma selects the
        // CUDA-core one
        const char *gimpl = getenv("KVC_GQA_IMPL");
        if (!(gimpl && gimpl[0] == 'f')) {
            int mnp = 8, mvs = 1;
            const char *mnpenv = getenv("KVC_GQA_PAIRS");
            if (mnpenv && (mnpenv[0] == '4' || mnpenv[0] == '6')) mnp = mnpenv[0] - '0';
            while (mnp > 4 && (size_t)mnp * gqa_mma_per_pair(stage_k, stage_v, group, mvs) > lim) mnp -= 2;
            const size_t m_smem = (size_t)mnp * gqa_mma_per_pair(stage_k, stage_v, group, mvs);
            if (m_smem + 2 * 16384 + 256 > 227 * 1024)
                return kvc_fail(KVC_ERR_CONFIG, "block extents too large for GQA staging");
            int m_cps = pick_chunks_per_split(max_chunks, (long)n_seqs * H, 1, mnp);
            const long m_max_sp =
                (long)(workspace_bytes / (sizeof(Partial) * (size_t)n_seqs * H * group));
            const SplitPlan m_plan = pick_split_plan(max_chunks, (long)n_seqs * H, 1, mnp,
                                                     (int)std::min(m_max_sp, 1L << 20), m_cps, 0.5);
            if (sizeof(Partial) * (size_t)n_seqs * H * group * m_plan.n > workspace_bytes)
                return kvc_fail(KVC_ERR_CONFIG, "attention workspace too small");
            dim3 gm((unsigned)(m_plan.n * H * n_seqs));
#define KVC_LAUNCH_GQAM(GG, NPP)                                                                   \
    do {                                                                                           \
        KVC_CUDA_TRY(cudaFuncSetAttribute(fused_attn_gqa_mma_kernel<GG, NPP, 1>,                     \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)m_smem)); \
        fused_attn_gqa_mma_kernel<GG, NPP, 1><<<gm, NPP * 64, m_smem, s>>>(                          \
            seqs_dev, H, q_dev, part, m_plan, stage_k, stage_v, err_dev);                          \
    } while (0)
            if (group == 2) {
                if (mnp >= 8) KVC_LAUNCH_GQAM(2, 8); else if (mnp >= 6) KVC_LAUNCH_GQAM(2, 6); else KVC_LAUNCH_GQAM(2, 4);
            } else {
                if (mnp >= 8) KVC_LAUNCH_GQAM(4, 8); else if (mnp >= 6) KVC_LAUNCH_GQAM(4, 6); else KVC_LAUNCH_GQAM(4, 4);
            }
#undef KVC_LAUNCH_GQAM
            int st = kvc_check_launch("fused_attn_gqa_mma_kernel");
            if (st) return st;
            combine_kernel<<<dim3(1, H * group, n_seqs), 128, 0, s>>>(seqs_dev, H, bs, q_dev, part,
                                                                      m_plan.n, out_dev, nullptr, 0,
                                                                      group);
            return kvc_check_launch("combine_kernel");
        }
#define KVC_LAUNCH_GQA(GG, NPP, VSS)                                                                   \
    do {                                                                                            \
        KVC_CUDA_TRY(cudaFuncSetAttribute(fused_attn_gqa_kernel<GG, NPP, VSS>,                         \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g_smem)); \
        fused_attn_gqa_kernel<GG, NPP, VSS><<<g3, NPP * 64, g_smem, s>>>(                                \
            seqs_dev, H, q_dev, part, g_plan, stage_k, stage_v, err_dev);                           \
    } while (0)
        if (group == 2) {
            if (np == 8) KVC_LAUNCH_GQA(2, 8, 1); else if (np == 6) KVC_LAUNCH_GQA(2, 6, 2); else KVC_LAUNCH_GQA(2, 4, 2);
        } else {
            if (np == 8) KVC_LAUNCH_GQA(4, 8, 1); else if (np == 6) KVC_LAUNCH_GQA(4, 6, 2); else KVC_LAUNCH_GQA(4, 4, 2);
        }
#undef KVC_LAUNCH_GQA
        int st = kvc_check_launch("fused_attn_gqa_kernel");
        if (st) return st;
        combine_kernel<<<dim3(1, H * group, n_seqs), 128, 0, s>>>(seqs_dev, H, bs, q_dev, part,
                                                                  g_splits, out_dev, nullptr, 0,
                                                                  group);
        return kvc_check_launch("combine_kernel");
    }
    const char *impl = getenv("KVC_FUSED_IMPL");
    const bool use_ws = !(impl && impl[0] == 'i');
    size_t ws_smem = WS_PAIRS * (2 * (size_t)(stage_k + stage_v) + 1024 + 64) +
                     dyn_lut_bytes;  // the 13-bit / 9-bit LUTs are dynamic
    if (const char *pad = getenv("KVC_WS_PAD")) ws_smem += (size_t)atoi(pad);  // experiments
    if (use_ws && max_chunks > 0 && ws_smem + static_lut_bytes + 256 <= 227 * 1024) {
        int ws_cps = pick_chunks_per_split(max_chunks, (long)n_seqs * H);
        if (const char *cenv = getenv("KVC_FUSED_CPS")) {  // experiments: chunks per split
            const int v = atoi(cenv);
            if (v >= 4 && v % 4 == 0) ws_cps = v;
        }
        const long ws_max_sp = (long)(workspace_bytes / (sizeof(Partial) * (size_t)n_seqs * H));
        // 5 chunk-times: fitted on config 2 (two CTAs per SM hide a short tail,
        // which a slot model without co-residency cannot see)
        const SplitPlan ws_plan = pick_split_plan(max_chunks, (long)n_seqs * H, 2, WS_PAIRS,
                                                  (int)std::min(ws_max_sp, 1L << 20), ws_cps, 5.0);
        const int ws_splits = ws_plan.n;
        if (sizeof(Partial) * (size_t)n_seqs * H * ws_splits > workspace_bytes)
            return kvc_fail(KVC_ERR_CONFIG, "attention workspace too small");
        dim3 g2((unsigned)(ws_splits * H * n_seqs));
        // V decoder: pair LUT (measured fastest); KVC_FUSED_VMODE=0 selects the
        // lane-replicated, bank-conflict-free single-symbol LUT6 instead.
        const char *venv = getenv("KVC_FUSED_VMODE");
        // default: plain pair LUT for K and V.  KVC_FUSED_VMODE / KVC_FUSED_KMODE
        // = 3 select the lane-substituted lookups (-16% smem wavefronts, but +14%
        // instructions and a dependent second LDS: measured 9% slower, profiles/)
        int vmode = (mode == 0 || mode == 1) ? 1 : vside;
        if ((mode == 0 || mode == 1) && venv && (venv[0] == '0' || venv[0] == '1' || venv[0] == '3' || venv[0] == '4'))
            vmode = venv[0] - '0';
        const char *kenv = getenv("KVC_FUSED_KMODE");
        const int kmode = (mode == 1 && kenv && kenv[0] == '3') ? 3 : mode;
#define KVC_LAUNCH_WS(M, VM)                                                                 \
    do {                                                                                     \
        KVC_CUDA_TRY(cudaFuncSetAttribute(fused_attn_ws_kernel<M, VM>,                       \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                          (int)ws_smem));                                    \
        fused_attn_ws_kernel<M, VM><<<g2, kThreadsWS, ws_smem, s>>>(                         \
            seqs_dev, H, q_dev, scores_dev, ctx_stride, part, ws_plan, stage_k, stage_v,     \
            err_dev);                                                                        \
    } while (0)
#define KVC_LAUNCH_WS_V(M)                                                                   \
    do {                                                                                     \
        if (vside == 7) KVC_LAUNCH_WS(M, 7);                                                 \
        else if (vside == 6) KVC_LAUNCH_WS(M, 6);                                            \
        else if (vside == 8) KVC_LAUNCH_WS(M, 8);                                            \
        else if (vside == 2) KVC_LAUNCH_WS(M, 2);                                            \
        else KVC_LAUNCH_WS(M, 5);                                                            \
    } while (0)
        // (K on the 9- or 10-bit copies only beside V on copies, see above)
#define KVC_LAUNCH_WS_VC(M)                                                                  \
    do {                                                                                     \
        if (vside == 7) KVC_LAUNCH_WS(M, 7);                                                 \
        else if (vside == 6) KVC_LAUNCH_WS(M, 6);                                            \
        else KVC_LAUNCH_WS(M, 8);                                                            \
    } while (0)
        if (mode != 0 && mode != 1) {
            if (kside == 7) KVC_LAUNCH_WS_V(7);
            else if (kside == 6) KVC_LAUNCH_WS_VC(6);
            else if (kside == 8) KVC_LAUNCH_WS_VC(8);
            else if (kside == 2) KVC_LAUNCH_WS_V(2);
            else KVC_LAUNCH_WS_V(5);
        }
#undef KVC_LAUNCH_WS_V
#undef KVC_LAUNCH_WS_VC
        else if (mode == 0) KVC_LAUNCH_WS(0, 0);
        else if (kmode == 3 && vmode == 3) KVC_LAUNCH_WS(3, 3);
        else if (vmode == 0) KVC_LAUNCH_WS(1, 0);
        else if (vmode == 1) KVC_LAUNCH_WS(1, 1);
        else if (vmode == 4) KVC_LAUNCH_WS(1, 4);
        else KVC_LAUNCH_WS(1, 3);
#undef KVC_LAUNCH_WS
        int st = kvc_check_launch("fused_attn_ws_kernel");
        if (st) return st;
        combine_kernel<<<dim3(1, H, n_seqs), 128, 0, s>>>(seqs_dev, H, bs, q_dev, part, ws_splits,
                                                          out_dev, scores_dev, ctx_stride);
        return kvc_check_launch("combine_kernel");
    }
    if (mode == 5) return kvc_fail(KVC_ERR_CONFIG, "13-bit codes: block extents too large for staging");
    if (max_chunks > 0) {
#define KVC_LAUNCH_FUSED(M)                                                                   \
    do {                                                                                      \
        KVC_CUDA_TRY(cudaFuncSetAttribute(fused_attn_kernel<M>,                               \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                          (int)smem));                                        \
        fused_attn_kernel<M><<<grid, kThreadsF, smem, s>>>(seqs_dev, H, q_dev, scores_dev,    \
                                                           ctx_stride, part, cps, n_splits,   \
                                                           stage_k, stage_v, err_dev);        \
    } while (0)
        if (mode == 0) KVC_LAUNCH_FUSED(0);
        else if (mode == 1) KVC_LAUNCH_FUSED(1);
        else KVC_LAUNCH_FUSED(2);
#undef KVC_LAUNCH_FUSED
        int st = kvc_check_launch("fused_attn_kernel");
        if (st) return st;
    }
    combine_kernel<<<dim3(1, H, n_seqs), 128, 0, s>>>(seqs_dev, H, bs, q_dev, part,
                                                      max_chunks > 0 ? n_splits : 0, out_dev,
                                                      scores_dev, ctx_stride);
    return kvc_check_launch("combine_kernel");
}

extern "C" size_t kvc_dense_workspace_bytes(int n_seqs, int H, int group, int D_, long ctx) {
    (void)D_;
    long splits = (ctx + 127) / 128 + 1;  // >= either kernel's split count
    return sizeof(Partial) * (size_t)n_seqs * H * (size_t)(group > 0 ? group : 1) * (size_t)splits;
}

extern "C" int kvc_dense_attention_f16(const void *k_dev, const void *v_dev, int n_seqs, int H,
                                       int D_, int group, long ctx, const float *q_dev,
                                       float *out_dev, void *workspace_dev, size_t workspace_bytes,
                                       void *stream) {
    if (D_ != D) return kvc_fail(KVC_ERR_CONFIG, "dense kernel: head_dim 128");
    if (group != 1 && group != 2 && group != 4 && group != 8)
        return kvc_fail(KVC_ERR_CONFIG, "dense kernel: group must be 1, 2, 4 or 8");
    if (ctx < 1) return kvc_fail(KVC_ERR_CONFIG, "empty context");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    long nh = (long)n_seqs * H;
    const char *ffma_env = getenv("KVC_DENSE_FFMA");  // the older FFMA kernel for G > 1
    if (group > 1 && !(ffma_env && ffma_env[0] == '1')) {
        // tensor-core kernel: one 4-warp CTA per SM (204 KB of cp.async stages);
        // ~4 waves of splits, tokens per split a multiple of 4 warps x 32
        long splits = (4L * num_sms() + nh - 1) / nh;
        long tps = (ctx + splits - 1) / splits;
        tps = (tps + kDmNW * kDmTile - 1) / (kDmNW * kDmTile) * (kDmNW * kDmTile);
        splits = (ctx + tps - 1) / tps;
        if (sizeof(Partial) * (size_t)nh * group * splits > workspace_bytes)
            return kvc_fail(KVC_ERR_CONFIG, "dense workspace too small");
        Partial *part = static_cast<Partial *>(workspace_dev);
        const __half *k = static_cast<const __half *>(k_dev), *v = static_cast<const __half *>(v_dev);
        dim3 grid((unsigned)splits, H, n_seqs);
#define KVC_LAUNCH_DM(GG)                                                                        \
    do {                                                                                         \
        KVC_CUDA_TRY(cudaFuncSetAttribute(dense_attn_mma_kernel<GG>,                              \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,           \
                                          (int)kDmSmem));                                        \
        dense_attn_mma_kernel<GG><<<grid, kDmNW * 32, kDmSmem, s>>>(k, v, H, ctx, q_dev, part,   \
                                                                    tps, (int)splits);           \
    } while (0)
        if (group == 2) KVC_LAUNCH_DM(2);
        else if (group == 4) KVC_LAUNCH_DM(4);
        else KVC_LAUNCH_DM(8);
#undef KVC_LAUNCH_DM
        int st = kvc_check_launch("dense_attn_mma_kernel");
        if (st) return st;
        dense_combine_kernel<<<dim3(1, H * group, n_seqs), 128, 0, s>>>(H * group, part, (int)splits,
                                                                         out_dev);
        return kvc_check_launch("dense_combine_kernel");
    }
    long target = (long)num_sms() * 8 * 2;
    long splits = (target + nh - 1) / nh;
    long tps = (ctx + splits - 1) / splits;
    if (tps < 256) tps = 256;
    tps = (tps + 63) / 64 * 64;
    splits = (ctx + tps - 1) / tps;
    if (sizeof(Partial) * (size_t)nh * group * splits > workspace_bytes)
        return kvc_fail(KVC_ERR_CONFIG, "dense workspace too small");
    Partial *part = static_cast<Partial *>(workspace_dev);
    dim3 grid((unsigned)splits, H, n_seqs);
    const __half *k = static_cast<const __half *>(k_dev), *v = static_cast<const __half *>(v_dev);
    switch (group) {
        case 1: dense_attn_kernel<1><<<grid, kDenseNW * 32, 0, s>>>(k, v, H, ctx, q_dev, part, tps, (int)splits); break;
        case 2: dense_attn_kernel<2><<<grid, kDenseNW * 32, 0, s>>>(k, v, H, ctx, q_dev, part, tps, (int)splits); break;
        case 4: dense_attn_kernel<4><<<grid, kDenseNW * 32, 0, s>>>(k, v, H, ctx, q_dev, part, tps, (int)splits); break;
        default: dense_attn_kernel<8><<<grid, kDenseNW * 32, 0, s>>>(k, v, H, ctx, q_dev, part, tps, (int)splits); break;
    }
    int st = kvc_check_launch("dense_attn_kernel");
    if (st) return st;
    dense_combine_kernel<<<dim3(1, H * group, n_seqs), 128, 0, s>>>(H * group, part, (int)splits, out_dev);
    return kvc_check_launch("dense_combine_kernel");
}
