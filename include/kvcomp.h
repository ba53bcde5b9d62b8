/*
 * kvcomp.h — C ABI of the B200-native KVComp Store/Fetch hot path.
 *
 * The reference (arxiv 2509.00579, package `kvpack`) is pure Python/numpy;
 * its "FFI" for this path is the Python call surface of kvcache.py and
 * attention.py.  Each entry point below replaces one reference function
 * (cited as file:line under /root/reference/pkg/src/kvpack/), and the Python
 * host layer (paper_2509_00579_b200/) binds them with ctypes exactly as
 * INTEGRATION.md shows.
 *
 * Conventions
 *   - plain pointers and sizes only; every *_dev pointer is CUDA device
 *     memory, every other pointer is host memory;
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream);
 *   - every function returns a kvc_status; nonzero codes map 1:1 onto the
 *     reference exception classes (errors.py:4-29);
 *   - kernels never allocate: the caller owns arenas, offsets, codebook
 *     tables, buffers and workspaces (sizes via the *_bytes helpers).
 *
 * Device data layout:
 *   arena      : bytes, exactly the reference serialisation (codec.py:229-244),
 *                blocks appended in block_index order, +16 B slack for TMA;
 *   offsets    : u32 per block (codec.py:298-299);
 *   counters   : kvc_arena_counters, device-resident, updated by the Store
 *                kernels (cursor, blocks, payload bits/bytes, max extent, err);
 *   codebook   : kvc_codebook_dev (encode table + decode LUTs), built on the
 *                host from the 256 code lengths and uploaded once.
 */
#ifndef KVCOMP_H
#define KVCOMP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes <-> reference exceptions (errors.py). */
typedef enum {
    KVC_OK = 0,
    KVC_ERR_CONFIG = 1,        /* ConfigError       errors.py:8  */
    KVC_ERR_TENSOR = 2,        /* TensorFormatError errors.py:12 */
    KVC_ERR_CODEBOOK = 3,      /* CodebookError     errors.py:16 */
    KVC_ERR_CODEC = 4,         /* CodecError        errors.py:20 */
    KVC_ERR_ARENA_FULL = 5,    /* ArenaFullError    errors.py:24 */
    KVC_ERR_CUDA = 6           /* CUDA runtime failure (no reference analogue) */
} kvc_status;

/* Quantisation modes (quantizer.py:37-42). */
enum { KVC_K_BLOCK = 0, KVC_V_TOKEN = 1, KVC_K_CHANNEL = 2 };
/* Input dtypes of the dense K/V tensors (tensor_io.py:30-51). */
enum { KVC_F16 = 0, KVC_F32 = 1, KVC_F64 = 2 /* kvc_quantize only */ };

/* Device-resident per-arena counters (codec.py:279-326 running totals). */
typedef struct {
    uint64_t cursor;         /* write cursor == arena size in bytes          */
    uint64_t n_blocks;       /* blocks appended so far (== len(offsets))      */
    uint64_t payload_bits;   /* sum of slice bit counts                       */
    uint64_t payload_bytes;  /* sum of ceil(bits/8) per block                 */
    uint32_t max_extent;     /* largest serialised block, bytes               */
    int32_t err;             /* sticky device error: kvc_status               */
} kvc_arena_counters;

/* Device codebook tables, built from the 256 code lengths by
 * kvc_codebook_build_tables (codebook.py:128-208 + decode LUTs). */
#define KVC_LUT_BITS 12
typedef struct {
    uint32_t words[256];            /* canonical codeword, right-aligned       */
    uint8_t lengths[256];           /* code length, 0 = absent                 */
    uint32_t lut[1 << KVC_LUT_BITS];/* 12-bit window -> sym | len<<8            */
    /* Fused-fetch LUT over 12-bit windows (16-byte aligned for TMA): when
     * max_len <= 6 each entry decodes exactly two symbols:
     * (l0+l1) | s0<<16 | s1<<24; otherwise one: l0 | s0<<16.  Low 4 bits =
     * bits consumed, bits 4..15 zero. */
    uint32_t fetch_lut[1 << KVC_LUT_BITS];
    /* fetch_lut with its bank bits swizzled: entry i stored at
     * i ^ ((i >> 7) & 31), so the bank of a lookup is window bits 7-11 XOR
     * bits 0-4 (fewer shared-memory bank conflicts for short V pairs). */
    uint32_t fetch_lut_x[1 << KVC_LUT_BITS];
    /* Single-symbol fused-fetch LUT over 13-bit windows for books whose
     * longest code is <= 13 bits (used when it is 13): entry = float bits of
     * the symbol | length (low 4 bits); zero when max_len > 13. */
    uint32_t lut13[1 << 13];
    uint32_t first_code[33];        /* canonical decode (lengths > 12)         */
    uint32_t count[33];
    uint32_t first_index[33];
    uint8_t sorted_symbols[256];
    int32_t fetch_syms;             /* 2 (pair LUT) or 1                      */
    int32_t max_len;
    int32_t n_symbols;
    int32_t single_symbol;          /* degenerate 1-symbol book (codebook.py:149-154) */
} kvc_codebook_dev;

/* One sequence's compressed layer cache, as seen by the Fetch kernels. */
typedef struct {
    const uint8_t *k_arena;
    const uint32_t *k_offsets;
    const kvc_arena_counters *k_counters;
    const kvc_codebook_dev *k_cb;
    const uint8_t *v_arena;
    const uint32_t *v_offsets;
    const kvc_arena_counters *v_counters;
    const kvc_codebook_dev *v_cb;
    const float *k_buffer;          /* [buffer+1, H, D] f32 pending tokens */
    const float *v_buffer;
    int32_t n_chunks;               /* compressed_tokens / block_size          */
    int32_t buffered;               /* tokens in the f32 buffers               */
    int32_t stage_bytes_k;          /* >= max K extent + 48, multiple of 16    */
    int32_t stage_bytes_v;
    int32_t k_max_len;              /* longest K / V code length (host copy)   */
    int32_t v_max_len;
    /* optional device int32[2] {n_chunks, buffered}: when non-NULL the kernels
     * read these two counts from it (kvc_buffer_append / kvc_set_live keep it
     * current), so a decode loop reuses one descriptor array across steps;
     * the host array passed beside it must carry the same values. */
    const int32_t *live;
} kvc_seq_desc;

/* ---------------------------------------------------------------- */
/* Library info                                                      */
/* ---------------------------------------------------------------- */
const char *kvc_version(void);
const char *kvc_last_error(void);   /* message of the last failing call (thread-local) */

/* ---------------------------------------------------------------- */
/* Codebook (host)  — replaces codebook.py:75-230                     */
/* ---------------------------------------------------------------- */

/* smooth_histogram (codebook.py:83-89) when max_code >= 0, then
 * build_codebook (codebook.py:211-218): optimal lengths with (weight,
 * lowest symbol) tie-breaking, 32-bit cap.  hist: 256 x u64. */
int kvc_codebook_lengths(const uint64_t *hist, int max_code, uint8_t *lengths_out);

/* codebook_from_lengths (codebook.py:179-208): Kraft check + canonical
 * words + decode LUTs, written into a host kvc_codebook_dev to upload. */
int kvc_codebook_build_tables(const uint8_t *lengths, kvc_codebook_dev *tables_out);

size_t kvc_codebook_bytes(void);

/* ---------------------------------------------------------------- */
/* Store — replaces kvcache.py:217-268 + quantizer.py:114-209 +       */
/* codec.py:77-138, :229-244, :308-326                               */
/* ---------------------------------------------------------------- */

/* Quantise n_chunks*H blocks of x[t, h, :] (t in [0, n_chunks*bs)) in block
 * order b = chunk*H + head.  codes_dev: [nb, bs, D] u8; metas_dev: [nb,
 * n_units, 2] f32 (min, scale); hist_dev (256 x u64, accumulated) may be
 * NULL.  row_stride = elements between consecutive tokens of x (H*D for
 * a contiguous [ctx, H, D] tensor). */
int kvc_quantize(const void *x_dev, int x_dtype, long row_stride, int n_chunks, int H, int D,
                 int bs, int mode, double rel, const float *k_ranges_dev, uint8_t *codes_dev,
                 float *metas_dev, uint64_t *hist_dev, void *stream);
/*   mode KVC_K_CHANNEL (quantizer.py:191-197): k_ranges_dev = f32 [2][H][D]
 *   whole-context (min, max) per channel; codes clipped to [0, ceil(1/rel)].
 *   k_ranges_dev is ignored (may be NULL) for the other modes. */

/* Entropy-code n_chunks*H_local quantised blocks (order b = chunk*H_local +
 * h) and append them to an arena in that order, reading and advancing the
 * device counters.  block_index = (chunk_base + chunk) * H_total + head_base
 * + h (quantizer.py:201; head_base/H_total let a head-sharded rank keep the
 * global numbering).  Overflow of `capacity` sets counters->err =
 * KVC_ERR_ARENA_FULL and writes nothing (codec.py:313-318).  max_len is the
 * codebook's longest code (sizes the shared-memory block image).
 * workspace_dev: kvc_encode_workspace_bytes(n_chunks*H_local, bs). */
int kvc_encode_append(const uint8_t *codes_dev, const float *metas_dev, int n_chunks,
                      int H_local, int H_total, int head_base, uint32_t chunk_base, int bs,
                      int D, int n_units, int max_len, const kvc_codebook_dev *cb_dev,
                      uint8_t *arena_dev, uint64_t capacity, uint32_t *offsets_dev,
                      kvc_arena_counters *counters_dev, void *workspace_dev, void *stream);
size_t kvc_encode_workspace_bytes(int nb, int bs);

/* Store pass A of prefill (kvcache.py:110-121): quantise the full blocks of K
 * and V and accumulate their code histograms (hist_dev: 512 x u64, K bins
 * then V bins).  No codes are written.  k_mode KVC_K_BLOCK or KVC_K_CHANNEL;
 * K_CHANNEL takes k_ranges_dev = f32 [2][H][D] whole-context (min, max) and
 * clips codes to [0, ceil(1/rel)] (quantizer.py:191-197). */
int kvc_store_hist(const void *k_dev, const void *v_dev, int x_dtype, long row_stride,
                   int n_chunks, int H, int D, int bs, int k_mode, double rel_k, double rel_v,
                   const float *k_ranges_dev, uint64_t *hist_dev, void *stream);

/* 1 if the single-pass Store kernels cover this block shape / code length. */
int kvc_store_supported(int bs, int D, int max_len);

/* One Store event with known codebooks (kvcache.py:217-239): quantise K and
 * V from x[t, h, :] (t < n_chunks*bs), Huffman-encode and append both arenas
 * in one launch; arena offsets come from a decoupled look-back scan in
 * block_index order (deterministic; the codes never leave shared memory). */
int kvc_store_append(const void *k_dev, const void *v_dev, int x_dtype, long row_stride,
                     int n_chunks, int H_local, int H_total, int head_base, int D, int bs,
                     int k_mode, double rel_k, double rel_v, const float *k_ranges_dev,
                     uint32_t chunk_base,
                     const kvc_codebook_dev *k_cb_dev, int k_max_len,
                     const kvc_codebook_dev *v_cb_dev, int v_max_len, uint8_t *k_arena_dev,
                     uint64_t k_capacity, uint32_t *k_offsets_dev,
                     kvc_arena_counters *k_counters_dev, uint8_t *v_arena_dev,
                     uint64_t v_capacity, uint32_t *v_offsets_dev,
                     kvc_arena_counters *v_counters_dev, void *workspace_dev,
                     size_t workspace_bytes, void *stream);
size_t kvc_store_workspace_bytes(int n_chunks, int H, int D, int bs);

/* Prefill without the look-back (kvcache.py:110-145; byte-identical arenas
 * to kvc_store_hist + kvc_store_append).  For alphabets < 32 codes
 * (kvc_store_prefill_supported):
 *   kvc_store_hist_blocks  pass A, also writing per-block code histograms
 *                          blk_hist_dev [2][n_chunks*H][32] u16 (K then V);
 *   kvc_store_prefill      block sizes from those histograms and the code
 *                          lengths, one exclusive scan -> arena offsets in
 *                          block_index order, then pass B writes every block
 *                          at its offset.  workspace >= 64 bytes. */
int kvc_store_prefill_supported(int bs, int D, double rel_k, double rel_v);
size_t kvc_store_blk_hist_bytes(int n_chunks, int H);
int kvc_store_hist_blocks(const void *k_dev, const void *v_dev, int x_dtype, long row_stride,
                          int n_chunks, int H, int D, int bs, int k_mode, double rel_k,
                          double rel_v, const float *k_ranges_dev, uint64_t *hist_dev,
                          uint16_t *blk_hist_dev, uint8_t *codes_dev, void *stream);
/* codes_dev (optional, may be NULL; used for head_dim 128 / block 64): pass A
 * leaves every block's codes and (min, scale) pairs there and pass B encodes
 * from them instead of re-quantising the input (kvc_store_codes_bytes). */
size_t kvc_store_codes_bytes(int n_chunks, int H);
int kvc_store_prefill(const void *k_dev, const void *v_dev, int x_dtype, long row_stride,
                      int n_chunks, int H_local, int H_total, int head_base, int D, int bs,
                      int k_mode, double rel_k, double rel_v, const float *k_ranges_dev,
                      uint32_t chunk_base,
                      const kvc_codebook_dev *k_cb_dev, int k_max_len,
                      const kvc_codebook_dev *v_cb_dev, int v_max_len, uint8_t *k_arena_dev,
                      uint64_t k_capacity, uint32_t *k_offsets_dev,
                      kvc_arena_counters *k_counters_dev, uint8_t *v_arena_dev,
                      uint64_t v_capacity, uint32_t *v_offsets_dev,
                      kvc_arena_counters *v_counters_dev, const uint16_t *blk_hist_dev,
                      const uint8_t *codes_dev, void *workspace_dev, size_t workspace_bytes,
                      void *stream);

/* ---------------------------------------------------------------- */
/* Fetch — replaces attention.py:59-188 and kvcache.py:182-212        */
/* ---------------------------------------------------------------- */

/* fused_k_scores (attention.py:59-109), any shape: scores_dev[s][h][t]
 * (row stride ctx_stride) for t < n_chunks*bs + buffered, x 1/sqrt(D). */
int kvc_k_scores(const kvc_seq_desc *seqs_dev, int n_seqs, int H, int D, int bs,
                 const float *q_dev, float *scores_dev, long ctx_stride, int *err_dev,
                 void *stream);

/* softmax_rows (attention.py:168-173) over rows of length n_cols[s]. */
int kvc_softmax_rows(float *x_dev, int n_rows, long n_cols, long row_stride, void *stream);

/* fused_v_output (attention.py:112-165), any shape: out_dev[s][h][:];
 * ws_dev holds kvc_v_output_workspace_bytes(n_seqs, H, D). */
int kvc_v_output(const kvc_seq_desc *seqs_dev, int n_seqs, int H, int D, int bs,
                 const float *w_dev, long ctx_stride, float *out_dev, float *ws_dev,
                 int *err_dev, void *stream);
size_t kvc_v_output_workspace_bytes(int n_seqs, int H, int D);

/* attention_step (attention.py:176-188) for a batch of sequences with the
 * single-pass fused kernel (Huffman decode -> dequant -> q.K^T -> online
 * softmax -> .V, decompressed KV never leaves shared memory/registers),
 * split over the context and combined.  scores_dev may be NULL.  q_dev
 * [n_seqs, H*group, D]; GQA: `group` query heads per KV head.
 * Covers head_dim 128, block 64 and codes of at most 13 bits (GQA groups 2
 * and 4: at most 6); the decoder is chosen per side from the batch's longest
 * code (pair LUT <= 6 bits, lane-copied single-symbol LUTs 7-10, shared
 * 12- and 13-bit LUTs).  Other shapes or books return KVC_ERR_CONFIG: the
 * caller runs kvc_k_scores / kvc_softmax_rows / kvc_v_output for them (as
 * attention.py does, per state). */
int kvc_attention(const kvc_seq_desc *seqs_dev, const kvc_seq_desc *seqs_host, int n_seqs,
                  int H, int D, int bs, int group, const float *q_dev, float *out_dev,
                  float *scores_dev, long ctx_stride, void *workspace_dev,
                  size_t workspace_bytes, int *err_dev, void *stream);
size_t kvc_attention_workspace_bytes(int n_seqs, int H, int group, int D, int max_chunks);

/* fetch_dequantized (kvcache.py:182-212): f64 dequant, f32 out
 * [ctx, H, D] (compressed region only; buffered rows untouched). */
int kvc_dequantize(const kvc_seq_desc *seq_dev, int H, int D, int bs, int which /*0=K,1=V*/,
                   int n_chunks, float *out_dev, int *err_dev, void *stream);

/* ---------------------------------------------------------------- */
/* Paged arena memory: CUDA virtual memory      */
/* ---------------------------------------------------------------- */
/* An arena reserves a virtual range once and maps fixed-size physical pages
 * (from a shared pool) as it grows, so it stays contiguous for the kernels
 * while physical memory is paged and shared between sequences.
 * kvc_vmm_granularity: the minimum page size; reserve/free_va: a virtual
 * range; create/release: one physical page; map/unmap: a page at a
 * page-aligned address (read/write for `device`).  Out of memory ->
 * KVC_ERR_ARENA_FULL. */
int kvc_vmm_granularity(int device, size_t *bytes);
int kvc_vmm_reserve(size_t bytes, uint64_t *va);
int kvc_vmm_free_va(uint64_t va, size_t bytes);
int kvc_vmm_create(int device, size_t bytes, uint64_t *handle);
int kvc_vmm_release(uint64_t handle);
int kvc_vmm_map(uint64_t va, size_t bytes, uint64_t handle, int device);
int kvc_vmm_unmap(uint64_t va, size_t bytes);

/* ---------------------------------------------------------------- */
/* Growing cache, device side — kvcache.py:150-177 without host syncs */
/* ---------------------------------------------------------------- */

/* append_token's buffer write for n_seqs states in one launch: row
 * buffered (read from seqs_dev[s].live[1], < cap_rows) of each state's K/V
 * f32 buffers <- k/v_rows_dev[s] ([n_seqs][H*D], f16 or f32, seq_stride
 * elements apart), then live[1] += 1.  Non-finite values -> *err_dev (NULL:
 * the state's K arena counters' sticky err, raised by the next check). */
int kvc_buffer_append(const kvc_seq_desc *seqs_dev, int n_seqs, int H, int D, int cap_rows,
                      const void *k_rows_dev, const void *v_rows_dev, int x_dtype,
                      long seq_stride, int *err_dev, void *stream);

/* After an overflow event compressed buffer rows [0, n_rows): move rows
 * [n_rows, n_rows + rem) to the front (rem < n_rows) and set live =
 * {n_chunks, rem} (kvcache.py:168-177), for n_seqs states at once. */
int kvc_buffer_shift(const kvc_seq_desc *seqs_dev, int n_seqs, int H, int D, int n_rows,
                     int rem, int n_chunks, void *stream);

/* live = {n_chunks, buffered} (state creation, prefill, restore). */
int kvc_set_live(int32_t *live_dev, int n_chunks, int buffered, void *stream);

/* ---------------------------------------------------------------- */
/* Per-block codec surface — replaces codec.py:59-472 single-block API */
/* ---------------------------------------------------------------- */

/* decompress_block (codec.py:356-391) for n arena ordinals: codes_dev
 * [n, bs, D] u8, metas_dev [n, n_units, 2] f32 (min, scale), block_index_dev
 * [n] u32 from each header.  Corrupt extents / slices -> *err_dev CodecError.
 * (compress_block / encode_slice: kvc_encode_append on a one-block arena.) */
int kvc_decode_blocks(const uint8_t *arena_dev, const uint32_t *offsets_dev,
                      const kvc_arena_counters *counters_dev, const int32_t *ordinals_dev, int n,
                      int bs, int n_units, int D, const kvc_codebook_dev *cb_dev,
                      uint8_t *codes_dev, float *metas_dev, uint32_t *block_index_dev,
                      int *err_dev, void *stream);

/* decode_slice / decode_slices (codec.py:141-226): the array-form tree walk,
 * one thread per slice, over an unpacked 0/1 bit array (packed = 0) or packed
 * MSB-first bytes (packed = 1) of n_bits bits.  out_dev [n_slices, out_len];
 * *bad_dev (initialise to n_slices) receives the lowest corrupt slice index. */
int kvc_decode_slices_tree(const uint8_t *bits_dev, int packed, uint64_t n_bits,
                           const int64_t *offsets_dev, const int64_t *counts_dev, int n_slices,
                           const int32_t *children_dev, const int32_t *is_symbol_dev,
                           const uint8_t *symbols_dev, int n_nodes, int out_len,
                           uint8_t *out_dev, int *bad_dev, void *stream);

/* CompressedArena.append (codec.py:308-326): one serialised block image
 * (nbytes, a multiple of 4) appended at the device cursor; capacity or
 * 32-bit overflow sets counters->err = KVC_ERR_ARENA_FULL and writes nothing. */
int kvc_arena_append(const uint8_t *image_dev, uint32_t nbytes, uint64_t payload_bits,
                     uint64_t payload_bytes, uint8_t *arena_dev, uint64_t capacity,
                     uint32_t *offsets_dev, kvc_arena_counters *counters_dev, void *stream);

/* CompressedArena.restore (codec.py:329-341): counters of an arena holding
 * `size` serialised bytes and n_blocks offsets, every extent validated as
 * _parse_block (codec.py:247-268); *n_slices_dev = total slices. */
int kvc_arena_restore(const uint8_t *arena_dev, uint64_t size, const uint32_t *offsets_dev,
                      int n_blocks, int n_units, kvc_arena_counters *counters_dev,
                      uint64_t *n_slices_dev, int *err_dev, void *stream);

/* Uncompressed fp16 decode-attention comparator (the north-star baseline):
 * K/V [n_seqs, H, ctx, D] f16 head-major, q [n_seqs, H*group, D] f32. */
int kvc_dense_attention_f16(const void *k_dev, const void *v_dev, int n_seqs, int H, int D,
                            int group, long ctx, const float *q_dev, float *out_dev,
                            void *workspace_dev, size_t workspace_bytes, void *stream);
size_t kvc_dense_workspace_bytes(int n_seqs, int H, int group, int D, long ctx);

#ifdef __cplusplus
}
#endif
#endif /* KVCOMP_H */
