/*
 * kvcomp_oracle.c — CPU restatement of the KVComp Store/Fetch algorithm.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path (and the `cpu_baseline` / `--impl reference` timing leg of bench.py).
 * Product code under paper_2509_00579_b200/ never links or calls it.
 *
 * Pinned against the unmodified reference: the .npz fixtures and big_digests.json
 * in tests/golden/ are produced by tests/golden/make_golden.py,
 * which runs the reference package itself; tests/test_oracle_golden.py
 * checks every function here against those fixtures bit-for-bit.
 *
 * Each function cites the reference (/root/reference/pkg/src/kvpack/...)
 * behaviour it restates.  Arithmetic notes:
 *   - quantisation is done in IEEE binary64 exactly as numpy does it
 *     (quantizer.py:114-141); build with -ffp-contract=off so no FMA
 *     contraction changes a rounding;
 *   - bitstreams are MSB-first, slices packed back-to-back, the block payload
 *     zero-padded to a byte, the serialised block zero-padded to 4 bytes
 *     (codec.py:119-138, :229-244).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* Minimal static-partition parallel-for over [0, n) on pthreads. */
typedef void (*range_fn)(long lo, long hi, int tid, void *ctx);
typedef struct { range_fn fn; void *ctx; long lo, hi; int tid; } prange;

static void *prange_run(void *p)
{
    prange *r = (prange *)p;
    r->fn(r->lo, r->hi, r->tid, r->ctx);
    return NULL;
}

static void parallel_for(long n, int n_threads, range_fn fn, void *ctx)
{
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    if (n_threads == 1 || n < 2) { fn(0, n, 0, ctx); return; }
    pthread_t th[256];
    prange rs[256];
    long per = (n + n_threads - 1) / n_threads;
    for (int t = 0; t < n_threads; ++t) {
        long lo = t * per, hi = lo + per < n ? lo + per : n;
        if (lo > n) lo = n;
        rs[t] = (prange){fn, ctx, lo, hi, t};
        pthread_create(&th[t], NULL, prange_run, &rs[t]);
    }
    for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
}

#define ORC_OK 0
#define ORC_CONFIG 1
#define ORC_CODEBOOK 3
#define ORC_CODEC 4
#define ORC_ARENA_FULL 5

/* ------------------------------------------------------------------ */
/* Quantisation (quantizer.py:107-141, :162-209)                        */
/* ------------------------------------------------------------------ */

/* Quantise n values x[i*stride] sharing one (min, scale) unit.  With
 * fixed_range (K_CHANNEL, quantizer.py:191-197) the unit range is given and
 * codes are clipped to [0, clamp_max]. */
static void quant_unit_r(const float *x, long stride, int n, double rel, uint8_t *codes,
                         long cstride, float *vmin_out, float *scale_out, const float *fixed_range,
                         int clamp_max)
{
    float lo = x[0], hi = x[0];
    if (fixed_range) {
        lo = fixed_range[0];
        hi = fixed_range[1];
    } else {
        for (int i = 1; i < n; ++i) {
            float v = x[(long)i * stride];
            if (v < lo) lo = v;
            if (v > hi) hi = v;
        }
    }
    /* min/max of f32 values are exact; scale = f32(rel64 * (max64 - min64)) */
    float scale = (float)(rel * ((double)hi - (double)lo));
    double s64 = (double)scale;
    for (int i = 0; i < n; ++i) {
        uint8_t c = 0;
        if (s64 > 0.0) {
            double t = ((double)x[(long)i * stride] - (double)lo) / s64;
            double f = floor(t);
            if (t - f >= 0.5) f += 1.0;
            if (fixed_range) {
                if (f < 0) f = 0;
                if (f > clamp_max) f = clamp_max;
            }
            c = (uint8_t)f;
        }
        codes[(long)i * cstride] = c;
    }
    *vmin_out = lo;
    *scale_out = scale;
}

static void quant_unit(const float *x, long stride, int n, double rel, uint8_t *codes,
                       long cstride, float *vmin_out, float *scale_out)
{
    quant_unit_r(x, stride, n, rel, codes, cstride, vmin_out, scale_out, NULL, 0);
}

/*
 * Quantise one (bs, D) block.  mode 0 = K_BLOCK (one unit per column),
 * mode 1 = V_TOKEN (one unit per row).  x rows are `row_stride` floats apart
 * (so a [ctx, H, D] tensor can be addressed in place).
 */
/* K_CHANNEL (mode 2): ranges = [D] mins then [D] maxs for this head. */
int orc_quantize_block_ranges(const float *x, long row_stride, int bs, int D, double rel,
                              const float *rmin, const float *rmax, uint8_t *codes, float *mins,
                              float *scales)
{
    int clamp_max = (int)ceil(1.0 / rel);
    for (int c = 0; c < D; ++c) {
        float r[2] = {rmin[c], rmax[c]};
        quant_unit_r(x + c, row_stride, bs, rel, codes + c, D, &mins[c], &scales[c], r, clamp_max);
    }
    return ORC_OK;
}

int orc_quantize_block(const float *x, long row_stride, int bs, int D, int mode, double rel,
                       uint8_t *codes, float *mins, float *scales)
{
    if (bs < 1 || D < 1) return ORC_CONFIG;
    if (mode == 0) {
        for (int c = 0; c < D; ++c)
            quant_unit(x + c, row_stride, bs, rel, codes + c, D, &mins[c], &scales[c]);
    } else {
        for (int r = 0; r < bs; ++r)
            quant_unit(x + (long)r * row_stride, 1, D, rel, codes + (long)r * D, 1, &mins[r],
                       &scales[r]);
    }
    return ORC_OK;
}

/* codebook.py:75-80 */
void orc_histogram(const uint8_t *codes, long n, uint64_t *hist)
{
    for (long i = 0; i < n; ++i) hist[codes[i]]++;
}

/* ------------------------------------------------------------------ */
/* Huffman code lengths (codebook.py:102-125)                           */
/* Priority = (weight, lowest contained symbol); merged node keeps the  */
/* smaller "lowest symbol".  A symbol's length = number of merges above */
/* it.  One present symbol gets length 1.                               */
/* ------------------------------------------------------------------ */

typedef struct { uint64_t w; int low; int node; } hnode;

static int hless(const hnode *a, const hnode *b)
{
    return a->w < b->w || (a->w == b->w && a->low < b->low);
}

static void hpush(hnode *h, int *n, hnode v)
{
    int i = (*n)++;
    h[i] = v;
    while (i > 0) {
        int p = (i - 1) / 2;
        if (!hless(&h[i], &h[p])) break;
        hnode t = h[i]; h[i] = h[p]; h[p] = t; i = p;
    }
}

static hnode hpop(hnode *h, int *n)
{
    hnode top = h[0];
    h[0] = h[--(*n)];
    int i = 0;
    for (;;) {
        int l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && hless(&h[l], &h[m])) m = l;
        if (r < *n && hless(&h[r], &h[m])) m = r;
        if (m == i) break;
        hnode t = h[i]; h[i] = h[m]; h[m] = t; i = m;
    }
    return top;
}

int orc_huffman_lengths(const uint64_t *hist, uint8_t *lengths)
{
    hnode heap[256];
    int parent[512];
    int n = 0, nodes = 0, present = 0, last = -1;
    memset(lengths, 0, 256);
    for (int s = 0; s < 256; ++s) {
        parent[s] = -1;
        if (hist[s]) { present++; last = s; }
    }
    if (present == 0) return ORC_CODEBOOK;
    if (present == 1) { lengths[last] = 1; return ORC_OK; }
    nodes = 256;
    for (int s = 0; s < 256; ++s)
        if (hist[s]) hpush(heap, &n, (hnode){hist[s], s, s});
    while (n > 1) {
        hnode a = hpop(heap, &n), b = hpop(heap, &n);
        int id = nodes++;
        parent[id] = -1;
        parent[a.node] = id;
        parent[b.node] = id;
        hpush(heap, &n, (hnode){a.w + b.w, a.low < b.low ? a.low : b.low, id});
    }
    for (int s = 0; s < 256; ++s) {
        if (!hist[s]) continue;
        int d = 0;
        for (int p = parent[s]; p >= 0; p = parent[p]) d++;
        if (d > 32) return ORC_CODEBOOK;
        lengths[s] = (uint8_t)d;
    }
    return ORC_OK;
}

/* codebook.py:83-89 */
int orc_smooth_histogram(const uint64_t *hist, int max_code, uint64_t *out)
{
    if (max_code < 0 || max_code > 255) return ORC_CODEBOOK;
    for (int s = 0; s < 256; ++s) out[s] = hist[s] + (s <= max_code ? 1u : 0u);
    return ORC_OK;
}

/* Canonical codewords by (length, symbol) + Kraft check
 * (codebook.py:128-141, :179-208). */
int orc_canonical_words(const uint8_t *lengths, uint32_t *words)
{
    int present = 0, first = -1;
    memset(words, 0, 256 * sizeof(uint32_t));
    for (int s = 0; s < 256; ++s)
        if (lengths[s]) { present++; if (first < 0) first = s; if (lengths[s] > 32) return ORC_CODEBOOK; }
    if (present == 0) return ORC_CODEBOOK;
    if (present == 1) {
        if (lengths[first] != 1) return ORC_CODEBOOK;
        words[first] = 0;
        return ORC_OK;
    }
    uint64_t kraft = 0;
    for (int s = 0; s < 256; ++s)
        if (lengths[s]) kraft += (uint64_t)1 << (32 - lengths[s]);
    if (kraft != ((uint64_t)1 << 32)) return ORC_CODEBOOK;
    uint64_t code = 0;
    int prev = 0;
    for (int len = 1; len <= 32; ++len) {
        for (int s = 0; s < 256; ++s) {
            if (lengths[s] != len) continue;
            if (prev) code <<= (len - prev);
            prev = len;
            words[s] = (uint32_t)code;
            code++;
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Block encode / serialise (codec.py:77-138, :229-244)                 */
/* ------------------------------------------------------------------ */

static long block_header_bytes(int bs, int n_units) { return 6 + 2L * bs + 8L * n_units; }

/* Serialised size of a block whose codes are given. */
long orc_block_size(const uint8_t *codes, int bs, int D, int n_units, const uint8_t *lengths,
                    uint16_t *counts_out, int *status)
{
    uint64_t bits = 0;
    *status = ORC_OK;
    for (int r = 0; r < bs; ++r) {
        uint32_t c = 0;
        for (int j = 0; j < D; ++j) {
            uint8_t l = lengths[codes[(long)r * D + j]];
            if (!l) { *status = ORC_CODEC; return -1; }
            c += l;
        }
        if (c > 0xFFFF) { *status = ORC_CODEC; return -1; }
        if (counts_out) counts_out[r] = (uint16_t)c;
        bits += c;
    }
    if (bits > 0xFFFFFFFFull) { *status = ORC_CODEC; return -1; }
    long raw = block_header_bytes(bs, n_units) + (long)((bits + 7) / 8);
    return (raw + 3) & ~3L;
}

/* Write the serialised block into out (which must hold orc_block_size bytes). */
int orc_encode_block(const uint8_t *codes, int bs, int D, const float *mins, const float *scales,
                     int n_units, uint32_t block_index, const uint8_t *lengths,
                     const uint32_t *words, uint8_t *out, long *out_len)
{
    int st;
    uint16_t *counts = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)bs);
    long total = orc_block_size(codes, bs, D, n_units, lengths, counts, &st);
    if (total < 0) { free(counts); return st; }
    memset(out, 0, (size_t)total);
    out[0] = block_index & 0xFF; out[1] = (block_index >> 8) & 0xFF;
    out[2] = (block_index >> 16) & 0xFF; out[3] = block_index >> 24;
    out[4] = bs & 0xFF; out[5] = (bs >> 8) & 0xFF;
    for (int r = 0; r < bs; ++r) { out[6 + 2 * r] = counts[r] & 0xFF; out[7 + 2 * r] = counts[r] >> 8; }
    uint8_t *meta = out + 6 + 2 * bs;
    for (int u = 0; u < n_units; ++u) {
        memcpy(meta + 8 * u, &mins[u], 4);
        memcpy(meta + 8 * u + 4, &scales[u], 4);
    }
    uint8_t *payload = out + block_header_bytes(bs, n_units);
    uint64_t pos = 0;
    for (long i = 0; i < (long)bs * D; ++i) {
        uint8_t s = codes[i];
        int l = lengths[s];
        uint32_t w = words[s];
        for (int b = l - 1; b >= 0; --b, ++pos)
            if ((w >> b) & 1u) payload[pos >> 3] |= (uint8_t)(0x80u >> (pos & 7));
    }
    free(counts);
    *out_len = total;
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Decode (codec.py:141-226, :247-268): the array-tree walk             */
/* ------------------------------------------------------------------ */

typedef struct { int child[512][2]; int is_sym[512]; int sym[512]; int n; } dtree;

static int build_tree(const uint8_t *lengths, const uint32_t *words, dtree *t)
{
    int present = 0, only = -1;
    memset(t, 0, sizeof(*t));
    t->n = 1;
    for (int s = 0; s < 256; ++s) if (lengths[s]) { present++; only = s; }
    if (present == 1) {
        t->child[0][0] = t->child[0][1] = 1;
        t->is_sym[1] = 1; t->sym[1] = only; t->n = 2;
        return ORC_OK;
    }
    for (int s = 0; s < 256; ++s) {
        int l = lengths[s], node = 0;
        if (!l) continue;
        for (int p = l - 1; p >= 0; --p) {
            int bit = (words[s] >> p) & 1;
            if (!t->child[node][bit]) {
                if (t->n >= 511) return ORC_CODEBOOK;
                t->child[node][bit] = t->n++;
            }
            node = t->child[node][bit];
        }
        t->is_sym[node] = 1;
        t->sym[node] = s;
    }
    return ORC_OK;
}

/* Decode one slice of exactly `nbits` bits starting at bit `pos`. */
static int decode_slice_bits(const uint8_t *buf, uint64_t pos, uint32_t nbits, const dtree *t,
                             uint8_t *out, int out_len)
{
    int node = 0, w = 0;
    for (uint32_t i = 0; i < nbits; ++i, ++pos) {
        int bit = (buf[pos >> 3] >> (7 - (pos & 7))) & 1;
        node = t->child[node][bit];
        if (t->is_sym[node]) {
            if (w < out_len) out[w] = (uint8_t)t->sym[node];
            w++;
            node = 0;
        }
    }
    return (w == out_len && node == 0) ? ORC_OK : ORC_CODEC;
}

/* Parse + decode one serialised block extent [0, len). */
int orc_decode_block(const uint8_t *ext, long len, int n_units, int D, const uint8_t *lengths,
                     uint8_t *codes, float *mins, float *scales, uint32_t *block_index,
                     int *n_slices_out)
{
    uint32_t words[256];
    dtree *t;
    if (len < 6 || (len % 4) != 0) return ORC_CODEC;
    if (orc_canonical_words(lengths, words) != ORC_OK) return ORC_CODEBOOK;
    uint32_t bi = ext[0] | (ext[1] << 8) | (ext[2] << 16) | ((uint32_t)ext[3] << 24);
    int ns = ext[4] | (ext[5] << 8);
    long meta_off = 6 + 2L * ns, pay_off = meta_off + 8L * n_units;
    if (pay_off > len) return ORC_CODEC;
    uint64_t bits = 0;
    for (int r = 0; r < ns; ++r) bits += (uint32_t)(ext[6 + 2 * r] | (ext[7 + 2 * r] << 8));
    long pad = len - pay_off - (long)((bits + 7) / 8);
    if (pad < 0 || pad > 3) return ORC_CODEC;
    for (int u = 0; u < n_units; ++u) {
        memcpy(&mins[u], ext + meta_off + 8 * u, 4);
        memcpy(&scales[u], ext + meta_off + 8 * u + 4, 4);
    }
    t = (dtree *)malloc(sizeof(dtree));
    if (build_tree(lengths, words, t) != ORC_OK) { free(t); return ORC_CODEBOOK; }
    uint64_t pos = 0;
    int st = ORC_OK;
    for (int r = 0; r < ns && st == ORC_OK; ++r) {
        uint32_t c = (uint32_t)(ext[6 + 2 * r] | (ext[7 + 2 * r] << 8));
        st = decode_slice_bits(ext + pay_off, pos, c, t, codes + (long)r * D, D);
        pos += c;
    }
    free(t);
    *block_index = bi;
    *n_slices_out = ns;
    return st;
}

/* ------------------------------------------------------------------ */
/* Store: quantise + encode a block-multiple token range and append     */
/* (kvcache.py:217-268, codec.py:308-326).  Blocks are produced in      */
/* block_index order (chunk-major, head-minor); encoding runs block-    */
/* parallel, the arena layout is a serial prefix sum of block sizes.    */
/* ------------------------------------------------------------------ */

typedef struct {
    const float *tokens; int H, D, bs, mode, n_units; double rel; uint32_t chunk_base;
    int H_total, head_base;
    const float *ranges;  /* K_CHANNEL: [2][H][D] (mins, maxs) of this shard, or NULL */
    const uint8_t *lengths; const uint32_t *words; uint8_t *tmp; long max_block;
    long *sizes; uint64_t *pbits; int err;
} compress_ctx;

static void compress_range(long lo, long hi, int tid, void *p)
{
    compress_ctx *c = (compress_ctx *)p;
    uint8_t *codes = (uint8_t *)malloc((size_t)c->bs * c->D);
    float *mins = (float *)malloc(sizeof(float) * (size_t)c->n_units);
    float *scales = (float *)malloc(sizeof(float) * (size_t)c->n_units);
    for (long b = lo; b < hi; ++b) {
        int chunk = (int)(b / c->H), head = (int)(b % c->H);
        const float *x = c->tokens + ((long)chunk * c->bs * c->H + head) * c->D;
        if (c->ranges)
            orc_quantize_block_ranges(x, (long)c->H * c->D, c->bs, c->D, c->rel,
                                      c->ranges + (long)head * c->D,
                                      c->ranges + ((long)c->H + head) * c->D, codes, mins, scales);
        else
            orc_quantize_block(x, (long)c->H * c->D, c->bs, c->D, c->mode, c->rel, codes, mins,
                               scales);
        long len = 0;
        uint8_t *dst = c->tmp + b * c->max_block;
        int s = orc_encode_block(codes, c->bs, c->D, mins, scales, c->n_units,
                                 (uint32_t)((c->chunk_base + (uint32_t)chunk) * (uint32_t)c->H_total +
                                            (uint32_t)(c->head_base + head)),
                                 c->lengths, c->words, dst, &len);
        if (s) c->err = s;
        c->sizes[b] = len;
        uint64_t bits = 0;
        for (int r = 0; r < c->bs && !s; ++r) bits += (uint32_t)(dst[6 + 2 * r] | (dst[7 + 2 * r] << 8));
        c->pbits[b] = bits;
    }
    free(codes); free(mins); free(scales);
}

/* tokens: [n_tok, H, D] f32 holding heads [head_base, head_base+H) of H_total
 * (a head shard).  Appends n_tok/bs*H blocks at *cursor with
 * block_index = (chunk_base + chunk) * H_total + head_base + h. */
int orc_compress_tokens_shard(const float *tokens, int n_tok, int H, int D, int bs, int mode,
                              double rel, uint32_t chunk_base, int H_total, int head_base,
                              const float *ranges, const uint8_t *lengths, uint8_t *arena,
                              long capacity, long *cursor, uint32_t *offsets_out,
                              uint64_t *payload_bits_out, int n_threads)
{
    uint32_t words[256];
    int st = orc_canonical_words(lengths, words);
    if (st) return st;
    long nb = (long)(n_tok / bs) * H;
    compress_ctx c = {tokens, H, D, bs, mode, mode == 1 ? bs : D, rel, chunk_base, H_total,
                      head_base, ranges, lengths, words, NULL, 0, NULL, NULL, ORC_OK};
    c.max_block = block_header_bytes(bs, c.n_units) + (long)bs * D * 4 + 4;
    c.tmp = (uint8_t *)malloc((size_t)(nb ? nb : 1) * (size_t)c.max_block);
    c.sizes = (long *)calloc((size_t)(nb ? nb : 1), sizeof(long));
    c.pbits = (uint64_t *)calloc((size_t)(nb ? nb : 1), sizeof(uint64_t));
    parallel_for(nb, n_threads, compress_range, &c);
    int err = c.err;
    if (!err) {
        long cur = *cursor;
        for (long b = 0; b < nb; ++b) {
            if ((capacity >= 0 && cur + c.sizes[b] > capacity) || cur + c.sizes[b] > 0xFFFFFFFFL) {
                err = ORC_ARENA_FULL;
                break;
            }
            memcpy(arena + cur, c.tmp + b * c.max_block, (size_t)c.sizes[b]);
            offsets_out[b] = (uint32_t)cur;
            payload_bits_out[b] = c.pbits[b];
            cur += c.sizes[b];
        }
        if (!err) *cursor = cur;
    }
    free(c.tmp); free(c.sizes); free(c.pbits);
    return err;
}

/* tokens: [n_tok, H, D] f32.  Appends n_tok/bs*H blocks at *cursor. */
int orc_compress_tokens(const float *tokens, int n_tok, int H, int D, int bs, int mode,
                        double rel, uint32_t chunk_base, const uint8_t *lengths,
                        uint8_t *arena, long capacity, long *cursor, uint32_t *offsets_out,
                        uint64_t *payload_bits_out, int n_threads)
{
    return orc_compress_tokens_shard(tokens, n_tok, H, D, bs, mode, rel, chunk_base, H, 0, NULL,
                                     lengths, arena, capacity, cursor, offsets_out,
                                     payload_bits_out, n_threads);
}

typedef struct {
    const float *tokens; int H, D, bs, mode, n_units; double rel; uint64_t (*local)[256];
    const float *ranges;
} hist_ctx;

static void hist_range(long lo, long hi, int tid, void *p)
{
    hist_ctx *c = (hist_ctx *)p;
    uint8_t *codes = (uint8_t *)malloc((size_t)c->bs * c->D);
    float *mins = (float *)malloc(sizeof(float) * (size_t)c->n_units);
    float *scales = (float *)malloc(sizeof(float) * (size_t)c->n_units);
    for (long b = lo; b < hi; ++b) {
        int chunk = (int)(b / c->H), head = (int)(b % c->H);
        const float *x = c->tokens + ((long)chunk * c->bs * c->H + head) * c->D;
        if (c->ranges)
            orc_quantize_block_ranges(x, (long)c->H * c->D, c->bs, c->D, c->rel,
                                      c->ranges + (long)head * c->D,
                                      c->ranges + ((long)c->H + head) * c->D, codes, mins, scales);
        else
            orc_quantize_block(x, (long)c->H * c->D, c->bs, c->D, c->mode, c->rel, codes, mins,
                               scales);
        orc_histogram(codes, (long)c->bs * c->D, c->local[tid]);
    }
    free(codes); free(mins); free(scales);
}

/* Prefill histogram over the full blocks of a [n_full, H, D] tensor (kvcache.py:116-121). */
int orc_tokens_histogram_r(const float *tokens, int n_tok, int H, int D, int bs, int mode,
                           double rel, const float *ranges, uint64_t *hist, int n_threads);

int orc_tokens_histogram(const float *tokens, int n_tok, int H, int D, int bs, int mode,
                         double rel, uint64_t *hist, int n_threads)
{
    return orc_tokens_histogram_r(tokens, n_tok, H, D, bs, mode, rel, NULL, hist, n_threads);
}

int orc_tokens_histogram_r(const float *tokens, int n_tok, int H, int D, int bs, int mode,
                           double rel, const float *ranges, uint64_t *hist, int n_threads)
{
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    long nb = (long)(n_tok / bs) * H;
    hist_ctx c = {tokens, H, D, bs, mode, mode == 1 ? bs : D, rel, NULL, ranges};
    c.local = (uint64_t (*)[256])calloc((size_t)n_threads, sizeof(uint64_t[256]));
    parallel_for(nb, n_threads, hist_range, &c);
    memset(hist, 0, 256 * sizeof(uint64_t));
    for (int t = 0; t < n_threads; ++t)
        for (int s = 0; s < 256; ++s) hist[s] += c.local[t][s];
    free(c.local);
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Fetch (attention.py:59-188): decode inside the dot products          */
/* ------------------------------------------------------------------ */

static long extent_end(const uint32_t *offsets, long n_blocks, long b, long cursor)
{
    return b + 1 < n_blocks ? (long)offsets[b + 1] : cursor;
}

typedef struct {
    const uint8_t *arena; const uint32_t *offsets; long n_blocks, cursor, ctx;
    int H, D, bs; const uint8_t *lengths; const float *q; const float *w;
    float *scores; float *parts; int err;
} fetch_ctx;

static void kscore_range(long lo, long hi, int tid, void *p)
{
    fetch_ctx *c = (fetch_ctx *)p;
    int D = c->D, bs = c->bs;
    uint8_t *codes = (uint8_t *)malloc((size_t)bs * D);
    float *mins = (float *)malloc(sizeof(float) * D);
    float *scales = (float *)malloc(sizeof(float) * D);
    float *folded = (float *)malloc(sizeof(float) * D);
    for (long b = lo; b < hi; ++b) {
        uint32_t bi; int ns;
        long s0 = c->offsets[b], s1 = extent_end(c->offsets, c->n_blocks, b, c->cursor);
        int st = orc_decode_block(c->arena + s0, s1 - s0, D, D, c->lengths, codes, mins, scales, &bi, &ns);
        if (st || ns != bs) { c->err = st ? st : ORC_CODEC; continue; }
        int head = (int)(bi % (uint32_t)c->H);
        long t0 = (long)(bi / (uint32_t)c->H) * bs;
        const float *qh = c->q + (long)head * D;
        float base = 0.f;
        for (int j = 0; j < D; ++j) { folded[j] = scales[j] * qh[j]; base += mins[j] * qh[j]; }
        for (int r = 0; r < bs; ++r) {
            float acc = 0.f;
            for (int j = 0; j < D; ++j) acc += (float)codes[(long)r * D + j] * folded[j];
            c->scores[(long)head * c->ctx + t0 + r] = acc + base;
        }
    }
    free(codes); free(mins); free(scales); free(folded);
}

/* scores[h, t] for all compressed tokens + buffered tokens, x 1/sqrt(D)
 * (attention.py:59-109: codes @ (scale*q) + mins @ q, then * 1/sqrt(D)). */
int orc_k_scores(const uint8_t *arena, const uint32_t *offsets, long n_blocks, long cursor,
                 int H, int D, int bs, const uint8_t *lengths, const float *q,
                 const float *kbuf, int buffered, long ctx, float *scores, int n_threads)
{
    fetch_ctx c = {arena, offsets, n_blocks, cursor, ctx, H, D, bs, lengths, q, NULL, scores, NULL, ORC_OK};
    long compressed = (n_blocks / (H ? H : 1)) * bs;
    parallel_for(n_blocks, n_threads, kscore_range, &c);
    for (int t = 0; t < buffered; ++t)
        for (int h = 0; h < H; ++h) {
            float acc = 0.f;
            for (int j = 0; j < D; ++j) acc += kbuf[((long)t * H + h) * D + j] * q[(long)h * D + j];
            scores[(long)h * ctx + compressed + t] = acc;
        }
    float inv = (float)(1.0 / sqrt((double)D));
    for (long i = 0; i < (long)H * ctx; ++i) scores[i] *= inv;
    return c.err;
}

/* attention.py:168-173.  The reference's e.sum() is numpy's pairwise
 * summation (error ~ eps log n); a naive f32 running sum drifts by ~1e-4
 * relative over a 128K-token row, so the sum is accumulated in binary64 and
 * rounded once (closer to the exact sum than either). */
void orc_softmax_rows(const float *x, long rows, long cols, float *out)
{
    for (long r = 0; r < rows; ++r) {
        const float *xr = x + r * cols;
        float *o = out + r * cols;
        float m = xr[0];
        for (long j = 1; j < cols; ++j) if (xr[j] > m) m = xr[j];
        double s = 0.0;
        for (long j = 0; j < cols; ++j) { o[j] = expf(xr[j] - m); s += (double)o[j]; }
        const float sf = (float)s;
        for (long j = 0; j < cols; ++j) o[j] /= sf;
    }
}

static void vout_range(long lo, long hi, int tid, void *p)
{
    fetch_ctx *c = (fetch_ctx *)p;
    int D = c->D, bs = c->bs;
    float *part = c->parts + (long)tid * c->H * D;
    uint8_t *codes = (uint8_t *)malloc((size_t)bs * D);
    float *mins = (float *)malloc(sizeof(float) * bs);
    float *scales = (float *)malloc(sizeof(float) * bs);
    for (long b = lo; b < hi; ++b) {
        uint32_t bi; int ns;
        long s0 = c->offsets[b], s1 = extent_end(c->offsets, c->n_blocks, b, c->cursor);
        int st = orc_decode_block(c->arena + s0, s1 - s0, bs, D, c->lengths, codes, mins, scales, &bi, &ns);
        if (st || ns != bs) { c->err = st ? st : ORC_CODEC; continue; }
        int head = (int)(bi % (uint32_t)c->H);
        long t0 = (long)(bi / (uint32_t)c->H) * bs;
        const float *wr = c->w + (long)head * c->ctx + t0;
        float wm = 0.f;
        for (int r = 0; r < bs; ++r) {
            float a = wr[r] * scales[r];
            wm += wr[r] * mins[r];
            for (int j = 0; j < D; ++j) part[(long)head * D + j] += a * (float)codes[(long)r * D + j];
        }
        for (int j = 0; j < D; ++j) part[(long)head * D + j] += wm;
    }
    free(codes); free(mins); free(scales);
}

/* out[h, :] = sum over blocks ((w*scale) @ codes + w @ mins) + buffered
 * (attention.py:112-165; per-worker partials summed in worker order). */
int orc_v_output(const uint8_t *arena, const uint32_t *offsets, long n_blocks, long cursor,
                 int H, int D, int bs, const uint8_t *lengths, const float *w,
                 const float *vbuf, int buffered, long ctx, float *out, int n_threads)
{
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    fetch_ctx c = {arena, offsets, n_blocks, cursor, ctx, H, D, bs, lengths, NULL, w, NULL, NULL, ORC_OK};
    long compressed = (n_blocks / (H ? H : 1)) * bs;
    c.parts = (float *)calloc((size_t)n_threads * H * D, sizeof(float));
    parallel_for(n_blocks, n_threads, vout_range, &c);
    memset(out, 0, sizeof(float) * (size_t)H * D);
    for (int th = 0; th < n_threads; ++th)
        for (long i = 0; i < (long)H * D; ++i) out[i] += c.parts[(long)th * H * D + i];
    free(c.parts);
    for (int t = 0; t < buffered; ++t)
        for (int h = 0; h < H; ++h) {
            float wt = w[(long)h * ctx + compressed + t];
            for (int j = 0; j < D; ++j) out[(long)h * D + j] += wt * vbuf[((long)t * H + h) * D + j];
        }
    return c.err;
}

/* Materialise dequantised f32 tensors (kvcache.py:182-212): f64 dequant, f32 store. */
int orc_dequantize_arena(const uint8_t *arena, const uint32_t *offsets, long n_blocks, long cursor,
                         int H, int D, int bs, int mode, const uint8_t *lengths, float *out)
{
    int n_units = mode == 1 ? bs : D;
    uint8_t *codes = (uint8_t *)malloc((size_t)bs * D);
    float *mins = (float *)malloc(sizeof(float) * n_units);
    float *scales = (float *)malloc(sizeof(float) * n_units);
    int err = ORC_OK;
    for (long b = 0; b < n_blocks && !err; ++b) {
        uint32_t bi; int ns;
        long s0 = offsets[b], s1 = extent_end(offsets, n_blocks, b, cursor);
        err = orc_decode_block(arena + s0, s1 - s0, n_units, D, lengths, codes, mins, scales, &bi, &ns);
        if (err) break;
        int head = (int)(bi % (uint32_t)H);
        long t0 = (long)(bi / (uint32_t)H) * bs;
        for (int r = 0; r < bs; ++r)
            for (int c = 0; c < D; ++c) {
                int u = mode == 1 ? r : c;
                double v = (double)mins[u] + (double)codes[(long)r * D + c] * (double)scales[u];
                out[((t0 + r) * H + head) * (long)D + c] = (float)v;
            }
    }
    free(codes); free(mins); free(scales);
    return err;
}
