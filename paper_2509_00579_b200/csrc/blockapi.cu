// blockapi.cu — the reference's per-block codec surface on the device:
//   decode_slice / decode_slices  codec.py:141-226  -> kvc_decode_slices_tree
//   CompressedArena.append        codec.py:308-326  -> kvc_arena_append
//   CompressedArena.restore       codec.py:329-341  -> kvc_arena_restore
// (compress_block / encode_slice reuse kvc_encode_append, decompress_block
// is kvc_decode_blocks in fetch_generic.cu.)  These are the drop-in API's
// single-block entry points, not the hot path: the Store/Fetch kernels
// never materialise per-block objects.
#include <climits>

#include "common.cuh"

namespace {

// One thread per slice: the reference's branch-free array-tree walk
// (codec.py:158-173 / :197-217) -- the bit picks the child, the node's
// symbol is written at the output cursor, the cursor advances by is_symbol
// and the node index resets to the root after a symbol.  After bit_count
// bits the slice must have produced exactly out_len symbols with the walk
// back at the root; otherwise the lowest bad slice index is recorded.
__global__ void tree_decode_kernel(const uint8_t *__restrict__ bits, int packed, uint64_t n_bits,
                                   const int64_t *__restrict__ offsets,
                                   const int64_t *__restrict__ counts, int n,
                                   const int32_t *__restrict__ children,
                                   const int32_t *__restrict__ is_symbol,
                                   const uint8_t *__restrict__ symbols, int n_nodes, int out_len,
                                   uint8_t *__restrict__ out, int *__restrict__ bad) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int64_t off = offsets[s], cnt = counts[s];
    uint8_t *row = out + (long)s * out_len;
    if (off < 0 || cnt < 0 || (uint64_t)(off + cnt) > n_bits) {
        atomicMin(bad, s);
        return;
    }
    int32_t index = 0;
    int64_t write_pos = 0;
    bool ok = true;
    for (int64_t p = off; p < off + cnt; ++p) {
        const uint32_t bit = packed ? (bits[p >> 3] >> (7 - (p & 7))) & 1u : (bits[p] & 1u);
        index = children[2 * index + bit];
        if (index < 0 || index >= n_nodes) {  // malformed tree (the reference would IndexError)
            ok = false;
            break;
        }
        const int32_t sym_flag = is_symbol[index] & 1;
        if (write_pos < out_len) row[write_pos] = symbols[index];
        write_pos += sym_flag;
        index &= ~(-sym_flag);
    }
    if (!ok || write_pos != out_len || index != 0) atomicMin(bad, s);
}

// Serialised block image -> arena at the cursor (codec.py:308-326): capacity
// and 32-bit offset checks first (ArenaFullError leaves the arena unchanged),
// then a coalesced copy and the counter update.  One CTA.
__global__ void arena_append_kernel(const uint8_t *__restrict__ image, uint32_t nbytes,
                                    uint64_t payload_bits, uint64_t payload_bytes,
                                    uint8_t *__restrict__ arena, uint64_t capacity,
                                    uint32_t *__restrict__ offsets,
                                    kvc_arena_counters *__restrict__ counters) {
    __shared__ int s_ok;
    const uint64_t start = counters->cursor;
    if (threadIdx.x == 0) {
        s_ok = !(start + nbytes > capacity || start + nbytes > 0xFFFFFFFFull);
        if (!s_ok && !counters->err) counters->err = KVC_ERR_ARENA_FULL;
    }
    __syncthreads();
    if (!s_ok) return;
    for (uint32_t i = threadIdx.x; i < nbytes; i += blockDim.x) arena[start + i] = image[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        offsets[counters->n_blocks] = (uint32_t)start;
        counters->cursor = start + nbytes;
        counters->n_blocks += 1;
        counters->payload_bits += payload_bits;
        counters->payload_bytes += payload_bytes;
        if (nbytes > counters->max_extent) counters->max_extent = nbytes;
    }
}

// Counters of a restored arena (codec.py:329-341): a warp per block parses
// its extent exactly as _parse_block (codec.py:247-268) -- header fits, size
// a multiple of 4, metadata inside the extent, 0..3 bytes of padding -- and
// accumulates payload bits/bytes, slices and the largest extent.
__global__ void arena_restore_kernel(const uint8_t *__restrict__ arena, uint64_t size,
                                     const uint32_t *__restrict__ offsets, int n_blocks,
                                     int n_units, kvc_arena_counters *__restrict__ counters,
                                     unsigned long long *__restrict__ n_slices, int *err) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= n_blocks) return;
    const uint64_t start = offsets[warp];
    const uint64_t end = warp + 1 < n_blocks ? (uint64_t)offsets[warp + 1] : size;
    const int64_t len = (int64_t)end - (int64_t)start;
    bool ok = len >= 6 && (len & 3) == 0 && end <= size;
    uint32_t ns = 0;
    if (ok) {
        const uint8_t *b = arena + start;
        ns = (uint32_t)b[4] | ((uint32_t)b[5] << 8);
        ok = 6 + 2 * (int64_t)ns + 8 * (int64_t)n_units <= len;
    }
    if (!ok) {
        if (lane == 0) kvc_set_err(err, KVC_ERR_CODEC);
        return;
    }
    const uint8_t *cnt = arena + start + 6;
    unsigned long long bits = 0;
    for (uint32_t r = lane; r < ns; r += 32) bits += (uint32_t)cnt[2 * r] | ((uint32_t)cnt[2 * r + 1] << 8);
#pragma unroll
    for (int o = 16; o; o >>= 1) bits += __shfl_xor_sync(0xffffffffu, bits, o);
    if (lane == 0) {
        const unsigned long long pbytes = (bits + 7) / 8;
        const int64_t pad = len - (6 + 2 * (int64_t)ns + 8 * (int64_t)n_units) - (int64_t)pbytes;
        if (pad < 0 || pad > 3) {
            kvc_set_err(err, KVC_ERR_CODEC);
            return;
        }
        atomicAdd(reinterpret_cast<unsigned long long *>(&counters->payload_bits), bits);
        atomicAdd(reinterpret_cast<unsigned long long *>(&counters->payload_bytes), pbytes);
        atomicAdd(n_slices, (unsigned long long)ns);
        atomicMax(&counters->max_extent, (uint32_t)len);
    }
}

}  // namespace

extern "C" int kvc_decode_slices_tree(const uint8_t *bits_dev, int packed, uint64_t n_bits,
                                      const int64_t *offsets_dev, const int64_t *counts_dev,
                                      int n_slices, const int32_t *children_dev,
                                      const int32_t *is_symbol_dev, const uint8_t *symbols_dev,
                                      int n_nodes, int out_len, uint8_t *out_dev, int *bad_dev,
                                      void *stream) {
    if (n_slices < 0 || out_len < 0 || n_nodes < 1) return kvc_fail(KVC_ERR_CONFIG, "bad shape");
    if (n_slices == 0) return KVC_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    tree_decode_kernel<<<(n_slices + 127) / 128, 128, 0, s>>>(
        bits_dev, packed, n_bits, offsets_dev, counts_dev, n_slices, children_dev, is_symbol_dev,
        symbols_dev, n_nodes, out_len, out_dev, bad_dev);
    return kvc_check_launch("tree_decode_kernel");
}

extern "C" int kvc_arena_append(const uint8_t *image_dev, uint32_t nbytes, uint64_t payload_bits,
                                uint64_t payload_bytes, uint8_t *arena_dev, uint64_t capacity,
                                uint32_t *offsets_dev, kvc_arena_counters *counters_dev,
                                void *stream) {
    if (nbytes == 0 || (nbytes & 3)) return kvc_fail(KVC_ERR_CODEC, "block image must be a non-empty multiple of 4 bytes");
    arena_append_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        image_dev, nbytes, payload_bits, payload_bytes, arena_dev, capacity, offsets_dev,
        counters_dev);
    return kvc_check_launch("arena_append_kernel");
}

extern "C" int kvc_arena_restore(const uint8_t *arena_dev, uint64_t size,
                                 const uint32_t *offsets_dev, int n_blocks, int n_units,
                                 kvc_arena_counters *counters_dev, uint64_t *n_slices_dev,
                                 int *err_dev, void *stream) {
    if (n_blocks < 0 || n_units < 0) return kvc_fail(KVC_ERR_CONFIG, "bad shape");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    kvc_arena_counters init{};
    init.cursor = size;
    init.n_blocks = (uint64_t)n_blocks;
    KVC_CUDA_TRY(cudaMemcpyAsync(counters_dev, &init, sizeof(init), cudaMemcpyHostToDevice, s));
    KVC_CUDA_TRY(cudaMemsetAsync(n_slices_dev, 0, sizeof(uint64_t), s));
    if (n_blocks == 0) return KVC_OK;
    const int threads = 256, warps = threads / 32;
    arena_restore_kernel<<<(n_blocks + warps - 1) / warps, threads, 0, s>>>(
        arena_dev, size, offsets_dev, n_blocks, n_units, counters_dev,
        reinterpret_cast<unsigned long long *>(n_slices_dev), err_dev);
    return kvc_check_launch("arena_restore_kernel");
}
