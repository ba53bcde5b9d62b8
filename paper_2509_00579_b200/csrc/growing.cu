// growing.cu — device bookkeeping of the growing cache (kvcache.py:150-177)
// for sync-free decode loops.  The f32 token buffers and the live
// {n_chunks, buffered} pair of each state stay on the device:
//   kvc_buffer_append : append_token's buffer write for a batch of states
//                       (one launch per layer step), buffered += 1;
//   kvc_buffer_shift  : after an overflow event compressed rows [0, n), move
//                       the remainder to the front and publish the new
//                       {n_chunks, buffered} (kvcache.py:168-177).
// The host keeps deterministic mirrors of both counts (it knows how many
// tokens it appended), so it never reads them back; the fetch kernels read
// the live pair through kvc_seq_desc.live.
#include <algorithm>

#include "common.cuh"

namespace {

template <typename T>
__global__ void buffer_append_kernel(const kvc_seq_desc *__restrict__ seqs, int HD, int cap_rows,
                                     const T *__restrict__ k_rows, const T *__restrict__ v_rows,
                                     long seq_stride, int *err) {
    const int s = blockIdx.x;
    const kvc_seq_desc sd = seqs[s];
    int32_t *live = const_cast<int32_t *>(sd.live);
    const int b = live[1];
    // default error word: the state's K arena counters (raised by check())
    if (err == nullptr) err = &const_cast<kvc_arena_counters *>(sd.k_counters)->err;
    if (b < 0 || b >= cap_rows) {
        if (threadIdx.x == 0) kvc_set_err(err, KVC_ERR_CODEC);
        return;
    }
    float *kb = const_cast<float *>(sd.k_buffer) + (long)b * HD;
    float *vb = const_cast<float *>(sd.v_buffer) + (long)b * HD;
    const T *kr = k_rows + s * seq_stride, *vr = v_rows + s * seq_stride;
    bool finite = true;
    for (int i = threadIdx.x; i < HD; i += blockDim.x) {
        const float kx = kvc_load(kr + i), vx = kvc_load(vr + i);
        finite &= isfinite(kx) && isfinite(vx);
        kb[i] = kx;
        vb[i] = vx;
    }
    // non-finite tokens are rejected (kvcache.py:162-163): recorded here,
    // raised by the host's next check (the validating host path raises now)
    if (!__syncthreads_and(finite) && threadIdx.x == 0) kvc_set_err(err, KVC_ERR_CODEC);
    if (threadIdx.x == 0) live[1] = b + 1;
}

__global__ void buffer_shift_kernel(const kvc_seq_desc *__restrict__ seqs, int HD, int n_rows,
                                    int rem, int n_chunks) {
    const int s = blockIdx.y;
    const kvc_seq_desc sd = seqs[s];
    float *kb = const_cast<float *>(sd.k_buffer), *vb = const_cast<float *>(sd.v_buffer);
    const long total = (long)rem * HD;
    // rows [n_rows, n_rows + rem) -> [0, rem); rem < n_rows, so no overlap
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
         i += (long)gridDim.x * blockDim.x) {
        kb[i] = kb[(long)n_rows * HD + i];
        vb[i] = vb[(long)n_rows * HD + i];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        int32_t *live = const_cast<int32_t *>(sd.live);
        live[0] = n_chunks;
        live[1] = rem;
    }
}

__global__ void set_live_kernel(int32_t *live, int n_chunks, int buffered) {
    live[0] = n_chunks;
    live[1] = buffered;
}

}  // namespace

extern "C" int kvc_set_live(int32_t *live_dev, int n_chunks, int buffered, void *stream) {
    if (n_chunks < 0 || buffered < 0) return kvc_fail(KVC_ERR_CONFIG, "bad live counts");
    set_live_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(live_dev, n_chunks, buffered);
    return kvc_check_launch("set_live_kernel");
}

extern "C" int kvc_buffer_append(const kvc_seq_desc *seqs_dev, int n_seqs, int H, int D,
                                 int cap_rows, const void *k_rows_dev, const void *v_rows_dev,
                                 int x_dtype, long seq_stride, int *err_dev, void *stream) {
    if (n_seqs < 1 || H < 1 || D < 1 || cap_rows < 1) return kvc_fail(KVC_ERR_CONFIG, "bad shape");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int HD = H * D, threads = HD >= 1024 ? 1024 : ((HD + 31) / 32) * 32;
    if (x_dtype == KVC_F32)
        buffer_append_kernel<float><<<n_seqs, threads, 0, s>>>(
            seqs_dev, HD, cap_rows, static_cast<const float *>(k_rows_dev),
            static_cast<const float *>(v_rows_dev), seq_stride, err_dev);
    else if (x_dtype == KVC_F16)
        buffer_append_kernel<__half><<<n_seqs, threads, 0, s>>>(
            seqs_dev, HD, cap_rows, static_cast<const __half *>(k_rows_dev),
            static_cast<const __half *>(v_rows_dev), seq_stride, err_dev);
    else
        return kvc_fail(KVC_ERR_TENSOR, "unsupported dtype");
    return kvc_check_launch("buffer_append_kernel");
}

extern "C" int kvc_buffer_shift(const kvc_seq_desc *seqs_dev, int n_seqs, int H, int D,
                                int n_rows, int rem, int n_chunks, void *stream) {
    if (n_seqs < 1 || rem < 0 || (rem > 0 && rem >= n_rows))
        return kvc_fail(KVC_ERR_CONFIG, "bad buffer shift");
    const long total = (long)rem * H * D;
    const int blocks = (int)std::max(1L, std::min(64L, (total + 255) / 256));
    buffer_shift_kernel<<<dim3(blocks, n_seqs), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        seqs_dev, H * D, n_rows, rem, n_chunks);
    return kvc_check_launch("buffer_shift_kernel");
}
