// host.cu — host-side pieces of the C ABI: status/error strings and the
// Huffman codebook builder (the paper builds the codebook on the CPU from
// the GPU histogram).
//
// Behaviour restated from the reference:
//   smooth_histogram      codebook.py:83-89
//   _huffman_lengths      codebook.py:102-125  (ties by (weight, lowest symbol))
//   _canonical_words      codebook.py:128-141  (order (length, symbol))
//   codebook_from_lengths codebook.py:179-208  (Kraft equality, 32-bit cap,
//                                              1-symbol books use a 1-bit code)
#include <cstdio>
#include <cstring>
#include <queue>
#include <string>
#include <vector>

#include "common.cuh"

static thread_local std::string g_last_error;

int kvc_fail(int status, const char *msg) {
    g_last_error = msg ? msg : "";
    return status;
}

int kvc_fail_cuda(cudaError_t e, const char *what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return KVC_ERR_CUDA;
}

int kvc_check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return kvc_fail_cuda(e, what);
    return KVC_OK;
}

extern "C" const char *kvc_version(void) { return "kvcomp-b200 0.1 (sm_100a)"; }
extern "C" const char *kvc_last_error(void) { return g_last_error.c_str(); }
extern "C" size_t kvc_codebook_bytes(void) { return sizeof(kvc_codebook_dev); }

namespace {
struct Node {
    uint64_t w;
    int low;
    int id;
};
struct NodeGreater {
    bool operator()(const Node &a, const Node &b) const {
        return a.w != b.w ? a.w > b.w : a.low > b.low;
    }
};
}  // namespace

extern "C" int kvc_codebook_lengths(const uint64_t *hist, int max_code, uint8_t *lengths_out) {
    if (!hist || !lengths_out) return kvc_fail(KVC_ERR_CONFIG, "null argument");
    uint64_t h[256];
    for (int s = 0; s < 256; ++s) h[s] = hist[s];
    if (max_code >= 0) {
        if (max_code > 255) return kvc_fail(KVC_ERR_CODEBOOK, "max_code outside [0, 255]");
        for (int s = 0; s <= max_code; ++s) h[s] += 1;
    }
    std::memset(lengths_out, 0, 256);
    int present = 0, only = -1;
    for (int s = 0; s < 256; ++s)
        if (h[s]) { ++present; only = s; }
    if (!present) return kvc_fail(KVC_ERR_CODEBOOK, "cannot build a codebook from an empty histogram");
    if (present == 1) {
        lengths_out[only] = 1;
        return KVC_OK;
    }
    std::priority_queue<Node, std::vector<Node>, NodeGreater> pq;
    std::vector<int> parent(512, -1);
    for (int s = 0; s < 256; ++s)
        if (h[s]) pq.push(Node{h[s], s, s});
    int next = 256;
    while (pq.size() > 1) {
        Node a = pq.top(); pq.pop();
        Node b = pq.top(); pq.pop();
        int id = next++;
        parent[a.id] = id;
        parent[b.id] = id;
        pq.push(Node{a.w + b.w, a.low < b.low ? a.low : b.low, id});
    }
    for (int s = 0; s < 256; ++s) {
        if (!h[s]) continue;
        int d = 0;
        for (int p = parent[s]; p >= 0; p = parent[p]) ++d;
        if (d > 32) return kvc_fail(KVC_ERR_CODEBOOK, "code length exceeds the 32-bit cap");
        lengths_out[s] = (uint8_t)d;
    }
    return KVC_OK;
}

// Fused-fetch LUT (see kvcomp.h): two symbols per 12-bit window when every
// code is <= 6 bits (the second code then always fits the remaining bits).
static void build_fetch_lut(kvc_codebook_dev *t) {
    const int pair = t->max_len <= 6;
    t->fetch_syms = pair ? 2 : 1;
    for (uint32_t i = 0; i < (1u << KVC_LUT_BITS); ++i) {
        uint32_t e0 = t->lut[i];
        uint32_t l0 = (e0 >> 8) & 0xFF, s0 = e0 & 0xFF;
        if (!l0 || t->max_len > KVC_LUT_BITS) {
            t->fetch_lut[i] = 0;
            continue;
        }
        if (pair) {
            uint32_t rest = (i << l0) & ((1u << KVC_LUT_BITS) - 1);
            uint32_t e1 = t->lut[rest];
            uint32_t l1 = (e1 >> 8) & 0xFF, s1 = e1 & 0xFF;
            t->fetch_lut[i] = (l0 + l1) | (s0 << 16) | (s1 << 24);
        } else {
            t->fetch_lut[i] = l0 | (s0 << 16);
        }
    }
    for (uint32_t i = 0; i < (1u << KVC_LUT_BITS); ++i) t->fetch_lut_x[i ^ ((i >> 7) & 31u)] = t->fetch_lut[i];
}

extern "C" int kvc_codebook_build_tables(const uint8_t *lengths, kvc_codebook_dev *t) {
    if (!lengths || !t) return kvc_fail(KVC_ERR_CONFIG, "null argument");
    std::memset(t, 0, sizeof(*t));
    int present = 0, only = -1, max_len = 0;
    for (int s = 0; s < 256; ++s) {
        if (!lengths[s]) continue;
        ++present;
        only = s;
        if (lengths[s] > max_len) max_len = lengths[s];
    }
    if (!present) return kvc_fail(KVC_ERR_CODEBOOK, "no symbols present in code-length table");
    if (max_len > 32) return kvc_fail(KVC_ERR_CODEBOOK, "code length exceeds the 32-bit cap");
    std::memcpy(t->lengths, lengths, 256);
    t->max_len = max_len;
    t->n_symbols = present;
    if (present == 1) {
        if (lengths[only] != 1) return kvc_fail(KVC_ERR_CODEBOOK, "single-symbol codebooks must use a 1-bit code");
        // Degenerate tree: both root branches reach the leaf (codebook.py:149-154).
        t->single_symbol = 1;
        t->words[only] = 0;
        for (int i = 0; i < (1 << KVC_LUT_BITS); ++i) t->lut[i] = (uint32_t)only | (1u << 8);
        t->first_code[1] = 0;
        t->count[1] = 2;  // both 1-bit patterns decode to the symbol
        t->first_index[1] = 0;
        t->sorted_symbols[0] = (uint8_t)only;
        t->sorted_symbols[1] = (uint8_t)only;
        build_fetch_lut(t);
        float f = (float)only;
        uint32_t fb;
        std::memcpy(&fb, &f, 4);
        for (int i = 0; i < (1 << 13); ++i) t->lut13[i] = fb | 1u;
        return KVC_OK;
    }
    uint64_t kraft = 0;
    for (int s = 0; s < 256; ++s)
        if (lengths[s]) kraft += 1ull << (32 - lengths[s]);
    if (kraft != (1ull << 32)) return kvc_fail(KVC_ERR_CODEBOOK, "code lengths violate the Kraft equality");
    // Canonical assignment in (length, symbol) order.
    uint64_t code = 0;
    int prev = 0, idx = 0;
    for (int len = 1; len <= 32; ++len) {
        for (int s = 0; s < 256; ++s) {
            if (lengths[s] != len) continue;
            if (prev) code <<= (len - prev);
            prev = len;
            if (t->count[len] == 0) {
                t->first_code[len] = (uint32_t)code;
                t->first_index[len] = (uint32_t)idx;
            }
            t->count[len]++;
            t->words[s] = (uint32_t)code;
            t->sorted_symbols[idx++] = (uint8_t)s;
            ++code;
        }
    }
    // 12-bit primary LUT: sym | len << 8 for every code of length <= 12.
    for (int s = 0; s < 256; ++s) {
        int l = lengths[s];
        if (!l || l > KVC_LUT_BITS) continue;
        uint32_t lo = t->words[s] << (KVC_LUT_BITS - l);
        uint32_t hi = (t->words[s] + 1) << (KVC_LUT_BITS - l);
        for (uint32_t i = lo; i < hi; ++i) t->lut[i] = (uint32_t)s | ((uint32_t)l << 8);
    }
    build_fetch_lut(t);
    if (max_len <= 13) {  // the fused single-symbol fetch over 13-bit windows (fine scales)
        for (int s = 0; s < 256; ++s) {
            const int l = lengths[s];
            if (!l) continue;
            float f = (float)s;
            uint32_t fb;
            std::memcpy(&fb, &f, 4);
            const uint32_t lo = t->words[s] << (13 - l), hi = (t->words[s] + 1) << (13 - l);
            for (uint32_t i = lo; i < hi; ++i) t->lut13[i] = fb | (uint32_t)l;
        }
    }
    return KVC_OK;
}
