"""CPU oracle for the KVComp Store/Fetch path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package, and only as the checker or
the CPU timing arm; the product package (``paper_2509_00579_b200``) never does.

It wraps ``oracle/kvcomp_oracle.c`` (a C restatement of the reference's
algorithm, built by ``oracle/Makefile`` into ``oracle/build/``) and mirrors the
reference's ``LayerCacheState`` lifecycle (kvcache.py:29-268) on top of it:
prefill -> histograms -> smoothed Huffman codebooks -> block encode/append,
buffered appends with overflow compression, and the fused fetch functions
(attention.py:59-188).  Pinned against fixtures produced by the reference
itself (tests/golden/make_golden.py); see tests/test_oracle_golden.py.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libkvcomp_oracle.so")
_lib = None

ORC_OK, ORC_CONFIG, ORC_CODEBOOK, ORC_CODEC, ORC_ARENA_FULL = 0, 1, 3, 4, 5
DEFAULT_REL = {"kblock": 0.05, "vtoken": 0.15}


class OracleError(RuntimeError):
    def __init__(self, status, what):
        super().__init__(f"oracle {what} failed with status {status}")
        self.status = status


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i, l, d = ctypes.c_int, ctypes.c_long, ctypes.c_double
        sig = {
            "orc_quantize_block": (i, [P, l, i, i, i, d, P, P, P]),
            "orc_histogram": (None, [P, l, P]),
            "orc_huffman_lengths": (i, [P, P]),
            "orc_smooth_histogram": (i, [P, i, P]),
            "orc_canonical_words": (i, [P, P]),
            "orc_block_size": (l, [P, i, i, i, P, P, P]),
            "orc_encode_block": (i, [P, i, i, P, P, i, ctypes.c_uint32, P, P, P, P]),
            "orc_decode_block": (i, [P, l, i, i, P, P, P, P, P, P]),
            "orc_compress_tokens": (i, [P, i, i, i, i, i, d, ctypes.c_uint32, P, P, l, P, P, P, i]),
            "orc_compress_tokens_shard": (i, [P, i, i, i, i, i, d, ctypes.c_uint32, i, i, P, P, P,
                                              l, P, P, P, i]),
            "orc_tokens_histogram": (i, [P, i, i, i, i, i, d, P, i]),
            "orc_tokens_histogram_r": (i, [P, i, i, i, i, i, d, P, P, i]),
            "orc_quantize_block_ranges": (i, [P, l, i, i, d, P, P, P, P, P]),
            "orc_k_scores": (i, [P, P, l, l, i, i, i, P, P, P, i, l, P, i]),
            "orc_softmax_rows": (None, [P, l, l, P]),
            "orc_v_output": (i, [P, P, l, l, i, i, i, P, P, P, i, l, P, i]),
            "orc_dequantize_arena": (i, [P, P, l, l, i, i, i, i, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _chk(st, what):
    if st != ORC_OK:
        raise OracleError(st, what)


# --------------------------------------------------------------------------
# Primitive restatements
# --------------------------------------------------------------------------

def quantize_block(x, mode, rel):
    """(bs, D) f32 block -> (codes u8, mins f32, scales f32); mode 'kblock'|'vtoken'."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    bs, D = x.shape
    m = 1 if mode == "vtoken" else 0
    n_units = bs if m else D
    codes = np.zeros((bs, D), np.uint8)
    mins = np.zeros(n_units, np.float32)
    scales = np.zeros(n_units, np.float32)
    _chk(lib().orc_quantize_block(_p(x), D, bs, D, m, float(rel), _p(codes), _p(mins), _p(scales)),
         "quantize")
    return codes, mins, scales


def histogram(codes):
    c = np.ascontiguousarray(codes, dtype=np.uint8).ravel()
    h = np.zeros(256, np.uint64)
    lib().orc_histogram(_p(c), c.size, _p(h))
    return h


def smooth_histogram(h, max_code):
    h = np.ascontiguousarray(h, dtype=np.uint64)
    out = np.zeros(256, np.uint64)
    _chk(lib().orc_smooth_histogram(_p(h), int(max_code), _p(out)), "smooth")
    return out


def huffman_lengths(h):
    h = np.ascontiguousarray(h, dtype=np.uint64)
    out = np.zeros(256, np.uint8)
    _chk(lib().orc_huffman_lengths(_p(h), _p(out)), "huffman")
    return out


def canonical_words(lengths):
    lengths = np.ascontiguousarray(lengths, dtype=np.uint8)
    out = np.zeros(256, np.uint32)
    _chk(lib().orc_canonical_words(_p(lengths), _p(out)), "canonical")
    return out


def encode_block(codes, mins, scales, block_index, lengths):
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    bs, D = codes.shape
    mins = np.ascontiguousarray(mins, dtype=np.float32)
    scales = np.ascontiguousarray(scales, dtype=np.float32)
    lengths = np.ascontiguousarray(lengths, dtype=np.uint8)
    words = canonical_words(lengths)
    out = np.zeros(6 + 2 * bs + 8 * mins.size + bs * D * 4 + 8, np.uint8)
    n = ctypes.c_long(0)
    _chk(lib().orc_encode_block(_p(codes), bs, D, _p(mins), _p(scales), mins.size, block_index,
                                _p(lengths), _p(words), _p(out), ctypes.byref(n)), "encode")
    return out[: n.value].tobytes()


def decode_block(extent, n_units, D, lengths, bs_hint=None):
    ext = np.frombuffer(bytes(extent), dtype=np.uint8)
    ns = int(ext[4]) | (int(ext[5]) << 8) if ext.size >= 6 else 0
    codes = np.zeros((max(ns, 1), D), np.uint8)
    mins = np.zeros(n_units, np.float32)
    scales = np.zeros(n_units, np.float32)
    bi = ctypes.c_uint32(0)
    nso = ctypes.c_int(0)
    lengths = np.ascontiguousarray(lengths, dtype=np.uint8)
    _chk(lib().orc_decode_block(_p(ext), ext.size, n_units, D, _p(lengths), _p(codes), _p(mins),
                                _p(scales), ctypes.byref(bi), ctypes.byref(nso)), "decode")
    return codes[:ns], mins, scales, bi.value


# --------------------------------------------------------------------------
# LayerCacheState mirror (kvcache.py:29-268)
# --------------------------------------------------------------------------

class OracleState:
    """CPU mirror of the reference LayerCacheState (K_BLOCK + V_TOKEN)."""

    def __init__(self, H, D, bs, buffer, rel_k, rel_v, k_lengths, v_lengths, itemsize=4,
                 n_threads=1, k_ranges=None):
        self.H, self.D, self.bs, self.buffer = H, D, bs, buffer
        # K_CHANNEL: float32 [2, H, D] whole-context (min, max) (kvcache.py:104-108)
        self.k_ranges = None if k_ranges is None else np.ascontiguousarray(k_ranges, np.float32)
        self.rel_k, self.rel_v = float(rel_k), float(rel_v)
        self.k_lengths = np.asarray(k_lengths, np.uint8).copy()
        self.v_lengths = np.asarray(v_lengths, np.uint8).copy()
        self.itemsize = itemsize
        self.n_threads = n_threads
        self.arena = {"k": bytearray(), "v": bytearray()}
        self.offsets = {"k": [], "v": []}
        self.payload_bits = {"k": 0, "v": 0}
        self.payload_bytes = {"k": 0, "v": 0}
        self.k_buf = np.zeros((buffer + 1, H, D), np.float32)
        self.v_buf = np.zeros((buffer + 1, H, D), np.float32)
        self.context_len = 0
        self.compressed_tokens = 0
        self.buffered = 0

    @staticmethod
    def max_code(rel):
        return int(math.ceil(1.0 / rel))

    @classmethod
    def prefill(cls, k, v, bs=64, buffer=None, rel_k=0.05, rel_v=0.15, codebooks=None,
                n_threads=1, k_mode="kblock"):
        itemsize = np.asarray(k).dtype.itemsize
        k = np.ascontiguousarray(k, dtype=np.float32)
        v = np.ascontiguousarray(v, dtype=np.float32)
        buffer = 2 * bs if buffer is None else buffer
        ctx, H, D = k.shape
        n_full = (ctx // bs) * bs
        ranges = None
        if k_mode == "kchannel":
            ranges = np.ascontiguousarray(np.stack([k.min(axis=0), k.max(axis=0)]), np.float32)
        if codebooks is None:
            hk = np.zeros(256, np.uint64)
            hv = np.zeros(256, np.uint64)
            if n_full:
                lib().orc_tokens_histogram_r(_p(k), n_full, H, D, bs, 0, rel_k,
                                             _p(ranges) if ranges is not None else None, _p(hk),
                                             n_threads)
                lib().orc_tokens_histogram(_p(v), n_full, H, D, bs, 1, rel_v, _p(hv), n_threads)
            kl = huffman_lengths(smooth_histogram(hk, cls.max_code(rel_k)))
            vl = huffman_lengths(smooth_histogram(hv, cls.max_code(rel_v)))
        else:
            kl, vl = codebooks
        st = cls(H, D, bs, buffer, rel_k, rel_v, kl, vl, itemsize, n_threads, k_ranges=ranges)
        if n_full:
            st._compress(k[:n_full], v[:n_full])
        r = ctx - n_full
        st.k_buf[:r] = k[n_full:]
        st.v_buf[:r] = v[n_full:]
        st.buffered = r
        st.context_len = ctx
        return st

    def _compress_one(self, which, tokens, mode, rel, lengths):
        n = tokens.shape[0]
        nb = (n // self.bs) * self.H
        arena = self.arena[which]
        n_units = self.bs if mode else self.D
        cap = len(arena) + nb * (6 + 2 * self.bs + 8 * n_units + self.bs * self.D * 4 + 4)
        buf = np.zeros(cap, np.uint8)
        buf[: len(arena)] = np.frombuffer(bytes(arena), np.uint8)
        cursor = ctypes.c_long(len(arena))
        offs = np.zeros(max(nb, 1), np.uint32)
        bits = np.zeros(max(nb, 1), np.uint64)
        tokens = np.ascontiguousarray(tokens, np.float32)
        ranges = self.k_ranges if (which == "k" and self.k_ranges is not None) else None
        _chk(lib().orc_compress_tokens_shard(_p(tokens), n, self.H, self.D, self.bs, mode, rel,
                                             self.compressed_tokens // self.bs, self.H, 0,
                                             _p(ranges) if ranges is not None else None,
                                             _p(lengths), _p(buf), -1, ctypes.byref(cursor),
                                             _p(offs), _p(bits), self.n_threads), "compress")
        self.arena[which] = bytearray(buf[: cursor.value].tobytes())
        self.offsets[which] += [int(o) for o in offs[:nb]]
        self.payload_bits[which] += int(bits[:nb].sum())
        self.payload_bytes[which] += int(((bits[:nb] + 7) // 8).sum())

    def _compress(self, k_tokens, v_tokens):
        self._compress_one("k", k_tokens, 0, self.rel_k, self.k_lengths)
        self._compress_one("v", v_tokens, 1, self.rel_v, self.v_lengths)
        self.compressed_tokens += k_tokens.shape[0]

    def append_token(self, k_vec, v_vec):
        self.k_buf[self.buffered] = np.asarray(k_vec, np.float32)
        self.v_buf[self.buffered] = np.asarray(v_vec, np.float32)
        self.buffered += 1
        self.context_len += 1
        if self.buffered > self.buffer:
            n = (self.buffered // self.bs) * self.bs
            self._compress(self.k_buf[:n].copy(), self.v_buf[:n].copy())
            rem = self.buffered - n
            if rem:
                self.k_buf[:rem] = self.k_buf[n: self.buffered]
                self.v_buf[:rem] = self.v_buf[n: self.buffered]
            self.buffered = rem

    # ----- arena views -----
    def arena_bytes(self, which):
        return bytes(self.arena[which])

    def block_offsets(self, which):
        return np.asarray(self.offsets[which], np.uint32)

    def _arena_args(self, which):
        a = np.frombuffer(bytes(self.arena[which]) + b"\0" * 16, np.uint8)
        o = np.asarray(self.offsets[which] or [0], np.uint32)
        return a, o, len(self.offsets[which]), len(self.arena[which])

    # ----- fetch -----
    def fused_k_scores(self, q):
        q = np.ascontiguousarray(q, np.float32)
        a, o, nb, cur = self._arena_args("k")
        scores = np.zeros((self.H, self.context_len), np.float32)
        kb = np.ascontiguousarray(self.k_buf)
        _chk(lib().orc_k_scores(_p(a), _p(o), nb, cur, self.H, self.D, self.bs,
                                _p(self.k_lengths), _p(q), _p(kb), self.buffered,
                                self.context_len, _p(scores), self.n_threads), "k_scores")
        return scores

    def fused_v_output(self, w):
        w = np.ascontiguousarray(w, np.float32)
        a, o, nb, cur = self._arena_args("v")
        out = np.zeros((self.H, self.D), np.float32)
        vb = np.ascontiguousarray(self.v_buf)
        _chk(lib().orc_v_output(_p(a), _p(o), nb, cur, self.H, self.D, self.bs,
                                _p(self.v_lengths), _p(w), _p(vb), self.buffered,
                                self.context_len, _p(out), self.n_threads), "v_output")
        return out

    def attention_step(self, q):
        s = self.fused_k_scores(q)
        w = softmax_rows(s)
        return self.fused_v_output(w), s

    def fetch_dequantized(self):
        outs = []
        for which, mode, lengths, buf in (("k", 0, self.k_lengths, self.k_buf),
                                          ("v", 1, self.v_lengths, self.v_buf)):
            a, o, nb, cur = self._arena_args(which)
            out = np.zeros((self.context_len, self.H, self.D), np.float32)
            _chk(lib().orc_dequantize_arena(_p(a), _p(o), nb, cur, self.H, self.D, self.bs, mode,
                                            _p(lengths), _p(out)), "dequantize")
            out[self.compressed_tokens:] = buf[: self.buffered]
            outs.append(out)
        return outs[0], outs[1]

    def stats(self):
        """bench.py:77-95 counters: (original, compressed, metadata, payload_bits, quantized)."""
        vals = self.context_len * self.H * self.D
        original = 2 * vals * self.itemsize
        pbytes = self.payload_bytes["k"] + self.payload_bytes["v"]
        pbits = self.payload_bits["k"] + self.payload_bits["v"]
        bufb = 2 * self.buffered * self.H * self.D * self.itemsize
        arena = len(self.arena["k"]) + len(self.arena["v"])
        nblk = len(self.offsets["k"]) + len(self.offsets["v"])
        meta = (arena - pbytes) + 4 * nblk + 512
        quant = 2 * self.compressed_tokens * self.H * self.D
        return original, pbytes + bufb, meta, pbits, quant

    def compression_ratio(self):
        o, c, m, _, _ = self.stats()
        return o / (c + m)


def compress_shard(tokens, bs, mode, rel, lengths, H_total, head_base, chunk_base=0,
                   n_threads=1):
    """Encode a head shard [n, H_local, D] into (arena bytes, offsets) with global
    block indices."""
    tokens = np.ascontiguousarray(tokens, np.float32)
    n, H, D = tokens.shape
    m = 1 if mode == "vtoken" else 0
    nb = (n // bs) * H
    n_units = bs if m else D
    buf = np.zeros(nb * (6 + 2 * bs + 8 * n_units + bs * D * 4 + 4) + 16, np.uint8)
    cursor = ctypes.c_long(0)
    offs = np.zeros(max(nb, 1), np.uint32)
    bits = np.zeros(max(nb, 1), np.uint64)
    lengths = np.ascontiguousarray(lengths, np.uint8)
    _chk(lib().orc_compress_tokens_shard(_p(tokens), n, H, D, bs, m, float(rel), chunk_base,
                                         H_total, head_base, None, _p(lengths), _p(buf), -1,
                                         ctypes.byref(cursor), _p(offs), _p(bits), n_threads),
         "compress_shard")
    return buf[: cursor.value].tobytes(), offs[:nb].copy()


def tokens_histogram(tokens, bs, mode, rel, n_threads=1):
    tokens = np.ascontiguousarray(tokens, np.float32)
    n, H, D = tokens.shape
    h = np.zeros(256, np.uint64)
    _chk(lib().orc_tokens_histogram(_p(tokens), (n // bs) * bs, H, D, bs,
                                    1 if mode == "vtoken" else 0, float(rel), _p(h), n_threads),
         "histogram")
    return h


def softmax_rows(x):
    x = np.ascontiguousarray(x, np.float32)
    out = np.zeros_like(x)
    rows = x.shape[0] if x.ndim > 1 else 1
    lib().orc_softmax_rows(_p(x), rows, x.shape[-1], _p(out))
    return out


def generate_synthetic(context_len, head_num, head_dim, seed=0, outlier_fraction=0.05,
                       outlier_magnitude=8.0, base_std=1.0):
    """Restatement of tensor_io.py:142-157 (PCG64 streams, f32 normal, outlier channels)."""
    mask_rng = np.random.default_rng([seed, 0x6F75746C])
    outliers = mask_rng.random((head_num, head_dim)) < outlier_fraction
    vrng = np.random.default_rng([seed, 0x76616C73])
    vals = vrng.standard_normal((context_len, head_num, head_dim), dtype=np.float32)
    vals *= np.float32(base_std)
    vals[:, outliers] *= np.float32(outlier_magnitude)
    return vals
