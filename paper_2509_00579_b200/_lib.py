"""ctypes binding of libkvcomp.so (the C ABI declared in include/kvcomp.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is present, every device entry point raises.  ``build()`` compiles the library
in-tree for sm_100a (nvcc cross-compiles without a GPU).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

from .errors import (ArenaFullError, CodebookError, CodecError, ConfigError, KvpackError,
                     TensorFormatError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KVC_LIB_PATH") or os.path.join(_HERE, "libkvcomp.so")
CSRC = os.path.join(_HERE, "csrc")

KVC_OK, KVC_ERR_CONFIG, KVC_ERR_TENSOR, KVC_ERR_CODEBOOK, KVC_ERR_CODEC, KVC_ERR_ARENA_FULL, \
    KVC_ERR_CUDA = range(7)
KVC_K_BLOCK, KVC_V_TOKEN, KVC_K_CHANNEL = 0, 1, 2
KVC_F16, KVC_F32, KVC_F64 = 0, 1, 2
LUT_BITS = 12


class CudaError(KvpackError, RuntimeError):
    """A CUDA runtime failure inside the library (no reference analogue)."""


_EXC = {
    KVC_ERR_CONFIG: ConfigError,
    KVC_ERR_TENSOR: TensorFormatError,
    KVC_ERR_CODEBOOK: CodebookError,
    KVC_ERR_CODEC: CodecError,
    KVC_ERR_ARENA_FULL: ArenaFullError,
    KVC_ERR_CUDA: CudaError,
}


class ArenaCounters(ctypes.Structure):
    _fields_ = [("cursor", ctypes.c_uint64), ("n_blocks", ctypes.c_uint64),
                ("payload_bits", ctypes.c_uint64), ("payload_bytes", ctypes.c_uint64),
                ("max_extent", ctypes.c_uint32), ("err", ctypes.c_int32)]


class CodebookTables(ctypes.Structure):
    _fields_ = [("words", ctypes.c_uint32 * 256), ("lengths", ctypes.c_uint8 * 256),
                ("lut", ctypes.c_uint32 * (1 << LUT_BITS)),
                ("fetch_lut", ctypes.c_uint32 * (1 << LUT_BITS)),
                ("fetch_lut_x", ctypes.c_uint32 * (1 << LUT_BITS)),
                ("lut13", ctypes.c_uint32 * (1 << 13)),
                ("first_code", ctypes.c_uint32 * 33),
                ("count", ctypes.c_uint32 * 33), ("first_index", ctypes.c_uint32 * 33),
                ("sorted_symbols", ctypes.c_uint8 * 256), ("fetch_syms", ctypes.c_int32),
                ("max_len", ctypes.c_int32), ("n_symbols", ctypes.c_int32),
                ("single_symbol", ctypes.c_int32)]


class SeqDesc(ctypes.Structure):
    _fields_ = [("k_arena", ctypes.c_void_p), ("k_offsets", ctypes.c_void_p),
                ("k_counters", ctypes.c_void_p), ("k_cb", ctypes.c_void_p),
                ("v_arena", ctypes.c_void_p), ("v_offsets", ctypes.c_void_p),
                ("v_counters", ctypes.c_void_p), ("v_cb", ctypes.c_void_p),
                ("k_buffer", ctypes.c_void_p), ("v_buffer", ctypes.c_void_p),
                ("n_chunks", ctypes.c_int32), ("buffered", ctypes.c_int32),
                ("stage_bytes_k", ctypes.c_int32), ("stage_bytes_v", ctypes.c_int32),
                ("k_max_len", ctypes.c_int32), ("v_max_len", ctypes.c_int32),
                ("live", ctypes.c_void_p)]


P = ctypes.c_void_p
I = ctypes.c_int
L = ctypes.c_long
D_ = ctypes.c_double
SZ = ctypes.c_size_t
U32 = ctypes.c_uint32
U64 = ctypes.c_uint64

SIGNATURES = {
    "kvc_version": (ctypes.c_char_p, []),
    "kvc_last_error": (ctypes.c_char_p, []),
    "kvc_codebook_lengths": (I, [P, I, P]),
    "kvc_codebook_build_tables": (I, [P, P]),
    "kvc_codebook_bytes": (SZ, []),
    "kvc_quantize": (I, [P, I, L, I, I, I, I, I, D_, P, P, P, P, P]),
    "kvc_encode_append": (I, [P, P, I, I, I, I, U32, I, I, I, I, P, P, U64, P, P, P, P]),
    "kvc_encode_workspace_bytes": (SZ, [I, I]),
    "kvc_store_append": (I, [P, P, I, L, I, I, I, I, I, I, I, D_, D_, P, U32, P, I, P, I, P, U64,
                             P, P, P, U64, P, P, P, SZ, P]),
    "kvc_store_workspace_bytes": (SZ, [I, I, I, I]),
    "kvc_store_hist": (I, [P, P, I, L, I, I, I, I, I, D_, D_, P, P, P]),
    "kvc_store_supported": (I, [I, I, I]),
    "kvc_store_prefill_supported": (I, [I, I, D_, D_]),
    "kvc_store_blk_hist_bytes": (SZ, [I, I]),
    "kvc_store_hist_blocks": (I, [P, P, I, L, I, I, I, I, I, D_, D_, P, P, P, P, P]),
    "kvc_store_codes_bytes": (SZ, [I, I]),
    "kvc_store_prefill": (I, [P, P, I, L, I, I, I, I, I, I, I, D_, D_, P, U32, P, I, P, I, P, U64,
                              P, P, P, U64, P, P, P, P, P, SZ, P]),
    "kvc_k_scores": (I, [P, I, I, I, I, P, P, L, P, P]),
    "kvc_softmax_rows": (I, [P, I, L, L, P]),
    "kvc_v_output": (I, [P, I, I, I, I, P, L, P, P, P, P]),
    "kvc_v_output_workspace_bytes": (SZ, [I, I, I]),
    "kvc_attention": (I, [P, P, I, I, I, I, I, P, P, P, L, P, SZ, P, P]),
    "kvc_attention_workspace_bytes": (SZ, [I, I, I, I, I]),
    "kvc_dequantize": (I, [P, I, I, I, I, I, P, P, P]),
    "kvc_dense_attention_f16": (I, [P, P, I, I, I, I, L, P, P, P, SZ, P]),
    "kvc_dense_workspace_bytes": (SZ, [I, I, I, I, L]),
    "kvc_decode_blocks": (I, [P, P, P, P, I, I, I, I, P, P, P, P, P, P]),
    "kvc_decode_slices_tree": (I, [P, I, U64, P, P, I, P, P, P, I, I, P, P, P]),
    "kvc_arena_append": (I, [P, U32, U64, U64, P, U64, P, P, P]),
    "kvc_arena_restore": (I, [P, U64, P, I, I, P, P, P, P]),
    "kvc_buffer_append": (I, [P, I, I, I, I, P, P, I, L, P, P]),
    "kvc_buffer_shift": (I, [P, I, I, I, I, I, I, P]),
    "kvc_set_live": (I, [P, I, I, P]),
    "kvc_vmm_granularity": (I, [I, P]),
    "kvc_vmm_reserve": (I, [SZ, P]),
    "kvc_vmm_free_va": (I, [U64, SZ]),
    "kvc_vmm_create": (I, [I, SZ, P]),
    "kvc_vmm_release": (I, [U64]),
    "kvc_vmm_map": (I, [U64, SZ, U64, I]),
    "kvc_vmm_unmap": (I, [U64, SZ]),
}

_lib = None


def build(verbose: bool = False) -> str:
    """Compile libkvcomp.so in-tree for sm_100a (nvcc; works without a GPU)."""
    cmd = ["make", "-C", CSRC, "-j8"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("libkvcomp build failed:\n" + out.stdout + out.stderr)
    if verbose:
        print(out.stdout)
    return LIB_PATH


def lib():
    """Load libkvcomp.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: the CUDA extension must be built (python -c "
                "'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        h = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(status: int, what: str = "") -> None:
    if status == KVC_OK:
        return
    msg = lib().kvc_last_error().decode(errors="replace")
    exc = _EXC.get(status, KvpackError)
    raise exc(f"{what}: {msg}" if what else msg)


def raise_device_error(code: int, what: str) -> None:
    if code:
        raise _EXC.get(int(code), KvpackError)(f"{what}: device reported status {int(code)}")


def exported_symbols():
    return list(SIGNATURES)
