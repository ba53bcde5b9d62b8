"""Hugging Face ``transformers`` integration: a compressed KV cache whose decode
steps run the fused Huffman-decode + attention kernel (the
paper's model integration, PAPER.md:276, :490 — the reference package itself
ships no model integration).

    from paper_2509_00579_b200.hf_cache import KVCompCache, enable_kvcomp_attention
    enable_kvcomp_attention(model)                       # attn_implementation "kvcomp"
    cache = KVCompCache(model.config)                    # default K_BLOCK 0.05 / V_TOKEN 0.15
    out = model.generate(ids, past_key_values=cache, max_new_tokens=32)

Per layer, per batch row, the cache holds a device ``LayerCacheState``:

* prefill (the first ``update`` of a layer): ``LayerCacheState.prefill`` of the
  prompt's post-RoPE keys and values (Store: quantise -> histogram -> codebooks
  -> encode); the prompt itself attends densely (sdpa) to its own keys, as a
  prefill must;
* decode (``update`` with one new token): ``append_token`` into the growing
  cache (overflow events compress whole blocks, kvcache.py:150-177) and the
  layer's attention runs ``attention_batched`` / ``attention_gqa`` straight from
  the compressed arenas — the decompressed KV never exists in HBM;
* a multi-token ``update`` after prefill (chunked prefill, speculative
  verification) appends the tokens and returns the dequantised context so the
  model's own attention handles the causal block.

Constraints: unpadded batches (each row its own length is fine: rows are
independent states), head_dim 128 / block 64 for the fused kernels (other
shapes use the generic decode kernels), groups 1, 2 or 4 for the decode-once
GQA kernel.  The attention scale must be 1/sqrt(head_dim) (the reference's);
other scales are folded into q.
"""

from __future__ import annotations

import math
from typing import List, Optional

import torch
from transformers.cache_utils import Cache, CacheLayerMixin

from .attention import attention_batched, attention_gqa
from .kvcache import LayerCacheState
from .quantizer import QuantConfig, QuantMode

_LAST_DECODE = None  # the layer whose decode update ran last (its attention runs next)


class KVCompLayer(CacheLayerMixin):
    """One decoder layer's compressed cache (transformers CacheLayerMixin API)."""

    is_sliding = False
    is_compileable = False

    def __init__(self, layer_idx: int, cfg_k: QuantConfig, cfg_v: QuantConfig):
        super().__init__()
        self.layer_idx = layer_idx
        self.cfg_k, self.cfg_v = cfg_k, cfg_v
        self.states: Optional[List[LayerCacheState]] = None
        self.cumulative_length = 0
        self.is_initialized = False
        self.keys = self.values = None
        self.decode_pending = False
        self._desc = None
        self._ws = None

    def __repr__(self):
        return f"KVCompLayer(layer={self.layer_idx}, tokens={self.cumulative_length})"

    def lazy_initialization(self, key_states: torch.Tensor, value_states: torch.Tensor) -> None:
        self.dtype, self.device = key_states.dtype, key_states.device
        self.is_initialized = True

    def update(self, key_states: torch.Tensor, value_states: torch.Tensor, *args, **kwargs):
        global _LAST_DECODE
        if not self.is_initialized:
            self.lazy_initialization(key_states, value_states)
        B, H, T, D = key_states.shape
        self.decode_pending = False
        if self.states is None:
            # prefill: [B, H, T, D] -> per row [T, H, D]
            kk = key_states.detach().transpose(1, 2)
            vv = value_states.detach().transpose(1, 2)
            # the batch rows through the pipelined prefill (row b+1's pass A runs
            # while row b's codebooks are built on the host)
            self.states = LayerCacheState.prefill_many(
                [(kk[b].contiguous(), vv[b].contiguous()) for b in range(B)],
                self.cfg_k, self.cfg_v)
            self.cumulative_length = T
            return key_states, value_states
        if len(self.states) != B:
            raise ValueError("batch size changed after prefill")
        from .kvcache import _BatchDesc, append_batched
        if self._desc is None:
            self._desc = _BatchDesc()
        for t in range(T):  # the batch rows' token t in one device append
            append_batched(self.states, key_states[:, :, t], value_states[:, :, t],
                           desc_cache=self._desc)
        self.cumulative_length += T
        if T == 1:
            self.decode_pending = True
            _LAST_DECODE = self
            return key_states, value_states  # placeholders: the kvcomp attention ignores them
        # multi-token update: hand the model the whole (dequantised) context
        ks, vs = zip(*(st.fetch_dequantized() for st in self.states))
        k_full = torch.stack([k.values.transpose(0, 1) for k in ks]).to(key_states.dtype)
        v_full = torch.stack([v.values.transpose(0, 1) for v in vs]).to(value_states.dtype)
        return k_full, v_full

    def attend(self, query: torch.Tensor, scaling: Optional[float]) -> torch.Tensor:
        """query [B, Hq, 1, D] -> attention output [B, 1, Hq, D] from the arenas."""
        from .attention import _BatchDesc
        B, HQ, _, D = query.shape
        H = self.states[0].head_num
        q = query[:, :, 0, :].float()
        if scaling is not None and abs(scaling * math.sqrt(D) - 1.0) > 1e-6:
            q = q * (scaling * math.sqrt(D))
        if self._desc is None:
            self._desc = _BatchDesc()
        if HQ == H:
            out, _, _ = attention_batched(self.states, q.contiguous(), desc_cache=self._desc)
        else:
            out = attention_gqa(self.states, q.contiguous(), HQ // H, desc_cache=self._desc,
                                check=False)
        self.decode_pending = False
        return out.to(query.dtype).unsqueeze(1)

    # --- transformers CacheLayerMixin surface --------------------------------
    def get_mask_sizes(self, query_length: int):
        return self.cumulative_length + query_length, 0

    def get_seq_length(self) -> int:
        return self.cumulative_length

    def get_max_cache_shape(self) -> int:
        return -1

    def reset(self) -> None:
        self.states = None
        self.cumulative_length = 0
        self.decode_pending = False

    def offload(self):
        pass

    def prefetch(self):
        pass

    def reorder_cache(self, beam_idx: torch.LongTensor) -> None:
        idx = beam_idx.tolist()
        if idx != list(range(len(idx))):
            raise NotImplementedError("beam search reordering of compressed caches")

    def check(self) -> None:
        for st in self.states or []:
            st.check()


class KVCompCache(Cache):
    """transformers ``Cache`` holding every decoder layer's KV compressed."""

    def __init__(self, config, cfg_k: Optional[QuantConfig] = None,
                 cfg_v: Optional[QuantConfig] = None):
        cfg_k = cfg_k or QuantConfig(QuantMode.K_BLOCK)
        cfg_v = cfg_v or QuantConfig(QuantMode.V_TOKEN)
        text = config.get_text_config(decoder=True) if hasattr(config, "get_text_config") else config
        layers = [KVCompLayer(i, cfg_k, cfg_v) for i in range(text.num_hidden_layers)]
        super().__init__(layers=layers)

    def compression_stats(self):
        """(compressed bytes, equivalent fp16 bytes) over all layers and rows."""
        comp = orig = 0
        for layer in self.layers:
            for st in layer.states or []:
                comp += st.k_arena.size_bytes + st.v_arena.size_bytes + \
                    2 * st.buffered * st.head_num * st.head_dim * 4
                orig += 2 * st.context_len * st.head_num * st.head_dim * 2
        return comp, orig


def kvcomp_attention(module, query, key, value, attention_mask, scaling=None, dropout=0.0,
                     **kwargs):
    """Attention function registered as "kvcomp": single-token decode steps of a
    KVCompCache layer run the fused compressed-cache kernel; everything else
    (prefill, multi-token updates, models without the cache) runs sdpa."""
    layer = _LAST_DECODE
    if (layer is not None and layer.decode_pending and query.shape[2] == 1
            and layer.layer_idx == getattr(module, "layer_idx", None)):
        return layer.attend(query, scaling), None
    from transformers.integrations.sdpa_attention import sdpa_attention_forward
    return sdpa_attention_forward(module, query, key, value, attention_mask, scaling=scaling,
                                  dropout=dropout, **kwargs)


def enable_kvcomp_attention(model=None) -> None:
    """Register the "kvcomp" attention (and its sdpa-style mask) with transformers
    and switch `model` to it."""
    from transformers import AttentionInterface
    from transformers.masking_utils import AttentionMaskInterface, sdpa_mask
    AttentionInterface.register("kvcomp", kvcomp_attention)
    AttentionMaskInterface.register("kvcomp", sdpa_mask)
    if model is not None:
        if hasattr(model, "set_attn_implementation"):
            model.set_attn_implementation("kvcomp")
        else:
            model.config._attn_implementation = "kvcomp"
