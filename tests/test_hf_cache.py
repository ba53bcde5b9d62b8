"""transformers integration (hf_cache.py): a random-init Llama-shaped model
(head_dim 128, GQA group 2) decoding through KVCompCache must match sdpa over
the same cache dequantised (fetch_dequantized), i.e. the fused kernel computes
exactly "decompress then attend"; and generate() runs end to end."""
import pytest
import torch

transformers = pytest.importorskip("transformers")


def _model(kv_heads):
    from transformers import LlamaConfig, LlamaForCausalLM
    torch.manual_seed(0)
    cfg = LlamaConfig(vocab_size=512, hidden_size=512, intermediate_size=1024,
                      num_hidden_layers=2, num_attention_heads=4, num_key_value_heads=kv_heads,
                      head_dim=128, max_position_embeddings=4096)
    return LlamaForCausalLM(cfg).cuda().float().eval()


def test_kvcomp_cache_importable_cpu():
    from paper_2509_00579_b200 import hf_cache
    assert hasattr(hf_cache, "KVCompCache") and hasattr(hf_cache, "kvcomp_attention")


@pytest.mark.gpu
@pytest.mark.parametrize("kv_heads", [2, 4])
def test_decode_matches_sdpa_over_dequantised_cache(kv_heads):
    from transformers import DynamicCache
    from paper_2509_00579_b200.hf_cache import KVCompCache, enable_kvcomp_attention
    from paper_2509_00579_b200.hf_cache import KVCompLayer
    calls = []
    orig = KVCompLayer.attend
    KVCompLayer.attend = lambda self, q, s: calls.append(self.layer_idx) or orig(self, q, s)
    model = _model(kv_heads)
    enable_kvcomp_attention(model)
    ids = torch.randint(0, 512, (2, 200), device="cuda")
    nxt = torch.randint(0, 512, (2, 1), device="cuda")
    with torch.no_grad():
        cache = KVCompCache(model.config)
        model(ids, past_key_values=cache, use_cache=True)
        # reference cache: the same compressed prompt, dequantised, dense
        ref = DynamicCache(config=model.config)
        for li, layer in enumerate(cache.layers):
            ks, vs = zip(*(st.fetch_dequantized() for st in layer.states))
            k = torch.stack([x.values.transpose(0, 1) for x in ks])
            v = torch.stack([x.values.transpose(0, 1) for x in vs])
            ref.update(k, v, li)
        a = model(nxt, past_key_values=cache, use_cache=True).logits
        model.set_attn_implementation("sdpa")
        b = model(nxt, past_key_values=ref, use_cache=True).logits
    KVCompLayer.attend = orig
    assert calls == [0, 1]  # both layers' decode attention ran from the compressed arenas
    err = float((a - b).abs().max() / b.abs().max())
    assert err < 1e-4, err
    assert cache.get_seq_length() == 201
    comp, orig = cache.compression_stats()
    assert comp < orig


@pytest.mark.gpu
def test_generate_end_to_end():
    from paper_2509_00579_b200.hf_cache import KVCompCache, enable_kvcomp_attention
    model = _model(2)
    enable_kvcomp_attention(model)
    ids = torch.randint(0, 512, (1, 300), device="cuda")
    cache = KVCompCache(model.config)
    with torch.no_grad():
        out = model.generate(ids, past_key_values=cache, max_new_tokens=8, do_sample=False)
    assert out.shape == (1, 308)
    assert cache.get_seq_length() in (307, 308)
    for layer in cache.layers:
        layer.check()


@pytest.mark.gpu
def test_generate_bf16_across_an_overflow_event():
    """A bf16 model (the Llama default): prefill takes bf16 KV (stored as a
    2-byte original), and 100 decode tokens after a 300-token prompt cross one
    growing-cache overflow event (44 buffered + 100 > buffer 128)."""
    from paper_2509_00579_b200.hf_cache import KVCompCache, enable_kvcomp_attention
    model = _model(2).to(torch.bfloat16)
    enable_kvcomp_attention(model)
    ids = torch.randint(0, 512, (2, 300), device="cuda")
    cache = KVCompCache(model.config)
    with torch.no_grad():
        out = model.generate(ids, past_key_values=cache, max_new_tokens=100, do_sample=False)
    assert out.shape == (2, 400)
    for layer in cache.layers:
        layer.check()
        for st in layer.states:
            assert st.compressed_tokens == 384 and st.context_len in (399, 400)
    comp, orig = cache.compression_stats()
    assert comp < orig
