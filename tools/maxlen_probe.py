import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2509_00579_b200 as kv
dev = torch.device('cuda', 0)
ck = kv.QuantConfig(kv.QuantMode.K_BLOCK, rel_quant_scale=1/255)
cv = kv.QuantConfig(kv.QuantMode.V_TOKEN, rel_quant_scale=1/255)
lens = []
for b in range(64):
    k = kv.generate_synthetic_device(kv.SyntheticSpec(8192, 32, 128, seed=b), dev)
    v = kv.generate_synthetic_device(kv.SyntheticSpec(8192, 32, 128, seed=b ^ 0x9E3779B9), dev)
    st = kv.LayerCacheState.prefill(k, v, ck, cv)
    lens.append((st.k_codebook.max_code_length, st.v_codebook.max_code_length))
print(lens)
print('states with codes > 12 bits:', sum(1 for a, b in lens if max(a, b) > 12))
