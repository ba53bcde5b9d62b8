"""Pin the CPU oracle (oracle/) against vectors produced by the reference itself."""
import numpy as np
import pytest

import oracle
from golden_cases import CASES, load, max_relative_error, unpack_cfg


@pytest.fixture(scope="module")
def kats():
    return load("kats")


def test_kat_quantize_unit(kats):
    codes, mins, scales = oracle.quantize_block(np.array([[0], [1], [2], [3]], np.float32),
                                                "kblock", 0.5)
    assert codes.ravel().tolist() == kats["kat_quant_codes"].tolist()
    assert [float(mins[0]), float(scales[0])] == kats["kat_quant_meta"].tolist()


def test_kat_codebook(kats):
    h = np.zeros(256, np.uint64)
    h[:4] = [4, 2, 1, 1]
    assert np.array_equal(oracle.huffman_lengths(h), kats["kat_cb_lengths"])
    assert np.array_equal(oracle.canonical_words(kats["kat_cb_lengths"]), kats["kat_cb_words"])


def test_kat_random_histograms(kats):
    for h, ln in zip(kats["kat_hists"], kats["kat_hist_lengths"]):
        assert np.array_equal(oracle.huffman_lengths(h), ln)


def test_kat_slice_encode(kats):
    blk = oracle.encode_block(np.array([[0, 1, 2, 3]], np.uint8), np.zeros(4, np.float32),
                              np.zeros(4, np.float32), 0, kats["kat_cb_lengths"])
    payload = np.frombuffer(blk, np.uint8)[6 + 2 + 32:]
    n = int(kats["kat_slice_count"])
    assert int.from_bytes(blk[6:8], "little") == n
    assert payload[: (n + 7) // 8].tolist() == kats["kat_slice_bytes"].tolist()


def test_kat_quant_grids(kats):
    for i, rel in enumerate(kats["kat_grid_rel"]):
        x = kats["kat_grid_x"][i]
        c, m, s = oracle.quantize_block(x, "kblock", rel)
        assert np.array_equal(c, kats["kat_grid_kcodes"][i])
        assert np.array_equal(m.view(np.uint32), kats["kat_grid_kmins"][i].view(np.uint32))
        assert np.array_equal(s.view(np.uint32), kats["kat_grid_kscales"][i].view(np.uint32))
        c, m, s = oracle.quantize_block(x, "vtoken", rel)
        assert np.array_equal(c, kats["kat_grid_vcodes"][i])
        assert np.array_equal(m.view(np.uint32), kats["kat_grid_vmins"][i].view(np.uint32))
        assert np.array_equal(s.view(np.uint32), kats["kat_grid_vscales"][i].view(np.uint32))


def _replay(g, n_threads=1):
    ctx, H, D, bs, buffer, appended, rel_k, rel_v = unpack_cfg(g)
    cbs = (g["inject_k"], g["inject_v"]) if "inject_k" in g else None
    st = oracle.OracleState.prefill(g["k_in"], g["v_in"], bs=bs, buffer=buffer, rel_k=rel_k,
                                    rel_v=rel_v, codebooks=cbs, n_threads=n_threads,
                                    k_mode=str(g.get("k_mode", "kblock")))
    if "k_ranges" in g:
        assert np.array_equal(st.k_ranges, g["k_ranges"])
    return st


def _check_state(st, g, prefix):
    for w in ("k", "v"):
        assert np.array_equal(st.k_lengths if w == "k" else st.v_lengths, g[prefix + w + "_lengths"])
        assert st.arena_bytes(w) == g[prefix + w + "_arena"].tobytes()
        assert np.array_equal(st.block_offsets(w), g[prefix + w + "_offsets"])
    c = g[prefix + "counters"]
    assert [st.context_len, st.compressed_tokens, st.buffered] == c[:3].tolist()
    assert [st.payload_bits["k"], st.payload_bytes["k"]] == c[3:5].tolist()
    assert [st.payload_bits["v"], st.payload_bytes["v"]] == c[6:8].tolist()
    assert list(st.stats()) == g[prefix + "stats"].tolist()
    assert st.compression_ratio() == pytest.approx(float(g[prefix + "ratio"]), rel=1e-12)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("n_threads", [1, 3])
def test_golden_store(case, n_threads):
    g = load(case)
    ctx, H, D, bs, buffer, appended, rel_k, rel_v = unpack_cfg(g)
    if "k_codes" in g and str(g.get("k_mode", "kblock")) == "kblock":
        for b in range(g["k_codes"].shape[0]):
            chunk, head = divmod(b, H)
            xk = g["k_in"][chunk * bs:(chunk + 1) * bs, head].astype(np.float32)
            xv = g["v_in"][chunk * bs:(chunk + 1) * bs, head].astype(np.float32)
            c, m, s = oracle.quantize_block(xk, "kblock", rel_k)
            assert np.array_equal(c, g["k_codes"][b])
            assert np.array_equal(m, g["k_mins"][b]) and np.array_equal(s, g["k_scales"][b])
            c, m, s = oracle.quantize_block(xv, "vtoken", rel_v)
            assert np.array_equal(c, g["v_codes"][b])
            assert np.array_equal(m, g["v_mins"][b]) and np.array_equal(s, g["v_scales"][b])
        assert np.array_equal(oracle.histogram(g["k_codes"]), g["k_hist"])
        assert np.array_equal(oracle.histogram(g["v_codes"]), g["v_hist"])
    st = _replay(g, n_threads)
    _check_state(st, g, "pre_")
    for t in range(appended):
        st.append_token(g["k_app"][t], g["v_app"][t])
    _check_state(st, g, "fin_")
    assert np.array_equal(st.k_buf[: st.buffered], g["fin_k_buffer"])


@pytest.mark.parametrize("case", CASES)
def test_golden_fetch(case):
    g = load(case)
    st = _replay(g)
    for t in range(int(g["cfg"][5])):
        st.append_token(g["k_app"][t], g["v_app"][t])
    for i in range(g["q"].shape[0]):
        out, scores = st.attention_step(g["q"][i])
        # reference bar: test_attention.py / C4 (<= 1e-5, normalised by max|ref|)
        assert max_relative_error(scores, g["att_scores"][i]) <= 1e-5
        assert max_relative_error(out, g["att_out"][i]) <= 1e-5
    assert max_relative_error(st.fused_v_output(g["w"]), g["vout_w"]) <= 1e-5
    kd, vd = st.fetch_dequantized()
    assert np.array_equal(kd, g["deq_k"]) and np.array_equal(vd, g["deq_v"])


def test_decode_roundtrip_and_corruption():
    g = load("c_fp16_d128")
    st = _replay(g)
    arena = st.arena_bytes("k")
    offs = st.block_offsets("k").tolist() + [len(arena)]
    codes, mins, scales, bi = oracle.decode_block(arena[offs[0]:offs[1]], 128, 128, st.k_lengths)
    assert np.array_equal(codes, g["k_codes"][0]) and bi == 0
    bad = bytearray(arena[offs[0]:offs[1]])
    bad[6] ^= 0x01   # perturb slice 0's bit count
    with pytest.raises(oracle.OracleError):
        oracle.decode_block(bytes(bad), 128, 128, st.k_lengths)


def test_synthetic_generator_matches_reference_inputs():
    g = load("c_fp16_d128")
    ctx, H, D = (int(x) for x in g["cfg"][:3])
    k = oracle.generate_synthetic(ctx + int(g["cfg"][5]), H, D, seed=3)
    v = oracle.generate_synthetic(ctx + int(g["cfg"][5]), H, D, seed=3 ^ 0x9E3779B9)
    assert np.array_equal(k[:ctx].astype(np.float16), g["k_in"])
    assert np.array_equal(v[:ctx].astype(np.float16), g["v_in"])
    assert np.array_equal(k[ctx:], g["k_app"])


def _digest_check(st, d):
    import hashlib
    for w in ("k", "v"):
        assert hashlib.sha256(st.arena_bytes(w)).hexdigest() == d[w + "_arena_sha256"]
        assert hashlib.sha256(st.block_offsets(w).astype("<u4").tobytes()).hexdigest() == \
            d[w + "_offsets_sha256"]
    assert st.k_lengths.tolist() == d["k_lengths"] and st.v_lengths.tolist() == d["v_lengths"]
    assert list(st.stats()) == d["stats"]


def test_big_digest_cfg1():
    """Config 1 (H32 x D128, 4K ctx, fp16) bitstreams == the reference's SHA-256."""
    import json, os
    from golden_cases import GOLDEN
    d = json.load(open(os.path.join(GOLDEN, "big_digests.json")))["cfg1"]
    k = oracle.generate_synthetic(4096, 32, 128, seed=0).astype(np.float16)
    v = oracle.generate_synthetic(4096, 32, 128, seed=0 ^ 0x9E3779B9).astype(np.float16)
    st = oracle.OracleState.prefill(k, v, n_threads=8)
    _digest_check(st, d)
    q = np.random.default_rng([0, 0x71726E67]).standard_normal((32, 128), dtype=np.float32)
    out, scores = st.attention_step(q)
    assert max_relative_error(out, np.array(d["att_out"])) <= 1e-5
    assert max_relative_error(scores[0, :64], np.array(d["att_scores_head0_first64"])) <= 1e-5


def test_big_digest_cfg4_streaming():
    """Config 4: 4K prefill + 8K single-token appends == the reference's SHA-256."""
    import json, os
    from golden_cases import GOLDEN
    d = json.load(open(os.path.join(GOLDEN, "big_digests.json")))["cfg4"]
    k = oracle.generate_synthetic(4096 + 8192, 32, 128, seed=0).astype(np.float16)
    v = oracle.generate_synthetic(4096 + 8192, 32, 128, seed=0 ^ 0x9E3779B9).astype(np.float16)
    st = oracle.OracleState.prefill(k[:4096], v[:4096], n_threads=8)
    for t in range(4096, 4096 + 8192):
        st.append_token(k[t], v[t])
    _digest_check(st, d)
