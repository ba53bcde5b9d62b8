"""Generate golden fixtures by running the UNMODIFIED reference (kvpack).

This script is the only place that touches /root/reference: it imports the
reference package from a temporary copy and records its outputs as small
``.npz`` fixtures (plus SHA-256 digests for the full-size BASELINE configs)
under ``tests/golden/``.  The fixtures pin both the CPU oracle (``oracle/``)
and the CUDA path; nothing at test/bench time needs the reference.

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --big      # + config-1/4 digests (~30 s)
    python tests/golden/make_golden.py --cfg2     # + config-2 slice (~2 min)

Reference call sites followed: kvcache.py:76-145 (prefill), :150-177
(append_token), attention.py:176-188 (attention_step), :112-165
(fused_v_output), kvcache.py:182-212 (fetch_dequantized), bench.py:77-95
(collect_stats), quantizer.py:162-209 (quantize_block).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import shutil
import sys
import tempfile
from dataclasses import replace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"


def _import_reference():
    tmp = tempfile.mkdtemp(prefix="kvpack_ref_")
    shutil.copytree(REF, os.path.join(tmp, "src"))
    sys.path.insert(0, os.path.join(tmp, "src"))
    import kvpack  # noqa: E402

    return kvpack


kv = _import_reference()


def _arena(a):
    return np.frombuffer(a.snapshot(), dtype=np.uint8).copy(), a.block_offsets.astype(np.uint32)


def _state_record(prefix, st):
    rec = {}
    ka, ko = _arena(st.k_arena)
    va, vo = _arena(st.v_arena)
    rec[prefix + "k_arena"] = ka
    rec[prefix + "k_offsets"] = ko
    rec[prefix + "v_arena"] = va
    rec[prefix + "v_offsets"] = vo
    rec[prefix + "k_lengths"] = st.k_codebook.code_lengths.astype(np.uint8)
    rec[prefix + "v_lengths"] = st.v_codebook.code_lengths.astype(np.uint8)
    rec[prefix + "k_words"] = st.k_codebook.code_words.astype(np.uint32)
    rec[prefix + "v_words"] = st.v_codebook.code_words.astype(np.uint32)
    rec[prefix + "k_tree_children"] = st.k_codebook.decode_tree.children.astype(np.int32)
    rec[prefix + "v_tree_children"] = st.v_codebook.decode_tree.children.astype(np.int32)
    rec[prefix + "counters"] = np.array(
        [st.context_len, st.compressed_tokens, st.buffered,
         st.k_arena.payload_bits, st.k_arena.payload_bytes, st.k_arena.n_slices,
         st.v_arena.payload_bits, st.v_arena.payload_bytes, st.v_arena.n_slices],
        dtype=np.int64)
    rec[prefix + "k_buffer"] = st._k_buffer[: st.buffered].copy()
    rec[prefix + "v_buffer"] = st._v_buffer[: st.buffered].copy()
    s = kv.collect_stats(st)
    rec[prefix + "stats"] = np.array(
        [s.original_bytes, s.compressed_bytes, s.metadata_bytes, s.payload_bits,
         s.quantized_values], dtype=np.int64)
    rec[prefix + "ratio"] = np.float64(s.compression_ratio)
    return rec


def _prefill_hist(k_work, v_work, cfg_k, cfg_v, H, ranges=None):
    """Raw (unsmoothed) prefill histograms, via the reference's own functions."""
    n_full = (k_work.shape[0] // cfg_k.block_size) * cfg_k.block_size
    hk = np.zeros(256, dtype=np.uint64)
    hv = np.zeros(256, dtype=np.uint64)
    kq, vq = [], []
    if n_full:
        from kvpack.kvcache import _quantize_tokens

        kq = _quantize_tokens(k_work[:n_full], cfg_k, 0, H, ranges)
        vq = _quantize_tokens(v_work[:n_full], cfg_v, 0, H, None)
        hk += kv.build_histogram(np.concatenate([b.codes.ravel() for b in kq]))
        hv += kv.build_histogram(np.concatenate([b.codes.ravel() for b in vq]))
    return hk, hv, kq, vq


def make_case(name, *, ctx, H, D, bs, buffer=None, rel_k=0.05, rel_v=0.15, dtype=np.float16,
              seed=0, appended=0, inject=None, constant=None, synthetic=True, n_q=2,
              k_mode="kblock"):
    cfg_k = kv.QuantConfig(kv.QuantMode(k_mode), block_size=bs, rel_quant_scale=rel_k,
                           buffer_size=buffer)
    cfg_v = kv.QuantConfig(kv.QuantMode.V_TOKEN, block_size=bs, rel_quant_scale=rel_v,
                           buffer_size=buffer)
    total = ctx + appended
    if constant is not None:
        kfull = np.full((total, H, D), constant[0], dtype=np.float32)
        vfull = np.full((total, H, D), constant[1], dtype=np.float32)
    elif synthetic:
        spec = kv.SyntheticSpec(total, H, D, seed=seed)
        kfull = kv.generate_synthetic(spec).values
        vfull = kv.generate_synthetic(replace(spec, seed=seed ^ 0x9E3779B9)).values
    else:
        rng = np.random.default_rng(seed)
        kfull = rng.standard_normal((total, H, D)).astype(np.float32)
        vfull = rng.standard_normal((total, H, D)).astype(np.float32)
    k_in = kfull[:ctx].astype(dtype)
    v_in = vfull[:ctx].astype(dtype)
    codebooks = None
    if inject is not None:
        codebooks = tuple(kv.codebook_from_lengths if False else kv.deserialize_codebook(
            bytes(np.asarray(x, dtype=np.uint8).tobytes())) for x in inject)
    rec = {
        "cfg": np.array([ctx, H, D, bs, cfg_k.buffer_size, appended], dtype=np.int64),
        "rel": np.array([cfg_k.rel_quant_scale, rel_v], dtype=np.float64),
        "k_mode": np.array(k_mode),
        "k_in": k_in, "v_in": v_in,
        "k_app": kfull[ctx:].astype(np.float32), "v_app": vfull[ctx:].astype(np.float32),
    }
    if inject is not None:
        rec["inject_k"] = np.asarray(inject[0], dtype=np.uint8)
        rec["inject_v"] = np.asarray(inject[1], dtype=np.uint8)
    k_ct, v_ct = kv.CacheTensor(k_in), kv.CacheTensor(v_in)
    ranges = None
    if k_mode == "kchannel":
        kw = k_ct.as_float32()
        ranges = (kw.min(axis=0).astype(np.float32), kw.max(axis=0).astype(np.float32))
        rec["k_ranges"] = np.stack(ranges)
    hk, hv, kq, vq = _prefill_hist(k_ct.as_float32(), v_ct.as_float32(), cfg_k, cfg_v, H, ranges)
    rec["k_hist"] = hk
    rec["v_hist"] = hv
    if kq:
        rec["k_codes"] = np.stack([b.codes for b in kq])
        rec["k_mins"] = np.stack([b.unit_mins for b in kq])
        rec["k_scales"] = np.stack([b.unit_scales for b in kq])
        rec["v_codes"] = np.stack([b.codes for b in vq])
        rec["v_mins"] = np.stack([b.unit_mins for b in vq])
        rec["v_scales"] = np.stack([b.unit_scales for b in vq])
    st = kv.LayerCacheState.prefill(k_ct, v_ct, cfg_k, cfg_v, codebooks=codebooks)
    rec.update(_state_record("pre_", st))
    for t in range(appended):
        st.append_token(kfull[ctx + t], vfull[ctx + t])
    rec.update(_state_record("fin_", st))
    # Fetch side on the final state.
    qrng = np.random.default_rng([seed, 0x71726E67])
    qs, outs, scores = [], [], []
    for _ in range(n_q):
        q = qrng.standard_normal((H, D), dtype=np.float32)
        res = kv.attention_step(st, q)
        qs.append(q)
        outs.append(res.out)
        scores.append(res.scores)
    rec["q"] = np.stack(qs)
    rec["att_out"] = np.stack(outs)
    rec["att_scores"] = np.stack(scores)
    w = qrng.random((H, st.context_len), dtype=np.float32)
    rec["w"] = w
    rec["vout_w"] = kv.fused_v_output(st, w)
    kd, vd = st.fetch_dequantized()
    rec["deq_k"] = kd.values
    rec["deq_v"] = vd.values
    tmpf = os.path.join(tempfile.mkdtemp(), "s.kvcz")
    kv.save_state(st, tmpf)
    rec["kvcz"] = np.frombuffer(open(tmpf, "rb").read(), np.uint8).copy()
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **rec)
    print(f"{name}: ctx={ctx}+{appended} H={H} D={D} bs={bs} k_maxlen={int(st.k_codebook.max_code_length)} "
          f"v_maxlen={int(st.v_codebook.max_code_length)} ratio={rec['fin_ratio']:.4f} "
          f"size={os.path.getsize(path)}")


def _fib_lengths(n):
    h = np.zeros(256, dtype=np.uint64)
    a, b = 1, 1
    for s in range(n):
        h[s] = a
        a, b = b, a + b
    return kv.build_codebook(h).code_lengths


def kat_cases():
    """Known-answer vectors from the reference tests (test_*.py), re-run here."""
    out = {}
    # test_quantizer.py:27-35 : [0,1,2,3] @ rel 0.5
    c, m = kv.quantize_unit(np.array([0, 1, 2, 3], dtype=np.float32), 0.5)
    out["kat_quant_codes"] = c.astype(np.uint8)
    out["kat_quant_meta"] = np.array([m.min_value, m.scale], dtype=np.float64)
    # test_codebook.py:77-82 : {4,2,1,1} -> lengths [1,2,3,3]
    h = np.zeros(256, dtype=np.uint64)
    h[:4] = [4, 2, 1, 1]
    cb = kv.build_codebook(h)
    out["kat_cb_lengths"] = cb.code_lengths.astype(np.uint8)
    out["kat_cb_words"] = cb.code_words.astype(np.uint32)
    # test_codec.py:125-139 style: encode [0,1,2,3] with that codebook
    bits, count = kv.encode_slice(np.array([0, 1, 2, 3], dtype=np.uint8), cb)
    out["kat_slice_bytes"] = np.packbits(bits)
    out["kat_slice_count"] = np.int64(count)
    # random histograms -> lengths (tie-breaking coverage)
    rng = np.random.default_rng(1234)
    hists, lens = [], []
    for i in range(64):
        hh = np.zeros(256, dtype=np.uint64)
        n = int(rng.integers(1, 257))
        sel = rng.choice(256, size=n, replace=False)
        if i % 3 == 0:
            hh[sel] = rng.integers(1, 5, size=n)        # many ties
        elif i % 3 == 1:
            hh[sel] = rng.integers(1, 1 << 20, size=n)
        else:
            hh[sel] = (1.6 ** rng.integers(0, 40, size=n)).astype(np.uint64)
        hists.append(hh)
        lens.append(kv.build_codebook(hh).code_lengths.astype(np.uint8))
    out["kat_hists"] = np.stack(hists)
    out["kat_hist_lengths"] = np.stack(lens)
    # quantize edge cases: half-step grid (adversarial ties), constants, tiny ranges
    grids = []
    rng = np.random.default_rng(99)
    for rel in (0.05, 0.15, 1 / 255, 0.5, 1.0, 0.3333):
        x = rng.standard_normal((64, 128)).astype(np.float32)
        x[:, :8] = np.float32(0.25) * rng.integers(-8, 8, size=(64, 8))   # half-step ties
        x[:, 8] = 3.0                                                      # constant column
        x[5, :] = -1.0                                                     # constant row
        x[:, 9] = np.float32(1e-30) * rng.standard_normal(64)               # scale underflow
        grids.append((rel, x))
    out["kat_grid_x"] = np.stack([g[1] for g in grids])
    out["kat_grid_rel"] = np.array([g[0] for g in grids])
    kc, km, ks, vc, vm, vs = [], [], [], [], [], []
    for rel, x in grids:
        cfgk = kv.QuantConfig(kv.QuantMode.K_BLOCK, 64, rel)
        cfgv = kv.QuantConfig(kv.QuantMode.V_TOKEN, 64, rel)
        qk = kv.quantize_block(x, kv.QuantMode.K_BLOCK, cfgk, 0, 0, 1)
        qv = kv.quantize_block(x, kv.QuantMode.V_TOKEN, cfgv, 0, 0, 1)
        kc.append(qk.codes); km.append(qk.unit_mins); ks.append(qk.unit_scales)
        vc.append(qv.codes); vm.append(qv.unit_mins); vs.append(qv.unit_scales)
    out.update(kat_grid_kcodes=np.stack(kc), kat_grid_kmins=np.stack(km),
               kat_grid_kscales=np.stack(ks), kat_grid_vcodes=np.stack(vc),
               kat_grid_vmins=np.stack(vm), kat_grid_vscales=np.stack(vs))
    np.savez_compressed(os.path.join(HERE, "kats.npz"), **out)
    print("kats: written")


def blockapi_cases():
    """The per-block codec surface (codec.py:59-472, quantizer.py:144-160,
    codebook.py:35-66/:144-176, CompressedArena.append/.restore) run on the
    reference, for the device-backed drop-ins (tests/test_gpu_blockapi.py)."""
    from kvpack import codec as rcodec

    out = {}
    H, D, bs = 2, 128, 64
    spec = kv.SyntheticSpec(bs * 3 + 9, H, D, seed=41)
    k = kv.generate_synthetic(spec).values.astype(np.float16)
    v = kv.generate_synthetic(replace(spec, seed=41 ^ 0x9E3779B9)).values.astype(np.float16)
    cfg_k, cfg_v = kv.QuantConfig(kv.QuantMode.K_BLOCK), kv.QuantConfig(kv.QuantMode.V_TOKEN)
    st = kv.LayerCacheState.prefill(kv.CacheTensor(k), kv.CacheTensor(v), cfg_k, cfg_v)
    out["k_in"], out["v_in"] = k, v
    kf, vf = k.astype(np.float32), v.astype(np.float32)
    # quantize_block + compress_block of block (chunk 1, head 1) for K and V
    qk = kv.quantize_block(kf[bs:2 * bs, 1], kv.QuantMode.K_BLOCK, cfg_k, 1, bs, H)
    qv = kv.quantize_block(vf[bs:2 * bs, 1], kv.QuantMode.V_TOKEN, cfg_v, 1, bs, H)
    blocks = []
    for nm, q, cb in (("k", qk, st.k_codebook), ("v", qv, st.v_codebook)):
        c = kv.compress_block(q, cb)
        blocks.append(c)
        out[nm + "_codes"] = q.codes
        out[nm + "_mins"], out[nm + "_scales"] = q.unit_mins, q.unit_scales
        out[nm + "_block_index"] = np.int64(c.block_index)
        out[nm + "_counts"] = c.slice_bit_counts.astype(np.uint16)
        out[nm + "_payload"] = np.frombuffer(c.payload, np.uint8).copy()
        out[nm + "_total_bits"] = np.int64(c.total_bits)
        out[nm + "_image"] = np.frombuffer(rcodec._serialize_block(c), np.uint8).copy()
        offs, tot = kv.scan_offsets(c.slice_bit_counts)
        out[nm + "_scan"], out[nm + "_scan_total"] = offs.astype(np.uint32), np.int64(tot)
        out[nm + "_dec_slice5"] = kv.decode_slice(c.payload, int(offs[5]),
                                                  int(c.slice_bit_counts[5]), cb.decode_tree, D)
        out[nm + "_dec_slices"] = kv.decode_slices(np.unpackbits(np.frombuffer(c.payload, np.uint8)),
                                                   offs, c.slice_bit_counts, cb.decode_tree, D)
        t = cb.decode_tree
        out[nm + "_tree_children"], out[nm + "_tree_is_symbol"] = t.children, t.is_symbol
        out[nm + "_tree_symbols"] = t.symbols
        bits, cnt = kv.encode_slice(q.codes[3], cb)
        out[nm + "_enc_slice3_bits"], out[nm + "_enc_slice3_count"] = bits.astype(np.uint8), np.int64(cnt)
    out["meta_overhead"] = np.array(kv.metadata_overhead(blocks, D), np.float64)
    # decompress_block of arena ordinals of the prefilled state
    ords = [0, 3, 5]
    out["dec_ords"] = np.array(ords, np.int64)
    for nm, ar, cb, mode in (("k", st.k_arena, st.k_codebook, kv.QuantMode.K_BLOCK),
                             ("v", st.v_arena, st.v_codebook, kv.QuantMode.V_TOKEN)):
        res = [kv.decompress_block(ar, o, cb, mode=mode, head_num=H, head_dim=D, block_size=bs)
               for o in ords]
        out[nm + "_dec_codes"] = np.stack([r.codes for r in res])
        out[nm + "_dec_mins"] = np.stack([r.unit_mins for r in res])
        out[nm + "_dec_scales"] = np.stack([r.unit_scales for r in res])
        out[nm + "_dec_idx"] = np.array([[r.block_index, r.head_index, r.ctx_start] for r in res],
                                        np.int64)
        out[nm + "_arena"] = np.frombuffer(ar.snapshot(), np.uint8).copy()
        out[nm + "_offsets"] = ar.block_offsets.astype(np.uint32)
        r = kv.CompressedArena.restore(ar.snapshot(), ar.block_offsets,
                                       rcodec.units_per_block(mode, D, bs))
        out[nm + "_restore_counters"] = np.array([r.payload_bits, r.payload_bytes, r.n_slices,
                                                  r.size_bytes, len(r)], np.int64)
    # iter_decoded_blocks (codec.py:394-452): out-of-order ordinals, groups of two blocks
    for nm, ar, cb, mode in (("k", st.k_arena, st.k_codebook, kv.QuantMode.K_BLOCK),
                             ("v", st.v_arena, st.v_codebook, kv.QuantMode.V_TOKEN)):
        mv = rcodec.DataMovement()
        it = list(rcodec.iter_decoded_blocks(ar, cb, n_units=rcodec.units_per_block(mode, D, bs),
                                             head_dim=D, ordinals=[5, 0, 3, 1], group_slices=100,
                                             movement=mv))
        out[nm + "_iter_ords"] = np.array([r[0] for r in it], np.int64)
        out[nm + "_iter_bidx"] = np.array([r[1] for r in it], np.int64)
        out[nm + "_iter_codes"] = np.stack([r[2] for r in it])
        out[nm + "_iter_mins"] = np.stack([r[3] for r in it])
        out[nm + "_iter_scales"] = np.stack([r[4] for r in it])
        out[nm + "_iter_movement"] = np.array([mv.bytes_read, mv.peak_scratch_values], np.int64)
    # CompressedArena.append: K block, V block, K block again, then a capacity refusal
    a = kv.CompressedArena()
    ords_app = [a.append(blocks[0]), a.append(blocks[1]), a.append(blocks[0])]
    out["append_ordinals"] = np.array(ords_app, np.int64)
    out["append_arena"] = np.frombuffer(a.snapshot(), np.uint8).copy()
    out["append_offsets"] = a.block_offsets.astype(np.uint32)
    out["append_counters"] = np.array([a.payload_bits, a.payload_bytes, a.n_slices], np.int64)
    cap = len(rcodec._serialize_block(blocks[0])) + 8
    a2 = kv.CompressedArena(capacity=cap)
    a2.append(blocks[0])
    try:
        a2.append(blocks[1])
        raise SystemExit("reference did not refuse the append")
    except kv.ArenaFullError:
        pass
    out["append_capacity"] = np.int64(cap)
    # quantize_unit on float64 units: KAT, values off the f32 grid, ties, constant
    rng = np.random.default_rng(77)
    units = [np.array([0, 1, 2, 3], np.float64), rng.standard_normal(97) * 1e3,
             np.linspace(-1.0, 1.0, 41), np.full(9, 2.5), rng.standard_normal(300)]
    rels = [0.5, 0.05, 0.05, 0.15, 1 / 255]
    uc, um = [], []
    for u, rel in zip(units, rels):
        c, m = kv.quantize_unit(u, rel)
        uc.append(c.astype(np.uint8))
        um.append([m.min_value, m.scale])
    out["unit_values"] = np.concatenate(units)
    out["unit_sizes"] = np.array([len(u) for u in units], np.int64)
    out["unit_rels"] = np.array(rels, np.float64)
    out["unit_codes"] = np.concatenate(uc)
    out["unit_metas"] = np.array(um, np.float64)
    # single-symbol codebook tree (codebook.py:149-154) and its decode
    h = np.zeros(256, np.uint64)
    h[7] = 5
    cb1 = kv.build_codebook(h)
    t1 = cb1.decode_tree
    out["single_tree_children"], out["single_tree_is_symbol"] = t1.children, t1.is_symbol
    out["single_tree_symbols"] = t1.symbols
    # run_ratio_sweep / run_simulation rows (ratio fields only; times differ)
    rows = kv.run_ratio_sweep([64, 200], [0.05, 0.2], head_num=2, head_dim=64, seed=3)
    out["sweep_rows"] = np.array([[r.context_len, r.original_bytes, r.compressed_bytes,
                                   r.metadata_bytes] for r in rows], np.int64)
    out["sweep_labels"] = np.array([r.config for r in rows])
    sim = kv.run_simulation(kv.SimulationSettings(prompt_len=100, gen_len=40, head_num=2,
                                                  head_dim=128, seed=5, warmup=1, reps=2),
                            cfg_k, cfg_v)
    out["sim_rows"] = np.array([[r.context_len, r.original_bytes, r.compressed_bytes,
                                 r.metadata_bytes] for r in sim.rows], np.int64)
    out["sim_label"] = np.array(sim.summary.config)
    np.savez_compressed(os.path.join(HERE, "blockapi.npz"), **out)
    print("blockapi: written")


def _digest(st):
    h = {}
    for nm, a in (("k", st.k_arena), ("v", st.v_arena)):
        h[nm + "_arena_sha256"] = hashlib.sha256(a.snapshot()).hexdigest()
        h[nm + "_offsets_sha256"] = hashlib.sha256(
            a.block_offsets.astype("<u4").tobytes()).hexdigest()
        h[nm + "_arena_bytes"] = a.size_bytes
        h[nm + "_blocks"] = len(a)
        h[nm + "_payload_bits"] = a.payload_bits
    h["k_lengths"] = st.k_codebook.code_lengths.tolist()
    h["v_lengths"] = st.v_codebook.code_lengths.tolist()
    s = kv.collect_stats(st)
    h["ratio"] = s.compression_ratio
    h["stats"] = [s.original_bytes, s.compressed_bytes, s.metadata_bytes, s.payload_bits,
                  s.quantized_values]
    h["context_len"] = st.context_len
    h["compressed_tokens"] = st.compressed_tokens
    h["buffered"] = st.buffered
    return h


def big_digests(do_cfg2=False):
    import time

    res = {}
    path = os.path.join(HERE, "big_digests.json")
    if os.path.exists(path):
        res = json.load(open(path))
    # Config 1: H 32 x D 128, ctx 4096, fp16, seed 0, default scales.
    spec = kv.SyntheticSpec(4096, 32, 128, seed=0)
    k = kv.generate_synthetic(spec).values.astype(np.float16)
    v = kv.generate_synthetic(replace(spec, seed=0 ^ 0x9E3779B9)).values.astype(np.float16)
    cfg_k = kv.QuantConfig(kv.QuantMode.K_BLOCK)
    cfg_v = kv.QuantConfig(kv.QuantMode.V_TOKEN)
    t0 = time.time()
    st = kv.LayerCacheState.prefill(kv.CacheTensor(k), kv.CacheTensor(v), cfg_k, cfg_v)
    d = _digest(st)
    q = np.random.default_rng([0, 0x71726E67]).standard_normal((32, 128), dtype=np.float32)
    r = kv.attention_step(st, q)
    d["att_out"] = r.out.tolist()
    d["att_scores_head0_first64"] = r.scores[0, :64].tolist()
    res["cfg1"] = d
    print(f"cfg1 done {time.time()-t0:.1f}s ratio={d['ratio']:.4f}")
    # Config 4: prefill 4096 then 8192 appends (growing cache), H 32 x 128.
    t0 = time.time()
    spec = kv.SyntheticSpec(4096 + 8192, 32, 128, seed=0)
    kf = kv.generate_synthetic(spec).values.astype(np.float16)
    vf = kv.generate_synthetic(replace(spec, seed=0 ^ 0x9E3779B9)).values.astype(np.float16)
    st = kv.LayerCacheState.prefill(kv.CacheTensor(kf[:4096]), kv.CacheTensor(vf[:4096]),
                                    cfg_k, cfg_v)
    for t in range(4096, 4096 + 8192):
        st.append_token(kf[t], vf[t])
    res["cfg4"] = _digest(st)
    print(f"cfg4 done {time.time()-t0:.1f}s")
    if do_cfg2:
        t0 = time.time()
        spec = kv.SyntheticSpec(32768, 40, 128, seed=0)
        k = kv.generate_synthetic(spec).values.astype(np.float16)
        v = kv.generate_synthetic(replace(spec, seed=0 ^ 0x9E3779B9)).values.astype(np.float16)
        st = kv.LayerCacheState.prefill(kv.CacheTensor(k), kv.CacheTensor(v), cfg_k, cfg_v)
        d = _digest(st)
        # one reference attention_step on the slice (attention.py:176-188, ~40 s)
        q = np.random.default_rng([0, 0x71726E67]).standard_normal((40, 128), dtype=np.float32)
        r = kv.attention_step(st, q)
        d["att_out"] = r.out.tolist()
        d["att_scores_head0_first64"] = r.scores[0, :64].tolist()
        d["att_scores_head39_last64"] = r.scores[39, -64:].tolist()
        res["cfg2_slice"] = d
        print(f"cfg2 slice done {time.time()-t0:.1f}s")
    with open(path, "w") as fh:
        json.dump(res, fh, indent=1)


def kvtn_cases():
    """KVTN files (tensor_io.py:100-143) written by the reference's
    write_tensor, for tests/test_kvtn_cpu.py."""
    rng = np.random.default_rng(19)
    out = {}
    for nm, dt, shape in (("f16", np.float16, (5, 3, 7)), ("f32", np.float32, (4, 2, 9))):
        vals = rng.standard_normal(shape).astype(dt)
        path = os.path.join(tempfile.mkdtemp(), "t.kvtn")
        kv.write_tensor(kv.CacheTensor(vals), path)
        with open(path, "rb") as fh:
            out[nm + "_file"] = np.frombuffer(fh.read(), np.uint8).copy()
        out[nm + "_values"] = vals
        back = kv.read_tensor(path).values
        assert np.array_equal(back.view(np.uint8), vals.view(np.uint8))
    np.savez_compressed(os.path.join(HERE, "kvtn.npz"), **out)
    print("kvtn: written")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--cfg2", action="store_true")
    ap.add_argument("--only", default=None, help="run one generator, e.g. blockapi_cases")
    args = ap.parse_args()
    if args.only:
        globals()[args.only]()
        return
    kat_cases()
    blockapi_cases()
    kvtn_cases()
    make_case("c_fp16_d128", ctx=64 * 3 + 37, H=2, D=128, bs=64, seed=3, appended=100)
    make_case("c_f32_d32_bs16", ctx=16 * 5 + 3, H=4, D=32, bs=16, dtype=np.float32,
              synthetic=False, seed=7, appended=40)
    make_case("c_fine_scales", ctx=64 * 2 + 10, H=2, D=64, bs=64, rel_k=1 / 255, rel_v=1 / 255,
              seed=5, appended=0)
    make_case("c_coarse_scales", ctx=64 * 2 + 1, H=3, D=128, bs=64, rel_k=0.5, rel_v=1.0,
              seed=6, appended=70)
    make_case("c_odd_shapes", ctx=8 * 6 + 5, H=3, D=6, bs=8, buffer=16, dtype=np.float32,
              synthetic=False, seed=8, appended=30)
    make_case("c_injected_long", ctx=64 * 2 + 5, H=2, D=128, bs=64, seed=9, appended=64,
              inject=(_fib_lengths(30), _fib_lengths(12)))
    make_case("c_constant", ctx=32, H=2, D=8, bs=8, dtype=np.float32, constant=(7.5, -2.5),
              appended=12, inject=(np.eye(256, dtype=np.uint8)[0], np.eye(256, dtype=np.uint8)[0]))
    make_case("c_prefill_short", ctx=5, H=2, D=16, bs=8, dtype=np.float32, synthetic=False,
              seed=10, appended=20)
    make_case("c_kchannel", ctx=64 * 3 + 11, H=2, D=64, bs=64, seed=12, appended=90,
              rel_k=None, k_mode="kchannel")
    make_case("c_kchannel_f32_bs8", ctx=8 * 3 + 2, H=2, D=4, bs=8, buffer=16, dtype=np.float32,
              synthetic=False, seed=30, appended=20, rel_k=0.05, k_mode="kchannel")
    # Fine quantisation scales on the hot shape (D 128, bs 64; BASELINE config 5
    # sweep points): 7-12 bit codes and 21-256 symbol alphabets, 3 prefill
    # blocks + > 128 appends (one growing-cache overflow event), so the
    # 256-bin Store histograms, the look-back prefill and the single-symbol
    # fused fetch are all pinned to the reference.
    for nm, rk, rv, sd in (("c_fine_d128_255", 1 / 255, 1 / 255, 21),
                           ("c_fine_d128_001", 0.01, 0.02, 22),
                           ("c_fine_d128_002", 0.02, 0.05, 23)):
        make_case(nm, ctx=64 * 3 + 20, H=2, D=128, bs=64, rel_k=rk, rel_v=rv, seed=sd,
                  appended=150)
    if args.big or args.cfg2:
        big_digests(args.cfg2)


if __name__ == "__main__":
    main()
