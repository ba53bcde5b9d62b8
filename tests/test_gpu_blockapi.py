"""The reference's per-block codec surface on the device, one golden test per
exported name (kvpack/__init__.py:9-75): quantize_unit, DecodeTree /
HuffmanCodebook.decode_tree, CompressedBlock + compress_block, encode_slice,
scan_offsets, decode_slice, decode_slices, decompress_block,
metadata_overhead, CompressedArena.append / .restore, run_ratio_sweep,
run_simulation.  Fixtures: tests/golden/blockapi.npz, written by
tests/golden/make_golden.py from the unmodified reference."""
import numpy as np
import pytest

from golden_cases import load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    return load("blockapi")


@pytest.fixture(scope="module")
def kv():
    import paper_2509_00579_b200 as kv
    return kv


@pytest.fixture(scope="module")
def state(kv, g):
    cfg_k, cfg_v = kv.QuantConfig(kv.QuantMode.K_BLOCK), kv.QuantConfig(kv.QuantMode.V_TOKEN)
    return kv.LayerCacheState.prefill(kv.CacheTensor(g["k_in"]), kv.CacheTensor(g["v_in"]),
                                      cfg_k, cfg_v)


def _np(t):
    return t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)


def _qblock(kv, g, nm):
    import torch
    return kv.QuantizedBlock(codes=torch.from_numpy(g[nm + "_codes"]).cuda(),
                             unit_mins=torch.from_numpy(g[nm + "_mins"]).cuda(),
                             unit_scales=torch.from_numpy(g[nm + "_scales"]).cuda(),
                             block_index=int(g[nm + "_block_index"]), head_index=1, ctx_start=64)


def _cb(state, nm):
    return state.k_codebook if nm == "k" else state.v_codebook


def test_quantize_unit(kv, g):
    off = 0
    for i, n in enumerate(g["unit_sizes"]):
        vals = g["unit_values"][off: off + n]
        codes, meta = kv.quantize_unit(vals, float(g["unit_rels"][i]))
        assert np.array_equal(_np(codes), g["unit_codes"][off: off + n]), i
        assert (meta.min_value, meta.scale) == tuple(g["unit_metas"][i]), i
        off += n
    with pytest.raises(kv.CodecError):
        kv.quantize_unit(np.array([]), 0.5)
    with pytest.raises(kv.CodecError):
        kv.quantize_unit(np.array([1.0, np.nan]), 0.5)
    with pytest.raises(kv.ConfigError):
        kv.quantize_unit(np.array([1.0]), 2.0)


def test_decode_tree(kv, g, state):
    for nm in ("k", "v"):
        t = _cb(state, nm).decode_tree
        assert isinstance(t, kv.DecodeTree)
        assert np.array_equal(t.children, g[nm + "_tree_children"])
        assert np.array_equal(t.is_symbol, g[nm + "_tree_is_symbol"])
        assert np.array_equal(t.symbols, g[nm + "_tree_symbols"])
    h = np.zeros(256, np.uint64)
    h[7] = 5
    t1 = kv.build_codebook(h).decode_tree
    assert np.array_equal(t1.children, g["single_tree_children"])
    assert np.array_equal(t1.is_symbol, g["single_tree_is_symbol"])
    assert np.array_equal(t1.symbols, g["single_tree_symbols"])


def test_compress_block(kv, g, state):
    for nm in ("k", "v"):
        c = kv.compress_block(_qblock(kv, g, nm), _cb(state, nm))
        assert isinstance(c, kv.CompressedBlock)
        assert c.block_index == int(g[nm + "_block_index"])
        assert np.array_equal(_np(c.slice_bit_counts), g[nm + "_counts"])
        assert np.array_equal(_np(c.payload), g[nm + "_payload"])
        assert np.array_equal(_np(c.unit_mins), g[nm + "_mins"])
        assert np.array_equal(_np(c.unit_scales), g[nm + "_scales"])
        assert c.total_bits == int(g[nm + "_total_bits"]) and c.n_slices == 64
    # a code absent from the codebook is a CodecError (codec.py:85-88)
    q = _qblock(kv, g, "v")
    q.codes[0, 0] = 200
    with pytest.raises(kv.CodecError):
        kv.compress_block(q, state.v_codebook)


def test_encode_slice(kv, g, state):
    for nm in ("k", "v"):
        bits, cnt = kv.encode_slice(g[nm + "_codes"][3], _cb(state, nm))
        assert cnt == int(g[nm + "_enc_slice3_count"])
        assert np.array_equal(_np(bits), g[nm + "_enc_slice3_bits"])
    with pytest.raises(kv.CodecError):
        kv.encode_slice(np.zeros(0, np.uint8), state.k_codebook)


def test_scan_offsets(kv, g):
    for nm in ("k", "v"):
        offs, tot = kv.scan_offsets(g[nm + "_counts"])
        assert np.array_equal(_np(offs), g[nm + "_scan"].astype(np.int64))
        assert tot == int(g[nm + "_scan_total"])
    with pytest.raises(kv.CodecError):
        kv.scan_offsets(np.zeros(0, np.uint16))
    with pytest.raises(kv.CodecError):
        kv.scan_offsets(np.full(70000, 65535, np.int64))


def test_decode_slice(kv, g, state):
    for nm in ("k", "v"):
        tree = _cb(state, nm).decode_tree
        offs = g[nm + "_scan"]
        out = kv.decode_slice(g[nm + "_payload"], int(offs[5]), int(g[nm + "_counts"][5]), tree,
                              128)
        assert np.array_equal(_np(out), g[nm + "_dec_slice5"])
    tree = state.k_codebook.decode_tree
    with pytest.raises(kv.CodecError):  # bit range outside the payload
        kv.decode_slice(g["k_payload"], len(g["k_payload"]) * 8 - 3, 10, tree, 128)
    with pytest.raises(kv.CodecError):  # wrong bit count: not exactly 128 symbols
        kv.decode_slice(g["k_payload"], 0, int(g["k_counts"][0]) - 1, tree, 128)


def test_decode_slices(kv, g, state):
    for nm in ("k", "v"):
        bits = np.unpackbits(g[nm + "_payload"])
        out = kv.decode_slices(bits, g[nm + "_scan"], g[nm + "_counts"],
                               _cb(state, nm).decode_tree, 128)
        assert np.array_equal(_np(out), g[nm + "_dec_slices"])
        assert np.array_equal(_np(out), g[nm + "_codes"])
    assert tuple(kv.decode_slices(np.zeros(8, np.uint8), [], [], state.k_codebook.decode_tree,
                                  128).shape) == (0, 128)
    bad = g["k_counts"].astype(np.int64).copy()
    bad[7] += 1
    with pytest.raises(kv.CodecError):
        kv.decode_slices(np.unpackbits(g["k_payload"]), g["k_scan"], bad,
                         state.k_codebook.decode_tree, 128)


def test_decompress_block(kv, g, state):
    for nm, ar, mode in (("k", state.k_arena, kv.QuantMode.K_BLOCK),
                         ("v", state.v_arena, kv.QuantMode.V_TOKEN)):
        assert ar.snapshot() == g[nm + "_arena"].tobytes()
        for i, o in enumerate(g["dec_ords"]):
            q = kv.decompress_block(ar, int(o), _cb(state, nm), mode=mode, head_num=2,
                                    head_dim=128, block_size=64)
            assert np.array_equal(_np(q.codes), g[nm + "_dec_codes"][i])
            assert np.array_equal(_np(q.unit_mins), g[nm + "_dec_mins"][i])
            assert np.array_equal(_np(q.unit_scales), g[nm + "_dec_scales"][i])
            assert [q.block_index, q.head_index, q.ctx_start] == list(g[nm + "_dec_idx"][i])
        with pytest.raises(kv.CodecError):
            kv.decompress_block(ar, len(ar), _cb(state, nm), mode=mode, head_num=2,
                                head_dim=128, block_size=64)


def test_metadata_overhead(kv, g, state):
    blocks = [kv.compress_block(_qblock(kv, g, nm), _cb(state, nm)) for nm in ("k", "v")]
    assert kv.metadata_overhead(blocks, 128) == tuple(g["meta_overhead"])
    with pytest.raises(kv.CodecError):
        kv.metadata_overhead([], 128)


def test_arena_restore(kv, g):
    for nm, n_units in (("k", 128), ("v", 64)):
        a = kv.CompressedArena.restore(g[nm + "_arena"].tobytes(), g[nm + "_offsets"], n_units)
        bits, pbytes, nsl, size, nb = (int(x) for x in g[nm + "_restore_counters"])
        assert (a.payload_bits, a.payload_bytes, a.n_slices, a.size_bytes, len(a)) == (
            bits, pbytes, nsl, size, nb)
        assert a.snapshot() == g[nm + "_arena"].tobytes()
        assert np.array_equal(a.block_offsets, g[nm + "_offsets"])
    broken = g["k_arena"].copy()
    broken[4] ^= 0x7F  # n_slices field: the metadata overruns the extent
    with pytest.raises(kv.CodecError):
        kv.CompressedArena.restore(broken.tobytes(), g["k_offsets"], 128)


def test_arena_append(kv, g, state):
    blocks = [kv.compress_block(_qblock(kv, g, nm), _cb(state, nm)) for nm in ("k", "v")]
    a = kv.CompressedArena()
    ords = [a.append(blocks[0]), a.append(blocks[1]), a.append(blocks[0])]
    assert ords == list(g["append_ordinals"])
    assert a.snapshot() == g["append_arena"].tobytes()
    assert np.array_equal(a.block_offsets, g["append_offsets"])
    assert [a.payload_bits, a.payload_bytes, a.n_slices] == list(g["append_counters"])
    # a block rebuilt from its fields (no cached image) serialises identically
    fresh = kv.CompressedBlock(block_index=blocks[1].block_index,
                               slice_bit_counts=blocks[1].slice_bit_counts,
                               unit_mins=blocks[1].unit_mins, unit_scales=blocks[1].unit_scales,
                               payload=blocks[1].payload)
    b = kv.CompressedArena()
    b.append(fresh)
    assert b.snapshot() == bytes(g["append_arena"][g["append_offsets"][1]:g["append_offsets"][2]])
    # capacity: the refused append raises ArenaFullError and changes nothing
    c = kv.CompressedArena(capacity=int(g["append_capacity"]))
    c.append(blocks[0])
    before = c.snapshot()
    with pytest.raises(kv.ArenaFullError):
        c.append(blocks[1])
    assert c.snapshot() == before and len(c) == 1
    c.check()  # the refusal left no sticky error behind


def test_run_ratio_sweep(kv, g):
    rows = kv.run_ratio_sweep([64, 200], [0.05, 0.2], head_num=2, head_dim=64, seed=3)
    got = np.array([[r.context_len, r.original_bytes, r.compressed_bytes, r.metadata_bytes]
                    for r in rows], np.int64)
    assert np.array_equal(got, g["sweep_rows"])
    assert [r.config for r in rows] == list(g["sweep_labels"])


def test_run_simulation(kv, g):
    cfg_k, cfg_v = kv.QuantConfig(kv.QuantMode.K_BLOCK), kv.QuantConfig(kv.QuantMode.V_TOKEN)
    sim = kv.run_simulation(kv.SimulationSettings(prompt_len=100, gen_len=40, head_num=2,
                                                  head_dim=128, seed=5, warmup=1, reps=2),
                            cfg_k, cfg_v)
    got = np.array([[r.context_len, r.original_bytes, r.compressed_bytes, r.metadata_bytes]
                    for r in sim.rows], np.int64)
    assert np.array_equal(got, g["sim_rows"])
    assert sim.summary.config == str(g["sim_label"])
    assert sim.max_divergence <= 1e-4
    assert sim.summary.fused_time > 0 and sim.summary.equivalent_decompression_throughput


def test_iter_decoded_blocks(kv, g, state):
    """codec.py:394-452: ordinals out of order, groups of two blocks (100
    slices), movement counters equal to the reference's."""
    for nm, ar, mode in (("k", state.k_arena, kv.QuantMode.K_BLOCK),
                         ("v", state.v_arena, kv.QuantMode.V_TOKEN)):
        mv = kv.DataMovement()
        rows = list(kv.iter_decoded_blocks(ar, _cb(state, nm), n_units=kv.units_per_block(mode, 128, 64),
                                           head_dim=128, ordinals=[5, 0, 3, 1], group_slices=100,
                                           movement=mv))
        assert [r[0] for r in rows] == list(g[nm + "_iter_ords"])
        assert [r[1] for r in rows] == list(g[nm + "_iter_bidx"])
        assert np.array_equal(np.stack([_np(r[2]) for r in rows]), g[nm + "_iter_codes"])
        assert np.array_equal(np.stack([_np(r[3]) for r in rows]), g[nm + "_iter_mins"])
        assert np.array_equal(np.stack([_np(r[4]) for r in rows]), g[nm + "_iter_scales"])
        assert [mv.bytes_read, mv.peak_scratch_values] == list(g[nm + "_iter_movement"])
        # all blocks in arena order, one group
        full = list(kv.iter_decoded_blocks(ar, _cb(state, nm), n_units=kv.units_per_block(mode, 128, 64),
                                           head_dim=128))
        assert [r[0] for r in full] == list(range(len(ar)))
        with pytest.raises(kv.CodecError):
            list(kv.iter_decoded_blocks(ar, _cb(state, nm), n_units=kv.units_per_block(mode, 128, 64),
                                        head_dim=128, ordinals=[len(ar)]))
