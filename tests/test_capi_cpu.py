"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host-side codebook builder matches the reference
(golden vectors from the reference itself).  No kernel launches here."""
import ctypes
import os
import re

import numpy as np
import pytest

from golden_cases import CASES, load

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2509_00579_b200 import _lib
    return _lib.lib()


def header_functions():
    src = open(os.path.join(ROOT, "include", "kvcomp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(kvc_\w+)\s*\(", src, flags=re.M)))


def test_exports_every_declared_symbol(lib):
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    from paper_2509_00579_b200 import _lib
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_struct_sizes(lib):
    from paper_2509_00579_b200 import _lib
    assert lib.kvc_codebook_bytes() == ctypes.sizeof(_lib.CodebookTables)
    assert ctypes.sizeof(_lib.ArenaCounters) == 40
    assert lib.kvc_version().startswith(b"kvcomp-b200")


def test_codebook_lengths_match_reference():
    from paper_2509_00579_b200 import build_codebook
    k = load("kats")
    for h, ln in zip(k["kat_hists"], k["kat_hist_lengths"]):
        assert np.array_equal(build_codebook(h).code_lengths, ln)
    cb = build_codebook(np.array([4, 2, 1, 1] + [0] * 252, np.uint64))
    assert np.array_equal(cb.code_lengths, k["kat_cb_lengths"])
    assert np.array_equal(cb.code_words, k["kat_cb_words"])


@pytest.mark.parametrize("case", CASES)
def test_smoothed_codebooks_match_reference(case):
    from paper_2509_00579_b200 import build_smoothed_codebook, codebook_from_lengths
    g = load(case)
    rel_k, rel_v = (float(x) for x in g["rel"])
    import math
    if "inject_k" not in g:
        kcb = build_smoothed_codebook(g["k_hist"], int(math.ceil(1 / rel_k)))
        vcb = build_smoothed_codebook(g["v_hist"], int(math.ceil(1 / rel_v)))
        assert np.array_equal(kcb.code_lengths, g["pre_k_lengths"])
        assert np.array_equal(vcb.code_lengths, g["pre_v_lengths"])
        assert np.array_equal(kcb.code_words, g["pre_k_words"])
        assert np.array_equal(vcb.code_words, g["pre_v_words"])
    for w in ("k", "v"):
        cb = codebook_from_lengths(g["pre_" + w + "_lengths"])
        assert np.array_equal(cb.code_words, g["pre_" + w + "_words"])


def test_codebook_errors_map_to_reference_exceptions():
    from paper_2509_00579_b200 import CodebookError, build_codebook, codebook_from_lengths
    with pytest.raises(CodebookError):
        build_codebook(np.zeros(256, np.uint64))
    bad = np.zeros(256, np.uint8)
    bad[:3] = [1, 2, 3]                      # Kraft sum != 1
    with pytest.raises(CodebookError):
        codebook_from_lengths(bad)
    one = np.zeros(256, np.uint8)
    one[7] = 2                               # single symbol must use 1 bit
    with pytest.raises(CodebookError):
        codebook_from_lengths(one)


def test_decode_lut_covers_every_window():
    from paper_2509_00579_b200 import codebook_from_lengths
    g = load("c_fp16_d128")
    cb = codebook_from_lengths(g["pre_k_lengths"])
    lut = np.frombuffer(bytes(cb.tables.lut), np.uint32)
    lens = (lut >> 8) & 0xFF
    syms = lut & 0xFF
    assert lens.min() >= 1
    # every window decodes to the symbol whose codeword prefixes it
    for i in range(0, 4096, 37):
        s, l = int(syms[i]), int(lens[i])
        assert (i >> (12 - l)) == int(cb.code_words[s]) and cb.code_lengths[s] == l


@pytest.mark.parametrize("case", CASES)
def test_decode_tree_matches_reference(case):
    """HuffmanCodebook.decode_tree (codebook.py:144-176): the reference's node
    numbering, host-side, from the reference-built codebooks' lengths."""
    from paper_2509_00579_b200 import codebook_from_lengths
    g = load(case)
    for w in ("k", "v"):
        t = codebook_from_lengths(g[f"fin_{w}_lengths"]).decode_tree
        assert np.array_equal(t.children, g[f"fin_{w}_tree_children"])
        assert t.n_nodes == len(g[f"fin_{w}_tree_children"])


def test_codebooks_shared_by_code_lengths():
    """codebook_from_lengths returns one immutable book per distinct length
    table (the tables and their device copy are reused across states); other
    lengths give a different book."""
    import numpy as np
    import pytest
    from paper_2509_00579_b200 import codebook_from_lengths
    lens = np.zeros(256, np.uint8)
    lens[:4] = [1, 2, 3, 3]
    a, b = codebook_from_lengths(lens), codebook_from_lengths(lens.copy())
    assert a is b
    with pytest.raises(ValueError):
        a.code_lengths[0] = 2
    lens[:4] = [2, 2, 2, 2]
    c = codebook_from_lengths(lens)
    assert c is not a and c.code_lengths[:4].tolist() == [2, 2, 2, 2]
    assert a.code_lengths[:4].tolist() == [1, 2, 3, 3]
