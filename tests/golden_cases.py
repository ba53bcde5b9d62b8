"""Helpers for replaying the golden fixtures (produced by make_golden.py)."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "c_*.npz")))


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def unpack_cfg(g):
    ctx, H, D, bs, buffer, appended = (int(x) for x in g["cfg"])
    rel_k, rel_v = (float(x) for x in g["rel"])
    return ctx, H, D, bs, buffer, appended, rel_k, rel_v


def max_relative_error(actual, reference):
    """helpers.py:115-119 of the reference tests: normalised by max|ref|."""
    ref = np.asarray(reference, dtype=np.float64)
    act = np.asarray(actual, dtype=np.float64)
    return float(np.abs(act - ref).max()) / max(float(np.abs(ref).max()), 1e-30)
