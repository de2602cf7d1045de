"""Shared test helpers (test infrastructure)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def coeff_dict(cf):
    from oracle.hps_oracle import COEFF_NAMES
    return {n: getattr(cf, n) for n in COEFF_NAMES}


def golden_tree(tag):
    z = golden("tree_small.npz")
    return {k.split("__", 1)[1]: z[k] for k in z.files if k.startswith(tag + "__")}
