"""Helpers to read the reference golden fixtures (tests/golden/*.npz)."""

import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def cases(prefix):
    return sorted(os.path.basename(f)[len(prefix) + 1:-4]
                  for f in glob.glob(os.path.join(GOLDEN, f"{prefix}_*.npz")))


def load(prefix, name):
    return np.load(os.path.join(GOLDEN, f"{prefix}_{name}.npz"), allow_pickle=False)


def simplices_by_dim(z):
    d = int(z["dim"])
    return {k: z[f"simplices_{k}"] for k in range(d + 1)}


def values_by_dim(z):
    d = int(z["dim"])
    return {k: z[f"values_{k}"] for k in range(d + 1)}
