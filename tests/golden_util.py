"""Helpers to read the committed golden fixtures (made by
``oracle/make_goldens.py`` from the real reference)."""

import glob
import hashlib
import json
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    return sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.json")))


def load(name):
    with open(os.path.join(GOLDEN_DIR, f"{name}.json")) as f:
        return json.load(f)


def sha_u64(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def sha_i64(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()


def input_of(g):
    """(keys uint64, pe_sizes) for a fixture, regenerated from its seed or
    read from its stored data."""
    from oracle import ams_oracle as O
    if "data" in g:
        p = g["p"]
        keys = [k for pe in range(p) for k, _, _ in g["data"][str(pe)]]
        return np.asarray(keys, dtype=np.uint64), list(g["input_pe_sizes"])
    keys = O.reference_input(g["dist"], g["p"], g["n_per_pe"], g["input_seed"])
    return keys, list(g["input_pe_sizes"])
