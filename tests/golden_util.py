"""Helpers to rebuild golden-fixture models without the reference package."""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

from paper_1010_0012_b200.model import GridMrf, SparseTruncatedPotential, \
    truncated_linear_potential

GOLDEN = Path(__file__).resolve().parent / "golden"


def manifest() -> dict:
    with open(GOLDEN / "manifest.json") as f:
        return json.load(f)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def sha_raw(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load_case(name: str):
    """(model, arrays) for a fixture saved with its model inputs."""
    z = dict(np.load(GOLDEN / f"{name}.npz"))
    H, W = (int(v) for v in z["grid_shape"])
    M = z["unaries"].shape[1]
    if "pe_indptr" in z:           # one potential per edge (reference generic engine)
        pots, off = [], 0
        for e, indptr in enumerate(z["pe_indptr"]):
            n = int(indptr[-1])
            pots.append(SparseTruncatedPotential(M, float(z["pe_fbar"][e]), indptr,
                                                 z["pe_indices"][off:off + n],
                                                 z["pe_values"][off:off + n]))
            off += n
        model = GridMrf(H, W, M, z["unaries"], pots, log_unaries=z["log_unaries"])
        return model, z
    if "col_indptr" in z:
        pot = SparseTruncatedPotential(M, float(z["fbar"]), z["col_indptr"], z["col_indices"],
                                       z["col_values"])
        pot._log = SparseTruncatedPotential(M, float(z["log_fbar"]), z["col_indptr"],
                                            z["col_indices"], z["log_col_values"])
    else:   # single node: no edges, any potential
        pot = truncated_linear_potential(M, 1.0, 2.0)
    model = GridMrf(H, W, M, z["unaries"], pot, log_unaries=z["log_unaries"])
    return model, z
