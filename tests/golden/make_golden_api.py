"""Golden fixtures for the reference-constructor surface (build container only).

``sparsebp.MrfModel(M, unaries, edges, potentials, grid_shape, log_unaries)``
(mrf.py:298-369) accepts the grid's edges in ANY order and orientation.  This
records, for a small grid whose edge list is permuted with half of the edges
reversed, what the reference itself returns: the canonical SweepSchedule pass
lists (bp.py:190-234) and the ``run_sweeps`` message store in the model's own
directed-edge ids (default schedule), for a shared potential (grid engine)
and for per-edge potentials (generic engine, which orients each potential by
its edge).  Usage: python tests/golden/make_golden_api.py
"""
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import sparsebp  # noqa: E402
from sparsebp import synth as ref_synth  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    rng = np.random.default_rng(77)
    H, W, M = 5, 7, 9
    u = rng.uniform(0.05, 1.0, size=(H * W, M))
    canon = np.array(sparsebp.mrf._grid_edges(H, W), dtype=np.int64)
    perm = rng.permutation(len(canon))
    edges = canon[perm]
    flip = rng.random(len(edges)) < 0.5
    edges[flip] = edges[flip][:, ::-1]
    pot = sparsebp.truncated_linear_potential(M, 0.6, 3.0)
    # per-edge: asymmetric random sparse potentials (orientation matters)
    pe = [ref_synth.random_sparse_potential(rng, M) for _ in range(len(edges))]
    man = {"generator": "tests/golden/make_golden_api.py", "cases": {}}
    arrays = {"unaries": u, "edges": edges, "grid_shape": np.array([H, W]),
              "pot_fbar": np.array(pot.fbar), "pot_indptr": pot.col_indptr,
              "pot_indices": pot.col_indices, "pot_values": pot.col_values,
              "pe_fbar": np.array([p.fbar for p in pe]),
              "pe_indptr": np.stack([p.col_indptr for p in pe]),
              "pe_indices": np.concatenate([p.col_indices for p in pe]),
              "pe_values": np.concatenate([p.col_values for p in pe])}
    shared = sparsebp.MrfModel(M, u, edges, pot, grid_shape=(H, W))
    per_edge = sparsebp.MrfModel(M, u, edges, pe, grid_shape=(H, W))
    # The grid engine's store mapping (bp.py:604-617) assumes canonically
    # oriented edges (b - a == 1 means horizontal): for a reversed edge it
    # reads the wrong slot.  The same shared potential as distinct objects
    # runs the generic engine (bp.py:652-654), whose store follows the
    # directed-edge semantics (2e: a->b) for every edge; the potential is
    # symmetric, so its orientation rule gives the same messages.
    copies = sparsebp.MrfModel(M, u, edges, [sparsebp.SparseTruncatedPotential(
        M, pot.fbar, pot.col_indptr, pot.col_indices, pot.col_values) for _ in edges],
        grid_shape=(H, W))
    arrays["reversed"] = flip
    for k, p in enumerate(sparsebp.SweepSchedule.canonical(shared).passes):
        arrays[f"pass{k}"] = p
    for tag, model in (("shared", shared), ("shared_generic", copies), ("per_edge", per_edge)):
        for dom in ("sum", "max"):
            if dom == "max" and tag == "per_edge" and not all(p.to_log().maxsum_safe for p in pe):
                continue
            store = sparsebp.run_sweeps(model, 3, kernel="fast", domain=dom)
            arrays[f"store_{tag}_{dom}"] = store.data
            man["cases"][f"{tag}_{dom}"] = {"sweeps": 3, "madds": int(store.stats.madds)}
    np.savez_compressed(OUT / "api_permuted_edges.npz", **arrays)
    with open(OUT / "manifest_api.json", "w") as f:
        json.dump(man, f, indent=1, sort_keys=True)
    print("wrote", sorted(man["cases"]))


if __name__ == "__main__":
    main()
