"""Reference constructor surface without a GPU: ``MrfModel`` with the
reference signature (mrf.py:298-369), its validation, arbitrary edge order /
orientation, and ``SweepSchedule`` (bp.py:190-234), pinned to fixtures made
by the reference itself (tests/golden/make_golden_api.py)."""

import numpy as np
import pytest

import paper_1010_0012_b200 as sbp
from golden_util import GOLDEN
from paper_1010_0012_b200.model import (MrfModel, SparseTruncatedPotential, SweepSchedule,
                                        edge_mapping, grid_edges, model_directed_ids)

Z = np.load(GOLDEN / "api_permuted_edges.npz")


def _pot():
    M = Z["unaries"].shape[1]
    return SparseTruncatedPotential(M, float(Z["pot_fbar"]), Z["pot_indptr"], Z["pot_indices"],
                                    Z["pot_values"])


def test_exports():
    assert sbp.MrfModel is MrfModel and sbp.SweepSchedule is SweepSchedule
    assert not hasattr(sbp, "disparity_to_image")


def test_reference_signature_and_canonical_schedule():
    H, W = (int(v) for v in Z["grid_shape"])
    model = sbp.MrfModel(Z["unaries"].shape[1], Z["unaries"], Z["edges"], _pot(),
                         grid_shape=(H, W))
    np.testing.assert_array_equal(model.edges, Z["edges"])
    assert model.n_edges == len(Z["edges"]) and model.n_nodes == H * W
    sched = sbp.SweepSchedule.canonical(model)
    assert sched.grid_canonical
    for k in range(4):
        np.testing.assert_array_equal(sched.passes[k], Z[f"pass{k}"])
    assert sched.n_updates_per_sweep == 2 * model.n_edges


def test_edge_mapping_roundtrip():
    H, W = (int(v) for v in Z["grid_shape"])
    model = sbp.MrfModel(Z["unaries"].shape[1], Z["unaries"], Z["edges"], _pot(),
                         grid_shape=(H, W))
    perm, flip = edge_mapping(model)
    canon = grid_edges(H, W)
    e = Z["edges"]
    np.testing.assert_array_equal(np.sort(e, axis=1), canon[perm])
    np.testing.assert_array_equal(flip, Z["reversed"])
    # canonical directed id -> model id sends a -> b to the model edge's (a, b) direction
    cid = np.arange(2 * len(canon))
    mid = model_directed_ids(model, cid)
    src_c = np.where(cid % 2 == 0, canon[cid // 2, 0], canon[cid // 2, 1])
    src_m = np.where(mid % 2 == 0, e[mid // 2, 0], e[mid // 2, 1])
    np.testing.assert_array_equal(src_c, src_m)
    store = sbp.MessageStore(model, "sum")
    for d in (0, 1, 17, 2 * len(e) - 1):
        assert store.edge_id(*store.endpoints(d)) == d


@pytest.mark.parametrize("bad,msg", [
    (dict(grid_shape=(4, 4)), "does not match"),
    (dict(edges="drop"), "4-connected"),
    (dict(edges="dup"), "duplicate"),
    (dict(edges="self"), "self-edges"),
    (dict(unaries="neg"), "nonnegative"),
])
def test_validation_matches_reference_messages(bad, msg):
    H, W = (int(v) for v in Z["grid_shape"])
    u = Z["unaries"].copy()
    e = Z["edges"].copy()
    gs = bad.get("grid_shape", (H, W))
    if bad.get("edges") == "drop":
        e = e[:-1]
    elif bad.get("edges") == "dup":
        e = np.concatenate([e[:-1], e[:1, ::-1]])
    elif bad.get("edges") == "self":
        e[0] = (3, 3)
    if bad.get("unaries") == "neg":
        u[2, 1] = -1.0
    with pytest.raises(ValueError, match=msg):
        sbp.MrfModel(u.shape[1], u, e, _pot() if bad.get("edges") != "drop"
                     else [_pot()] * len(e), grid_shape=gs)


def test_generic_model_constructs_but_gpu_path_refuses():
    u = Z["unaries"][:4]
    m = sbp.MrfModel(u.shape[1], u, [(0, 1), (1, 2), (2, 3), (0, 3)], _pot())
    assert m.grid_shape is None and m.n_edges == 4
    with pytest.raises(NotImplementedError):
        sbp.run_sweeps(m, 2)
