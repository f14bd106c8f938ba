"""Generate the golden fixtures that pin the CPU oracle to the reference.

Runs ONLY in the build container, where the reference package is importable
from /root/reference/pkg/src (it does not exist on the GPU box; the outputs
are committed under tests/golden/).  Usage:

    python tests/golden/make_golden.py

What it records, all computed by the reference's own code:

* synchronous (Jacobi) iterations composed from the reference's compiled
  update bodies ``_grid_h_{sum,max}``, ``_std_*``, ``_fast_*``, ``_pruned_*``
  and ``_norm_*_store`` (numba_kernels.py:35-101,194-271) inside one numba
  function over ping-pong ``_grid_store_init`` buffers (bp.py:587-601), with
  the orientation / weight choice of ``_grid_setup`` (bp.py:466-489);
* the reference's public ``run_sweeps`` (canonical sequential schedule),
  ``compute_beliefs``, ``compute_max_marginals`` and ``map_labels``;
* ``enumerate_exact`` marginals on chains (oracle.py:59-119);
* potentials, stereo images and unary fields built by the reference
  (mrf.py:207-285, stereo.py:82-183) from this repo's seeded generator.

Small cases store full f64 arrays; large ones store sha256 digests of the
f64 bytes (the oracle must reproduce them bit-for-bit) plus labels.
The reference tree is never written: numba's cache goes to /tmp and
bytecode writing is disabled.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
from numba import njit  # noqa: E402

import sparsebp  # noqa: E402
from sparsebp import synth as ref_synth  # noqa: E402
from sparsebp import numba_kernels as nk  # noqa: E402
from sparsebp.bp import _grid_store_init  # noqa: E402
from sparsebp.stereo import GrayImage, StereoParams  # noqa: E402

from paper_1010_0012_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def sha_raw(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------------------
# synchronous schedule composed from the reference bodies
# ---------------------------------------------------------------------------

@njit
def _h(domain, vals, mi, n, excl, h, M):
    if domain == 0:
        nk._grid_h_sum(vals, mi[0], mi[1], mi[2], mi[3], n, excl, h, M)
    else:
        nk._grid_h_max(vals, mi[0], mi[1], mi[2], mi[3], n, excl, h, M)


@njit
def _upd(domain, kernel, h, tT, fb, ip, ix, w, out, M):
    if domain == 0:
        if kernel == 0:
            nk._std_sum(h, tT, out, M)
        elif kernel == 1:
            nk._fast_sum(h, fb, ip, ix, w, out, M)
        else:
            nk._pruned_sum(h, ip, ix, w, out, M)
    else:
        if kernel == 0:
            nk._std_max(h, tT, out, M)
        elif kernel == 1:
            nk._fast_max(h, fb, ip, ix, w, out, M)
        else:
            nk._pruned_max(h, ip, ix, w, out, M)


@njit
def sync_iter(domain, kernel, H, W, M, vals, mi, mo,
              t0, fb0, ip0, ix0, w0, t1, fb1, ip1, ix1, w1, fails):
    h = np.empty(M, dtype=np.float64)
    out = np.empty(M, dtype=np.float64)
    nf = 0
    for n in range(H * W):
        r = n // W
        c = n % W
        for direction in range(4):
            if direction == 0:
                exists = c + 1 < W
            elif direction == 1:
                exists = c > 0
            elif direction == 2:
                exists = r + 1 < H
            else:
                exists = r > 0
            if not exists:
                continue
            _nl, _ll, _ls, step, excl, wdir, _o = nk._grid_step(direction, H, W)
            _h(domain, vals, mi, n, excl, h, M)
            if direction == 0 or direction == 2:
                _upd(domain, kernel, h, t0, fb0, ip0, ix0, w0, out, M)
            else:
                _upd(domain, kernel, h, t1, fb1, ip1, ix1, w1, out, M)
            if domain == 0:
                ok = nk._norm_sum_store(out, mo[wdir], n + step, M)
            else:
                ok = nk._norm_max_store(out, mo[wdir], n + step, M)
            if not ok and nf < fails.shape[0]:
                fails[nf, 0] = n
                fails[nf, 1] = direction
                nf += 1
    return nf


KID = {"standard": 0, "fast": 1, "pruned": 2}


@njit
def generic_sync_iter(domain, kernel, M, src, rev, opid, in_indptr, in_eids, vals, old, new,
                      tablesT, fbars, indptrs, indices_flat, values_flat, residuals_flat, fails):
    """One synchronous iteration over every directed edge, composed from the
    reference generic engine's own bodies (numba_kernels.py:422-485)."""
    h = np.empty(M, dtype=np.float64)
    out = np.empty(M, dtype=np.float64)
    nf = 0
    for d in range(src.shape[0]):
        q = opid[d]
        nk._generic_h(vals, old, in_indptr, in_eids, src[d], rev[d], h, M, domain == 1)
        if domain == 0:
            if kernel == 0:
                nk._std_sum(h, tablesT[q], out, M)
            elif kernel == 1:
                nk._fast_sum(h, fbars[q], indptrs[q], indices_flat, residuals_flat, out, M)
            else:
                nk._pruned_sum(h, indptrs[q], indices_flat, values_flat, out, M)
            ok = nk._normalize_sum_into(out, new[d], M)
        else:
            if kernel == 0:
                nk._std_max(h, tablesT[q], out, M)
            elif kernel == 1:
                nk._fast_max(h, fbars[q], indptrs[q], indices_flat, values_flat, out, M)
            else:
                nk._pruned_max(h, indptrs[q], indices_flat, values_flat, out, M)
            ok = nk._normalize_max_into(out, new[d], M)
        if not ok and nf < fails.shape[0]:
            fails[nf] = d
            nf += 1
    return nf


def ref_generic_sync_run(model, iters, domain, kernel):
    eng = sparsebp.bp._GenericEngine(model, kernel, domain)
    a = sparsebp.MessageStore(model, domain).data.copy()
    b = a.copy()
    fails = np.zeros(64, dtype=np.int64)
    for _ in range(iters):
        nf = generic_sync_iter(0 if domain == "sum" else 1, KID[kernel], model.M, eng.src,
                               eng.rev, eng.opid, eng.in_indptr, eng.in_eids, eng.values_in, a,
                               b, eng.tablesT, eng.fbars, eng.indptrs, eng.indices_flat,
                               eng.values_flat, eng.residuals_flat, fails)
        assert nf == 0
        a, b = b, a
    return a


def save_per_edge(name, model, results):
    pots = model.potentials
    M = model.M
    arrays = {"unaries": np.asarray(model.unaries), "log_unaries": np.asarray(model.log_unaries),
              "grid_shape": np.array(model.grid_shape),
              "pe_fbar": np.array([p.fbar for p in pots]),
              "pe_indptr": np.stack([p.col_indptr for p in pots]),
              "pe_indices": np.concatenate([p.col_indices for p in pots]),
              "pe_values": np.concatenate([p.col_values for p in pots])}
    arrays.update(results)
    np.savez_compressed(OUT / f"{name}.npz", **arrays)


def add_per_edge_cases(tag, model, sweeps):
    for dom in ("sum", "max"):
        for ker in ("fast", "standard"):
            data = ref_generic_sync_run(model, sweeps, dom, ker)
            name = f"pe_sync_{tag}_{dom}_{ker}"
            save_per_edge(name, model, {"store": data})
            manifest["cases"][name] = {"kind": "pe_sync", "domain": dom, "kernel": ker,
                                       "iters": sweeps, "store_sha": sha(data),
                                       "grid": list(model.grid_shape), "M": model.M}
            store = sparsebp.run_sweeps(model, sweeps, kernel=ker, domain=dom)
            name = f"pe_seq_{tag}_{dom}_{ker}"
            save_per_edge(name, model, {"store": store.data})
            manifest["cases"][name] = {"kind": "pe_seq", "domain": dom, "kernel": ker,
                                       "sweeps": sweeps, "store_sha": sha(store.data),
                                       "madds": int(store.stats.madds),
                                       "grid": list(model.grid_shape), "M": model.M}


def oriented_args(model, domain, kernel):
    """Mirror of bp._grid_setup (bp.py:466-489) as flat argument tuples."""
    pot = model.potentials[0].to_log() if domain == "max" else model.potentials[0]
    M = model.M
    dummy_t = np.zeros((1, 1))
    dummy = (0.0, np.zeros(M + 1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    if kernel == "standard":
        table = pot.densify().table if hasattr(pot, "densify") else pot.table
        return [(np.ascontiguousarray(table.T),) + dummy, (np.ascontiguousarray(table),) + dummy]
    out = []
    for p in (pot, pot.transpose()):
        if kernel == "fast":
            w = p.col_residuals if domain == "sum" else p.col_values
        else:
            w = p.col_values
        out.append((dummy_t, p.fbar, p.col_indptr, p.col_indices, np.ascontiguousarray(w)))
    return out


def ref_sync_run(model, iters, domain, kernel):
    H, W = model.grid_shape
    M = model.M
    vals = model.unaries if domain == "sum" else model.log_unaries
    a = _grid_store_init(model, domain)
    if model.n_edges == 0:          # run_sweeps returns immediately (bp.py:656-659)
        return a, None
    b = a.copy()
    o0, o1 = oriented_args(model, domain, kernel)
    fails = np.zeros((64, 2), dtype=np.int64)
    for it in range(iters):
        nf = sync_iter(0 if domain == "sum" else 1, KID[kernel], H, W, M, vals, a, b,
                       *o0, *o1, fails)
        if nf:
            return a, {"iteration": it, "fails": fails[:nf].tolist()}
        a, b = b, a
    return a, None


# ---------------------------------------------------------------------------
# model builders (reference objects)
# ---------------------------------------------------------------------------

def ref_stereo_model(H, W, M, alpha, T, sigma, seed, potential="linear"):
    left, right, _ = synth.noisy_stereo_pair(H, W, M, sigma, seed)
    params = StereoParams(M=M, alpha=alpha, T_b=T if potential == "linear" else 2.0,
                          beta=0.1, T_u=255.0)
    unaries, log_unaries = sparsebp.stereo_unary_field(GrayImage(left), GrayImage(right), params)
    if potential == "linear":
        pot = sparsebp.truncated_linear_potential(M, alpha, T)
    else:
        d = np.abs(np.arange(M)[:, None] - np.arange(M)[None, :]).astype(np.float64)
        table = np.exp(-alpha * np.minimum(d * d, T))
        pot = sparsebp.sparse_from_dense(table, fbar=table[0, -1])
    model = sparsebp.build_grid_mrf(H, W, M, unaries, pot, log_unary_provider=log_unaries)
    return model, left, right


def model_inputs(model):
    """Arrays a test needs to rebuild the same model without the reference."""
    base = {
        "unaries": np.asarray(model.unaries),
        "log_unaries": np.asarray(model.log_unaries),
        "grid_shape": np.array(model.grid_shape),
    }
    if model.n_edges == 0:
        return base
    pot = model.potentials[0]
    return {
        **base,
        "fbar": np.array(pot.fbar),
        "col_indptr": pot.col_indptr,
        "col_indices": pot.col_indices,
        "col_values": pot.col_values,
        "log_fbar": np.array(pot.to_log().fbar),
        "log_col_values": pot.to_log().col_values,
    }


def save_full(name, model, results):
    arrays = dict(model_inputs(model))
    arrays.update(results)
    np.savez_compressed(OUT / f"{name}.npz", **arrays)


manifest: dict = {"generator": "tests/golden/make_golden.py", "cases": {}}


def add_sync_case(name, model, domain, kernel, iters, full=True):
    msgs4, fail = ref_sync_run(model, iters, domain, kernel)
    entry = {"kind": "sync", "domain": domain, "kernel": kernel, "iters": iters,
             "grid": list(model.grid_shape), "M": model.M}
    if fail is not None:
        store = sparsebp.MessageStore(model, domain)
        ids = sorted(store.edge_id(int(n), int(n + {0: 1, 1: -1, 2: model.grid_shape[1],
                                                       3: -model.grid_shape[1]}[d]))
                     for n, d in fail["fails"])
        entry["degenerate"] = {"iteration": fail["iteration"], "directed_edge_ids": ids}
        save_full(name, model, {})
        manifest["cases"][name] = entry
        return
    store = sparsebp.bp._grid_store_to_messages(model, msgs4, domain)
    entry["msgs4_sha"] = sha(msgs4)
    entry["store_sha"] = sha(store.data)
    res = {}
    if domain == "sum":
        bt = sparsebp.compute_beliefs(model, store)
        labels = sparsebp.map_labels(bt)
        entry["beliefs_sha"] = sha(bt.beliefs)
        entry["normalizers_sha"] = sha(bt.normalizers)
        scores = bt.beliefs
    else:
        scores = sparsebp.compute_max_marginals(model, store)
        labels = sparsebp.map_labels(scores)
        entry["scores_sha"] = sha(scores)
    entry["labels_sha"] = sha_raw(labels.astype(np.int64))
    if full:
        res = {"msgs4": msgs4, "store": store.data, "scores": scores, "labels": labels}
        if domain == "sum":
            res["normalizers"] = bt.normalizers
        save_full(name, model, res)
    else:
        gap = np.partition(scores, model.M - 2, axis=1)
        gap = gap[:, -1] - gap[:, -2]
        rng = np.random.default_rng(0)
        rows = np.sort(rng.choice(model.n_nodes, size=min(64, model.n_nodes), replace=False))
        np.savez_compressed(OUT / f"{name}.npz", labels=labels.astype(np.int16),
                            top2_gap=gap.astype(np.float32), sample_nodes=rows,
                            sample_msgs=msgs4[:, rows], sample_scores=scores[rows])
    manifest["cases"][name] = entry


def add_seq_case(name, model, domain, kernel, sweeps, full=True):
    entry = {"kind": "seq", "domain": domain, "kernel": kernel, "sweeps": sweeps,
             "grid": list(model.grid_shape), "M": model.M}
    try:
        store = sparsebp.run_sweeps(model, sweeps, kernel=kernel, domain=domain)
    except sparsebp.DegenerateMessageError as exc:
        entry["degenerate_edge"] = list(exc.edge)
        save_full(name, model, {})
        manifest["cases"][name] = entry
        return
    entry["store_sha"] = sha(store.data)
    entry["madds"] = int(store.stats.madds)
    if domain == "sum":
        bt = sparsebp.compute_beliefs(model, store)
        entry["beliefs_sha"] = sha(bt.beliefs)
        scores = bt.beliefs
    else:
        scores = sparsebp.compute_max_marginals(model, store)
        entry["scores_sha"] = sha(scores)
    labels = sparsebp.map_labels(scores)
    entry["labels_sha"] = sha_raw(labels.astype(np.int64))
    if full:
        save_full(name, model, {"store": store.data, "scores": scores, "labels": labels})
    manifest["cases"][name] = entry


def main():
    # --- seeded generator vs the reference's random_dot_pair -----------------
    gen = {}
    for (H, W, M, seed) in [(48, 64, 16, 0), (288, 384, 32, 0), (768, 1024, 64, 0),
                            (1536, 2048, 128, 0), (1024, 1024, 256, 0), (10, 14, 8, 3)]:
        disp = synth.rect_disparity(H, W, M, np.random.default_rng(seed))
        lref, rref = sparsebp.random_dot_pair(H, W, disp, seed=seed + 1)
        lmine, rmine = synth.random_dot_pair(H, W, disp, seed=seed + 1)
        assert np.array_equal(lref.pixels, lmine) and np.array_equal(rref.pixels, rmine)
        gen[f"{H}x{W}_M{M}_s{seed}"] = {"left": sha_raw(lref.pixels),
                                         "right": sha_raw(rref.pixels),
                                         "disp": sha_raw(disp)}
    manifest["random_dot_pair"] = gen

    # --- potentials (reference constructors) ----------------------------------
    pots = {}
    for (M, alpha, T) in [(16, 1.0, 2.0), (32, 0.5, 3.0), (128, 0.5, 8.0), (256, 0.5, 2.0),
                          (256, 0.5, 5.0), (256, 0.5, 9.0), (256, 0.5, 17.0), (256, 0.5, 33.0),
                          (5, 1.0, 2.0), (13, 0.7, 3.0), (8, 1.0, 2.5), (7, 1e-9, 3.0)]:
        p = sparsebp.truncated_linear_potential(M, alpha, T)
        t = p.transpose()
        lg = p.to_log()
        pots[f"linear_M{M}_a{alpha}_T{T}"] = {
            "fbar": p.fbar, "nnz": p.nnz, "m": p.m,
            "indptr": sha_raw(p.col_indptr), "indices": sha_raw(p.col_indices),
            "values": sha(p.col_values), "residuals": sha(p.col_residuals),
            "t_indptr": sha_raw(t.col_indptr), "t_indices": sha_raw(t.col_indices),
            "t_values": sha(t.col_values), "log_fbar": lg.fbar, "log_values": sha(lg.col_values),
            "dense": sha(p.densify().table)}
    for (M, alpha, cap) in [(64, 0.2, 16.0), (16, 0.2, 16.0)]:
        d = np.abs(np.arange(M)[:, None] - np.arange(M)[None, :]).astype(np.float64)
        table = np.exp(-alpha * np.minimum(d * d, cap))
        p = sparsebp.sparse_from_dense(table, fbar=table[0, -1])
        t = p.transpose()
        lg = p.to_log()
        pots[f"quadratic_M{M}_a{alpha}_cap{cap}"] = {
            "fbar": p.fbar, "nnz": p.nnz, "m": p.m, "maxsum_safe": lg.maxsum_safe,
            "indptr": sha_raw(p.col_indptr), "indices": sha_raw(p.col_indices),
            "values": sha(p.col_values), "residuals": sha(p.col_residuals),
            "t_indptr": sha_raw(t.col_indptr), "t_indices": sha_raw(t.col_indices),
            "t_values": sha(t.col_values), "log_fbar": lg.fbar, "log_values": sha(lg.col_values),
            "dense": sha(p.densify().table)}
    manifest["potentials"] = pots

    # --- stereo unary fields ---------------------------------------------------
    uni = {}
    for name, (H, W, M, sigma, seed) in {"C1": (48, 64, 16, 5.0, 0), "C2": (288, 384, 32, 5.0, 0),
                                         "C3": (768, 1024, 64, 10.0, 0),
                                         "small": (10, 14, 8, 5.0, 3)}.items():
        left, right, _ = synth.noisy_stereo_pair(H, W, M, sigma, seed)
        u, lu = sparsebp.stereo_unary_field(GrayImage(left), GrayImage(right),
                                            StereoParams(M=M, beta=0.1, T_u=255.0))
        uni[name] = {"unaries": sha(u), "log_unaries": sha(lu), "right": sha_raw(right)}
    manifest["unaries"] = uni

    # --- synchronous cases, small (full arrays) ------------------------------
    small, _, _ = ref_stereo_model(10, 14, 8, 1.0, 2.0, 5.0, 3)
    for dom in ("sum", "max"):
        for ker in ("fast", "standard", "pruned"):
            add_sync_case(f"sync_small_{dom}_{ker}", small, dom, ker, 6)
    quad, _, _ = ref_stereo_model(9, 11, 16, 0.2, 16.0, 10.0, 5, potential="quadratic")
    add_sync_case("sync_quad_max", quad, "max", "fast", 8)
    add_sync_case("sync_quad_sum", quad, "sum", "fast", 8)
    oddm, _, _ = ref_stereo_model(7, 19, 13, 0.7, 3.0, 5.0, 7)
    add_sync_case("sync_oddM_sum", oddm, "sum", "fast", 7)
    add_sync_case("sync_oddM_max", oddm, "max", "fast", 7)
    wide, _, _ = ref_stereo_model(6, 40, 37, 0.3, 9.0, 5.0, 11)
    add_sync_case("sync_wide_sum", wide, "sum", "fast", 5)
    add_sync_case("sync_wide_max", wide, "max", "fast", 5)
    for k in range(4):
        rng = np.random.default_rng(100 + k)
        rm = ref_synth.random_grid_model(rng, max_side=8, max_M=24, shared_potential=True)
        for dom in ("sum", "max"):
            add_sync_case(f"sync_random{k}_{dom}", rm, dom, "fast", 5)
    for (H, W) in [(1, 9), (9, 1), (1, 1), (2, 2)]:
        rng = np.random.default_rng(H * 31 + W)
        g = rng.uniform(0.1, 1.0, size=(H * W, 4))
        m = sparsebp.build_grid_mrf(H, W, 4, g, sparsebp.truncated_linear_potential(4, 1.0, 2.0))
        for dom in ("sum", "max"):
            add_sync_case(f"sync_grid{H}x{W}_{dom}", m, dom, "fast", 12)

    # degenerate: message 0->1 of a 1x2 grid is all-zero (fbar = 0, pruned support)
    pot = sparsebp.SparseTruncatedPotential(2, 0.0, np.array([0, 1, 2]), np.array([1, 1]),
                                            np.array([1.0, 1.0]))
    deg = sparsebp.build_grid_mrf(1, 2, 2, np.array([[1.0, 0.0], [1.0, 1.0]]), pot)
    add_sync_case("sync_degenerate_sum", deg, "sum", "fast", 3)
    add_seq_case("seq_degenerate_sum", deg, "sum", "fast", 3)
    # the same failure with a banded (Toeplitz) potential: only d = +1 is stored
    bpot = sparsebp.SparseTruncatedPotential(2, 0.0, np.array([0, 1, 1]), np.array([1]),
                                             np.array([1.0]))
    bdeg = sparsebp.build_grid_mrf(2, 3, 2, np.array([[1.0, 0.0]] * 6), bpot)
    add_sync_case("sync_degenerate_band_sum", bdeg, "sum", "fast", 3)
    add_seq_case("seq_degenerate_band_sum", bdeg, "sum", "fast", 3)

    # --- chains vs exact enumeration (BP is exact on trees) ------------------
    for (W, M, seed) in [(6, 3, 1), (5, 4, 2)]:
        rng = np.random.default_rng(seed)
        g = rng.uniform(0.1, 1.0, size=(W, M))
        chain = sparsebp.build_grid_mrf(1, W, M, g, sparsebp.truncated_linear_potential(M, 0.8, 2.0))
        ex = sparsebp.enumerate_exact(chain)
        name = f"chain_exact_W{W}_M{M}"
        save_full(name, chain, {"marginals": ex.marginals, "map_config": ex.map_config})
        manifest["cases"][name] = {"kind": "exact", "grid": [1, W], "M": M,
                                   "map_unique": bool(ex.map_unique), "log_Z": ex.log_Z}

    # --- per-edge (inhomogeneous) potentials: the reference generic engine -----
    for k in range(3):
        rng = np.random.default_rng(200 + k)
        pm = ref_synth.random_grid_model(rng, max_side=7, max_M=20, shared_potential=False)
        add_per_edge_cases(f"r{k}", pm, 4)

    # --- BASELINE C1 / C2 (digests + labels) --------------------------------
    c1, _, _ = ref_stereo_model(48, 64, 16, 1.0, 2.0, 5.0, 0)
    add_sync_case("C1_sync_sum", c1, "sum", "fast", 10, full=False)
    add_sync_case("C1_sync_max", c1, "max", "fast", 10, full=False)
    add_sync_case("C1_sync_sum_standard", c1, "sum", "standard", 10, full=False)
    c2, _, _ = ref_stereo_model(288, 384, 32, 0.5, 3.0, 5.0, 0)
    add_sync_case("C2_sync_sum", c2, "sum", "fast", 50, full=False)
    add_sync_case("C2_sync_max", c2, "max", "fast", 50, full=False)

    # --- reference canonical (sequential) schedule ---------------------------
    for dom in ("sum", "max"):
        add_seq_case(f"seq_small_{dom}_fast", small, dom, "fast", 3)
        add_seq_case(f"seq_small_{dom}_standard", small, dom, "standard", 3)
    add_seq_case("seq_C1_sum_fast", c1, "sum", "fast", 10, full=False)
    add_seq_case("seq_C1_max_fast", c1, "max", "fast", 10, full=False)

    with open(OUT / "manifest.json", "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
    print(f"wrote {len(manifest['cases'])} cases to {OUT}")


if __name__ == "__main__":
    main()
