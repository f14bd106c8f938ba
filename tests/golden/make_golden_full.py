"""Full-size golden fixtures for the BASELINE configs (C3, C4, C5, C4 sequential).

Runs ONLY in the build container, where the reference is importable from
/root/reference/pkg/src; the outputs under ``tests/golden/full/`` are
committed and read by ``tests/test_gpu_fullsize.py`` on the GPU box.

Every number is the reference's own arithmetic at the BASELINE grid size and
iteration count:

* synchronous iterations: the reference's compiled bodies ``_grid_h_*``,
  ``_fast_*`` and ``_norm_*_store`` (numba_kernels.py:44-90,194-271) composed
  in one ``numba.prange`` Jacobi iteration over ping-pong
  ``_grid_store_init`` buffers (bp.py:587-601), weights / orientation as
  ``_grid_setup`` (bp.py:466-489).  Every (node, direction) writes its own
  target slot, so the parallel loop is bitwise identical to the serial one
  in ``make_golden.py`` (checked below on C1/C2 against the committed
  digests before any large case runs);
* the canonical sequential sweep: the reference's pass loop
  (numba_kernels.py:296-316, 364-384) with its independent lines (rows for
  L->R / R->L, columns for T->B / B->T) in ``prange``; every line is the
  reference's own in-place chain, so the sweep is bitwise identical to
  ``sparsebp.run_sweeps`` (checked below on C1/C2 against its digests);
* ``_grid_store_to_messages``, ``compute_beliefs``, ``compute_max_marginals``
  and ``map_labels`` from the reference (bp.py:604-617, 711-744).

A case records: uint8 MAP labels of every node (M <= 256), the ids and f64
top-2 gaps of every node whose gap is below a generous tie band (the test
applies its own fp32 band), 64 (C5: 32) sampled nodes' incoming messages
(4, k, M), scores / beliefs and normalisers in f64, and sha256 digests of
the full f64 arrays.

Usage:  python tests/golden/make_golden_full.py [case ...]
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

import numpy as np  # noqa: E402
from numba import njit, prange  # noqa: E402

import sparsebp  # noqa: E402
from sparsebp import numba_kernels as nk  # noqa: E402
from sparsebp.bp import _grid_store_init  # noqa: E402

from make_golden import oriented_args, ref_stereo_model  # noqa: E402

GOLD = Path(__file__).resolve().parent
OUT = GOLD / "full"
MANIFEST = OUT / "manifest_full.json"


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def sha_raw(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@njit(parallel=True)
def sync_iter_par(domain, H, W, M, vals, mi, mo, fb0, ip0, ix0, w0, fb1, ip1, ix1, w1, bad):
    """One Jacobi iteration: rows in parallel, the reference bodies per node."""
    for r in prange(H):
        h = np.empty(M, dtype=np.float64)
        out = np.empty(M, dtype=np.float64)
        for c in range(W):
            n = r * W + c
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
                if domain == 0:
                    nk._grid_h_sum(vals, mi[0], mi[1], mi[2], mi[3], n, excl, h, M)
                    if direction == 0 or direction == 2:
                        nk._fast_sum(h, fb0, ip0, ix0, w0, out, M)
                    else:
                        nk._fast_sum(h, fb1, ip1, ix1, w1, out, M)
                    ok = nk._norm_sum_store(out, mo[wdir], n + step, M)
                else:
                    nk._grid_h_max(vals, mi[0], mi[1], mi[2], mi[3], n, excl, h, M)
                    if direction == 0 or direction == 2:
                        nk._fast_max(h, fb0, ip0, ix0, w0, out, M)
                    else:
                        nk._fast_max(h, fb1, ip1, ix1, w1, out, M)
                    ok = nk._norm_max_store(out, mo[wdir], n + step, M)
                if not ok:
                    bad[r] = 1


@njit(parallel=True)
def seq_pass_par(domain, direction, H, W, M, vals, msgs, fb, ip, ix, w, bad):
    """One reference directional pass (numba_kernels.py:296-316/364-384) with
    its independent lines in parallel; each line is the reference's in-place
    chain in the reference order."""
    n_lines, line_len, line_stride, step, excl, wdir, origin = nk._grid_step(direction, H, W)
    m0, m1, m2, m3 = msgs[0], msgs[1], msgs[2], msgs[3]
    mw = msgs[wdir]
    for line in prange(n_lines):
        h = np.empty(M, dtype=np.float64)
        out = np.empty(M, dtype=np.float64)
        base = line * line_stride + origin
        for pos in range(line_len):
            src = base + pos * step
            if domain == 0:
                nk._grid_h_sum(vals, m0, m1, m2, m3, src, excl, h, M)
                nk._fast_sum(h, fb, ip, ix, w, out, M)
                ok = nk._norm_sum_store(out, mw, src + step, M)
            else:
                nk._grid_h_max(vals, m0, m1, m2, m3, src, excl, h, M)
                nk._fast_max(h, fb, ip, ix, w, out, M)
                ok = nk._norm_max_store(out, mw, src + step, M)
            if not ok:
                bad[line] = 1
                break


def run_sync(model, iters, domain):
    H, W = model.grid_shape
    vals = model.unaries if domain == "sum" else model.log_unaries
    a = _grid_store_init(model, domain)
    b = a.copy()
    o0, o1 = oriented_args(model, domain, "fast")
    bad = np.zeros(H, np.int64)
    dom = 0 if domain == "sum" else 1
    for it in range(iters):
        t = time.time()
        sync_iter_par(dom, H, W, model.M, vals, a, b, *o0[1:], *o1[1:], bad)
        assert not bad.any(), f"degenerate message at iteration {it}"
        a, b = b, a
        print(f"  sync it {it} {time.time() - t:.1f}s", flush=True)
    del b
    return a


def run_seq(model, sweeps, domain):
    H, W = model.grid_shape
    vals = model.unaries if domain == "sum" else model.log_unaries
    msgs = _grid_store_init(model, domain)
    o0, o1 = oriented_args(model, domain, "fast")
    dom = 0 if domain == "sum" else 1
    for s in range(sweeps):
        t = time.time()
        for direction in range(4):
            o = o0 if direction in (0, 2) else o1
            bad = np.zeros(max(H, W), np.int64)
            seq_pass_par(dom, direction, H, W, model.M, vals, msgs, *o[1:], bad)
            assert not bad.any(), f"degenerate message in sweep {s}"
        print(f"  seq sweep {s} {time.time() - t:.1f}s", flush=True)
    return msgs


def finish(name, model, msgs4, domain, entry, n_sample):
    """Reference post-processing + the compact record of one case."""
    store = sparsebp.bp._grid_store_to_messages(model, msgs4, domain)
    entry["msgs4_sha"] = sha(msgs4)
    entry["store_sha"] = sha(store.data)
    rng = np.random.default_rng(12345)
    nodes = np.sort(rng.choice(model.n_nodes, size=n_sample, replace=False))
    res = {"sample_nodes": nodes, "sample_msgs": np.ascontiguousarray(msgs4[:, nodes])}
    del msgs4
    if domain == "sum":
        bt = sparsebp.compute_beliefs(model, store)
        del store
        scores = bt.beliefs
        entry["beliefs_sha"] = sha(bt.beliefs)
        entry["normalizers_sha"] = sha(bt.normalizers)
        res["sample_normalizers"] = bt.normalizers[nodes]
        rel = True
    else:
        scores = sparsebp.compute_max_marginals(model, store)
        del store
        entry["scores_sha"] = sha(scores)
        rel = False
    labels = sparsebp.map_labels(scores)
    entry["labels_sha"] = sha_raw(labels.astype(np.int64))
    top2 = np.partition(scores, model.M - 2, axis=1)[:, -2:]
    gap = top2[:, 1] - top2[:, 0]
    band = 1e-3 * scores.max(axis=1) if rel else np.full(len(gap), 1e-2)
    near = np.flatnonzero(gap <= band)
    entry["n_near_tie"] = int(near.size)
    entry["label_hist"] = np.bincount(labels, minlength=model.M).tolist()
    res.update(labels=labels.astype(np.uint8), near_nodes=near, near_gap=gap[near],
               near_rowmax=scores.max(axis=1)[near], sample_scores=scores[nodes])
    np.savez_compressed(OUT / f"{name}.npz", **res)
    return entry


CASES = {
    # name: (config, domain, schedule, iterations, sampled nodes)
    "C3_sync_max": ("C3", "max", "sync", 100, 64),
    "C4_sync_sum": ("C4", "sum", "sync", 100, 64),
    "C4_seq_sum": ("C4", "sum", "seq", 50, 64),
}
for _T in (2, 5, 9, 17, 33):
    for _d in ("sum", "max"):
        CASES[f"C5_T{_T}_sync_{_d}"] = (f"C5_T{_T}", _d, "sync", 20, 32)


def build(cfg_name):
    from paper_1010_0012_b200 import synth
    cfg = synth.CONFIGS[cfg_name]
    t = time.time()
    model, _, _ = ref_stereo_model(cfg.height, cfg.width, cfg.M, cfg.alpha, cfg.T, cfg.sigma, 0,
                                   potential=cfg.potential)
    print(f"  built {cfg_name} in {time.time() - t:.1f}s", flush=True)
    return model


def self_check(man):
    """prange compositions == committed digests of the serial composition /
    the reference run_sweeps (C1 and C2)."""
    small = json.load(open(GOLD / "manifest.json"))["cases"]
    c1 = ref_stereo_model(48, 64, 16, 1.0, 2.0, 5.0, 0)[0]
    c2 = ref_stereo_model(288, 384, 32, 0.5, 3.0, 5.0, 0)[0]
    for name, model, dom, it in [("C1_sync_sum", c1, "sum", 10), ("C1_sync_max", c1, "max", 10),
                                 ("C2_sync_sum", c2, "sum", 50), ("C2_sync_max", c2, "max", 50)]:
        assert sha(run_sync(model, it, dom)) == small[name]["msgs4_sha"], name
    for name, dom in [("seq_C1_sum_fast", "sum"), ("seq_C1_max_fast", "max")]:
        msgs = run_seq(c1, 10, dom)
        store = sparsebp.bp._grid_store_to_messages(c1, msgs, dom)
        assert sha(store.data) == small[name]["store_sha"], name
    # and directly against the reference's own run_sweeps on C2 (3 sweeps)
    ref = sparsebp.run_sweeps(c2, 3, kernel="fast", domain="sum")
    mine = sparsebp.bp._grid_store_to_messages(c2, run_seq(c2, 3, "sum"), "sum")
    assert np.array_equal(ref.data, mine.data)
    man["self_check"] = "prange sync == serial composition (C1, C2 both domains); " \
                        "prange seq == reference run_sweeps (C1 10 sweeps, C2 3 sweeps)"
    print("self-check passed", flush=True)


def main(argv):
    OUT.mkdir(exist_ok=True)
    man = json.load(open(MANIFEST)) if MANIFEST.exists() else {
        "generator": "tests/golden/make_golden_full.py", "cases": {}}
    names = argv or list(CASES)
    if "self_check" not in man:
        self_check(man)
        json.dump(man, open(MANIFEST, "w"), indent=1, sort_keys=True)
    models = {}
    for name in names:
        cfg_name, dom, sched, iters, ns = CASES[name]
        print(f"case {name}", flush=True)
        if cfg_name not in models:
            models.clear()
            models[cfg_name] = build(cfg_name)
        model = models[cfg_name]
        t = time.time()
        msgs4 = run_sync(model, iters, dom) if sched == "sync" else run_seq(model, iters, dom)
        entry = {"config": cfg_name, "domain": dom, "schedule": sched, "iters": iters,
                 "grid": list(model.grid_shape), "M": model.M, "seed": 0,
                 "run_seconds_8_threads": round(time.time() - t, 1)}
        man["cases"][name] = finish(name, model, msgs4, dom, entry, ns)
        del msgs4
        json.dump(man, open(MANIFEST, "w"), indent=1, sort_keys=True)
        print(f"  wrote {name} ({entry['n_near_tie']} near-tie nodes)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
