"""Memory-safety and race checks of every kernel family without
compute-sanitizer (closed on this GPU pool: runs under it left GPUs needing a
reset).  For each family (register / TMA-staged / rolled / shared-memory-tap
band kernels, temporal blocking, the sequential chain kernel, ELL in f32 and
f64, the dense comparison kernel, the fused convergence test):

* guard zones: the value table and both message buffers are views into
  larger allocations whose margins hold a sentinel; after the run the margins
  must be untouched (no out-of-bounds write) -- and because the margins are
  NaN, an out-of-bounds read would poison the messages, which must stay finite
  and match the f64 oracle;
* write coverage: the buffer an iteration writes is filled with the sentinel
  first; afterwards every real message slot holds a finite, normalised
  message and every ghost slot / halo row still holds what it held (each
  kernel writes exactly the slots it owns);
* races: three runs with different launch geometries (resident-block caps)
  and the default give identical bits.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import paper_1010_0012_b200 as sbp  # noqa: E402
from paper_1010_0012_b200 import _lib as L  # noqa: E402
from paper_1010_0012_b200 import synth  # noqa: E402
from paper_1010_0012_b200.engine import SEQUENTIAL, SYNCHRONOUS, GridEngine  # noqa: E402

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

GUARD = 1 << 16    # floats of margin on each side
SENT = float("nan")

FAMILIES = [
    # id, config, domain, schedule, env, kernel, potential kind
    ("band_reg", "C1", "sum", SYNCHRONOUS, {}, "fast", None),
    ("band_staged", "C3", "max", SYNCHRONOUS, {}, "fast", None),
    ("band_rolled", "C4", "sum", SYNCHRONOUS, {"SBP_TAP": "0"}, "fast", None),
    ("tap_c4", "C4", "sum", SYNCHRONOUS, {}, "fast", None),     # R = 7 padded to the R = 8 tap kernel
    ("tap_reg", "C5_T9", "sum", SYNCHRONOUS, {"SBP_TAP": "1", "SBP_TAP_STAGED": "0"}, "fast", None),
    ("tap_staged", "C5_T17", "max", SYNCHRONOUS, {"SBP_TAP": "1", "SBP_TAP_VL": "8",
                                                   "SBP_TAP_STAGED": "1"}, "fast", None),
    ("tap2", "C5_T33", "max", SYNCHRONOUS, {"SBP_TAP": "1", "SBP_TAP_VL": "8",
                                             "SBP_TAP_STAGED": "2"}, "fast", None),
    ("fused", "C5_T2", "sum", SYNCHRONOUS, {"SBP_FUSE": "3"}, "fast", None),
    ("chain", "C4", "sum", SEQUENTIAL, {}, "fast", None),
    ("chain_max", "C2", "max", SEQUENTIAL, {}, "fast", None),
    ("dense", "C3", "sum", SYNCHRONOUS, {}, "standard", None),
    ("dense_simt_m128", "C4", "sum", SYNCHRONOUS, {"SBP_DENSE_TC": "0"}, "standard", None),
    ("dense_tc", "C4", "sum", SYNCHRONOUS, {}, "standard", None),          # tcgen05, one CTA
    ("dense_tc_pair", "C5_T9", "sum", SYNCHRONOUS, {}, "standard", None),  # tcgen05, CTA pair
    ("ell", "C2", "sum", SYNCHRONOUS, {}, "fast", "ell"),
    ("ell_f64", "C2", "sum", SYNCHRONOUS, {"SBP_PRECISION": "f64"}, "fast", "ell"),
    ("ell_chain", "C2", "max", SEQUENTIAL, {}, "fast", "ell"),
]


def _model(name, kind):
    H, W = (13, 21) if synth.CONFIGS[name].M >= 128 else (17, 26)
    m = synth.build_config_model(synth.CONFIGS[name], height=H, width=W)
    if kind == "ell":
        d = m.shared_potential.densify().table.copy()
        d[2, 4] = 0.5 * (d[2, 4] + 1.0)
        m = sbp.GridMrf(H, W, m.M, m.unaries, sbp.sparse_from_dense(d, fbar=m.shared_potential.fbar),
                        log_unaries=m.log_unaries)
    return m


@pytest.fixture
def env(monkeypatch):
    def apply(values):
        for k, v in values.items():
            monkeypatch.setenv(k, v)
        L.lib().sbp_reload_config()
    yield apply
    monkeypatch.undo()
    L.lib().sbp_reload_config()


def _guarded(t: torch.Tensor):
    """A NaN-margined copy of t: (big, view)."""
    big = torch.full((t.numel() + 2 * GUARD,), SENT, dtype=t.dtype, device=t.device)
    view = big[GUARD:GUARD + t.numel()].view(t.shape)
    view.copy_(t)
    return big, view


def _margins_intact(big):
    m = torch.cat([big[:GUARD], big[-GUARD:]])
    return bool(torch.isnan(m).all())


@pytest.mark.parametrize("fam", FAMILIES, ids=[f[0] for f in FAMILIES])
def test_guard_zones_and_write_coverage(fam, env):
    _, name, dom, sched, variant, kernel, kind = fam
    env(variant)
    model = _model(name, kind)
    eng = GridEngine(model, dom, kernel, schedule=sched)
    bigs = []
    for i in range(2):
        big, view = _guarded(eng.msgs[i])
        eng.msgs[i] = view
        bigs.append(big)
    bigv, eng.values = _guarded(eng.values)
    eng.reset(full=True)
    M, W = model.M, model.grid_shape[1]
    rows = eng.rows
    # write coverage, one iteration: poison everything the iteration may write
    cur = eng.current
    if sched == SYNCHRONOUS and eng.fuse < 2:
        nxt = eng.msgs[1 - eng.cur]
        keep = nxt.clone()
        real = torch.ones(4, rows + 2, W, dtype=torch.bool, device=nxt.device)
        real[:, 0], real[:, rows + 1] = False, False
        H = model.grid_shape[0]
        real[0, 1, :] = False          # ghost slots of border nodes (bp.py:587-601)
        real[3, rows, :] = False
        real[1, :, 0] = False
        real[2, :, W - 1] = False
        nxt[real] = SENT
        eng.step(1)
        torch.cuda.synchronize()
        got = eng.current
        assert torch.isfinite(got[real][:, :M]).all(), "a real slot was not written"
        assert torch.equal(torch.nan_to_num(got[~real], nan=7.0),
                           torch.nan_to_num(keep[~real], nan=7.0)), "ghost / halo slot written"
        del H
    eng.step(4)
    torch.cuda.synchronize()
    eng.raise_if_degenerate()
    for big in bigs + [bigv]:
        assert _margins_intact(big), "write outside a buffer"
    # no NaN read from a margin reached the messages, and they match the oracle
    cur = eng.current[:, 1:rows + 1, :, :M]
    assert torch.isfinite(cur).all() or dom == "max"
    iters = eng.iterations
    ref = (oracle.sync_run(model, iters, dom, kernel) if sched == SYNCHRONOUS
           else oracle.seq_run(model, iters, dom, kernel)[0])
    got = cur.reshape(4, -1, M).double().cpu().numpy()
    if dom == "sum":
        assert oracle.rel_deviation(got, ref, floor=1e-30) <= 1e-5
    else:
        fin = np.isfinite(ref)
        assert np.array_equal(np.isfinite(got), fin)
        assert np.abs(got[fin] - ref[fin]).max() <= 1e-5 * max(1.0, np.abs(ref[fin]).max())


@pytest.mark.parametrize("fam", [f for f in FAMILIES if f[0] not in ("fused",)],
                         ids=[f[0] for f in FAMILIES if f[0] not in ("fused",)])
def test_launch_geometry_does_not_change_bits(fam, env):
    """Persistent kernels walk pixel groups with a grid stride; different
    grid sizes change which warp handles which node and the interleaving.
    Any race or cross-warp dependency would show up as different bits."""
    _, name, dom, sched, variant, kernel, kind = fam
    model = _model(name, kind)
    outs = []
    for cap in (None, "1", "7"):
        v = dict(variant)
        if cap is not None:
            v["SBP_MAX_BLOCKS"] = cap
        env(v)
        store = sbp.run_sweeps(model, 5, kernel=kernel, domain=dom, schedule=sched)
        outs.append(store.engine.msgs4())
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[0], outs[2])
