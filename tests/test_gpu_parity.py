"""GPU parity: libiga (CUDA, sm_100a) vs the CPU oracle, through the C ABI.

Pattern: bit-exact.  Values: within 1e-11 of the row's max |entry| (north_star), plus the
per-term-group runs of reading A-17 so that small terms are checked on their own scale.
"""
import numpy as np
import pytest

import oracle
import workloads
from parity_util import ROW_TOL, gather_rows, oracle_rows_parallel, rowmax_rel_err, vec_rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1305_4452_b200 as iga
    return iga


def _gpu_assemble(iga, w, a=None, b=None, params=None, Udot=None, want_F=True, split=False):
    sp = iga.Space.from_workload(w)
    if split == "general":
        sp.set_option("general", 1)          # fused kernels without the uniform-table fast path
    elif split:
        sp.set_option("split", 1)
    dev = torch.device("cuda", 0)
    U = torch.from_numpy(w.U).to(dev)
    Ud = torch.from_numpy(Udot if Udot is not None else w.Udot).to(dev)
    rp, ci = sp.csr_pattern()
    ph = iga.make_phys(w.phys, params if params is not None else w.params)
    vals, F = sp.form_jacobian(ph, w.a if a is None else a, w.b if b is None else b, U, Ud, want_F=want_F)
    Fr = sp.form_residual(ph, U, Ud)
    sp.check()
    torch.cuda.synchronize()
    return sp, rp.cpu().numpy(), ci.cpu().numpy(), vals.cpu().numpy(), (F.cpu().numpy() if F is not None else None), \
        Fr.cpu().numpy()


SMALL = [(1, 16), (1, 5), (2, 3), (2, 16), (3, 5), (3, 12), (4, 2), (4, 5), (5, 5), (5, 7), (6, 5), (6, 9),
         (7, 5), (7, 9), (7, 20), (8, 5), (8, 6)]


SMALL_2D_TILES = [(1, 17), (2, 9), (2, 21), (3, 16), (3, 33), (3, 40)]   # several tiles + ragged tails


@pytest.mark.parametrize("split", [False, True, "general"])
@pytest.mark.parametrize("cid,n", SMALL + SMALL_2D_TILES)
def test_small_full_parity(cid, n, split):
    """Whole matrix vs dense-then-CSR oracle on small meshes (several elements / tiles, ragged
    sizes), through both the fused kernels and the generic split path."""
    iga = _gpu()
    w = workloads.make(cid, n=n)
    rng = np.random.default_rng(100 + cid)
    Ud = rng.uniform(-0.1, 0.1, w.U.size) if w.phys in (1, 3, 4) else w.Udot
    sp, rp, ci, vals, F, Fr = _gpu_assemble(iga, w, Udot=Ud, split=split)
    osp = oracle.Space.from_workload(w)
    K, T, Fo = osp.assemble_dense(w.phys, w.params, w.a, w.b, w.U, Ud)
    orp, oci, ovals = oracle.dense_to_csr(K, T)
    assert np.array_equal(rp, orp), "row_ptr differs"
    assert np.array_equal(ci, oci), "col_idx differs"
    assert rowmax_rel_err(orp, ovals, vals) <= ROW_TOL
    assert vec_rel_err(Fo, F) <= ROW_TOL
    assert vec_rel_err(Fo, Fr) <= ROW_TOL


@pytest.mark.parametrize("cid,n,groups", [
    (2, 8, [dict(params=[1.0, 0.0, 0.0]), dict(params=[0.0, 1.0, 0.0])]),            # kappa | sigma
    (3, 9, [dict(a=1.0, b=0.0), dict(a=0.0, b=1.0)]),                               # mass | d/dc
    (5, 5, [dict(a=1.0, b=0.0), dict(a=0.0, b=1.0)]),                               # d/dUdot | d/dU
    (1, 6, [dict(params=[1.0, 0.0, 1.0]), dict(params=[0.0, 1.0, 1.0])]),
    # NSK: d/dUdot | d/dU, and a capillarity-dominated state (Korteweg terms on their own scale)
    (6, 6, [dict(a=1.0, b=0.0), dict(a=0.0, b=1.0),
            dict(params=[3.0, 1.0, 8.0 / 27.0, 0.85, 0.0, 0.0, 1e-2]),
            dict(params=[0.0, 1.0, 0.0, 0.85, 1.0 / 512, -2.0 / 3.0 / 512, 0.0])]),
])
def test_term_groups(cid, n, groups):
    """A-17: the 1e-11 row-max rule hides small terms; check each term group on its own scale."""
    iga = _gpu()
    w = workloads.make(cid, n=n)
    rng = np.random.default_rng(7)
    Ud = rng.uniform(-0.1, 0.1, w.U.size) if w.phys in (1, 3, 4) else w.Udot
    osp = oracle.Space.from_workload(w)
    for g in groups:
        a, b, prm = g.get("a", w.a), g.get("b", w.b), g.get("params", w.params)
        sp, rp, ci, vals, F, Fr = _gpu_assemble(iga, w, a=a, b=b, params=prm, Udot=Ud)
        K, T, Fo = osp.assemble_dense(w.phys, prm, a, b, w.U, Ud)
        orp, oci, ovals = oracle.dense_to_csr(K, T)
        assert np.array_equal(ci, oci)
        assert rowmax_rel_err(orp, ovals, vals) <= ROW_TOL, g
        assert vec_rel_err(Fo, F) <= ROW_TOL


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5, 6, 7, 8])
def test_full_size_probe_rows(cid):
    """BASELINE full sizes, the launch bench.py times: complete probe rows vs the oracle's
    row-subset assembly (SURVEY O-10), pattern of those rows bit-exact, row lengths of ALL rows.
    (Rows are gathered on the device: config 5's CSR is 50 GB.)"""
    iga = _gpu()
    w = workloads.make(cid)
    sp = iga.Space.from_workload(w)
    dev = torch.device("cuda", 0)
    U = torch.from_numpy(w.U).to(dev)
    Ud = torch.from_numpy(w.Udot).to(dev)
    rp_d, ci_d = sp.csr_pattern()
    ph = iga.make_phys(w.phys, w.params)
    vals_d, F_d = sp.form_jacobian(ph, w.a, w.b, U, Ud, want_F=True)
    Fr_d = sp.form_residual(ph, U, Ud)
    sp.check()
    rp = rp_d.cpu().numpy()
    osp = oracle.Space.from_workload(w)
    assert sp.ndof == osp.ndof and sp.nrows == osp.ndof
    # SURVEY O-10: 3^d structured 5^d probe blocks (seam / partition plane / interior per axis) and
    # 64 seeded random ones, complete rows, the oracle on the host cores
    rows = workloads.probe_rows_o10(w)
    ref = oracle_rows_parallel(osp, w, rows)
    idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows])
    idx_d = torch.from_numpy(idx).to(dev)
    sci = ci_d[idx_d].cpu().numpy()
    svals = vals_d[idx_d].cpu().numpy()
    srp = np.zeros(len(rows) + 1, np.int64)
    srp[1:] = np.cumsum(rp[rows + 1] - rp[rows])
    assert np.array_equal(srp, ref["rowptr"])
    assert np.array_equal(sci, ref["cols"])
    assert ref["touched"].all()
    assert rowmax_rel_err(ref["rowptr"], ref["vals"], svals) <= ROW_TOL
    F = F_d.cpu().numpy()
    Fr = Fr_d.cpu().numpy()
    assert vec_rel_err(ref["F"], F[rows]) <= ROW_TOL
    assert vec_rel_err(ref["F"], Fr[rows]) <= ROW_TOL
    # every row length (closed-form row_ptr) against the oracle's Alg. 3 count
    all_rows = np.arange(sp.nrows, dtype=np.int64)
    rl = np.zeros(len(all_rows), np.int64)
    import ctypes as C
    oracle.lib().orc_pattern_rows(osp.h, len(all_rows), all_rows.ctypes.data_as(C.POINTER(C.c_int64)),
                                  rl.ctypes.data_as(C.POINTER(C.c_int64)), None)
    assert np.array_equal(np.diff(rp), rl)
    assert bool(torch.isfinite(vals_d).all())


@pytest.mark.parametrize("cid", [4, 5, 6, 8])
def test_full_size_full_pattern_streamed(cid):
    """O-10 "the pattern check is always full, streamed row by row": every row of the BASELINE-size
    CSR (config 5: 4.19e9 column indices, 16.8 GB on the device) against the oracle's Alg. 3
    pattern, in row chunks."""
    iga = _gpu()
    w = workloads.make(cid)
    sp = iga.Space.from_workload(w)
    rp_d, ci_d = sp.csr_pattern()
    osp = oracle.Space.from_workload(w)
    rp = rp_d.cpu().numpy()
    assert rp[0] == 0 and rp[-1] == sp.nnz == ci_d.numel()
    chunk = max(1, (1 << 26) // max(1, int(np.diff(rp[:2])[0])))
    for r0 in range(0, sp.nrows, chunk):
        r1 = min(sp.nrows, r0 + chunk)
        orp, oci = osp.pattern_rows(np.arange(r0, r1, dtype=np.int64))
        assert np.array_equal(rp[r0:r1 + 1] - rp[r0], orp), f"row_ptr differs in rows [{r0}, {r1})"
        got = ci_d[int(rp[r0]):int(rp[r1])].cpu().numpy()
        assert np.array_equal(got, oci), f"col_idx differs in rows [{r0}, {r1})"


@pytest.mark.parametrize("cid", [1, 2, 3, 7])
def test_full_size_full_pattern(cid):
    iga = _gpu()
    w = workloads.make(cid)
    sp = iga.Space.from_workload(w)
    rp, ci = sp.csr_pattern()
    osp = oracle.Space.from_workload(w)
    orp, oci = osp.pattern()
    assert np.array_equal(rp.cpu().numpy(), orp)
    assert np.array_equal(ci.cpu().numpy(), oci)


def test_host_variant_matches_device():
    iga = _gpu()
    w = workloads.make(3, n=16)
    sp = iga.Space.from_workload(w)
    dev = torch.device("cuda", 0)
    ph = iga.make_phys(w.phys, w.params)
    vals, F = sp.form_jacobian(ph, w.a, w.b, torch.from_numpy(w.U).to(dev), torch.from_numpy(w.Udot).to(dev),
                               want_F=True)
    vh = torch.empty(sp.nnz, dtype=torch.float64).pin_memory()
    fh = torch.empty(sp.nrows, dtype=torch.float64).pin_memory()
    Uh = torch.from_numpy(w.U).pin_memory()
    Udh = torch.from_numpy(w.Udot).pin_memory()
    sp.form_jacobian_host(ph, w.a, w.b, Uh, Udh, vh, fh)
    osp = oracle.Space.from_workload(w)
    K, T, Fo = osp.assemble_dense(w.phys, w.params, w.a, w.b, w.U, w.Udot)
    orp, _, ovals = oracle.dense_to_csr(K, T)
    assert rowmax_rel_err(orp, ovals, vh.numpy()) <= ROW_TOL
    assert rowmax_rel_err(orp, ovals, vals.cpu().numpy()) <= ROW_TOL
    assert vec_rel_err(Fo, fh.numpy()) <= ROW_TOL


@pytest.mark.parametrize("cid,n,slabs", [(5, 7, 3), (4, 6, 3), (8, 8, 4), (5, 8, 2)])
def test_host_variant_pipelined_3d(cid, n, slabs):
    """iga_form_jacobian_host on 3D spaces assembles in slabs along axis 0 and copies each node
    layer's rows back as soon as its last element is done (periodic configs 5, 8: the first p
    layers go last; open config 4: layers in order).  The values must equal the oracle's."""
    iga = _gpu()
    w = workloads.make(cid, n=n)
    sp = iga.Space.from_workload(w)
    sp.set_option("hb_slabs", slabs)
    ph = iga.make_phys(w.phys, w.params)
    vh = torch.full((sp.nnz,), float("nan"), dtype=torch.float64).pin_memory()
    fh = torch.full((sp.nrows,), float("nan"), dtype=torch.float64).pin_memory()
    Uh = torch.from_numpy(w.U).pin_memory()
    Udh = torch.from_numpy(w.Udot).pin_memory()
    sp.form_jacobian_host(ph, w.a, w.b, Uh, Udh, vh, fh)
    osp = oracle.Space.from_workload(w)
    K, T, Fo = osp.assemble_dense(w.phys, w.params, w.a, w.b, w.U, w.Udot)
    orp, _, ovals = oracle.dense_to_csr(K, T)
    assert not torch.isnan(vh).any(), "rows never copied back"
    assert rowmax_rel_err(orp, ovals, vh.numpy()) <= ROW_TOL
    assert vec_rel_err(Fo, fh.numpy()) <= ROW_TOL


def test_singular_map_flag():
    """A-7: an inverted geometry (detJ < 0) is reported as IGA_ERR_SINGULAR_MAP."""
    iga = _gpu()
    w = workloads.make(1, n=4)
    w.ctrl = w.ctrl[:, :, ::-1].copy()          # swap x <-> y: orientation reversed, detJ = -1
    sp = iga.Space.from_workload(w)
    U = torch.zeros(sp.ndof, dtype=torch.float64, device="cuda")
    sp.form_jacobian(iga.make_phys(w.phys, w.params), 0.0, 1.0, U)
    with pytest.raises(iga.IgaError) as ei:
        sp.check()
    assert ei.value.code == 3


def test_nonfinite_flag():
    """c = 0 makes mu' infinite in Cahn-Hilliard: IGA_ERR_NONFINITE."""
    iga = _gpu()
    w = workloads.make(3, n=6)
    sp = iga.Space.from_workload(w)
    U = torch.zeros(sp.ndof, dtype=torch.float64, device="cuda")
    sp.form_residual(iga.make_phys(w.phys, w.params), U)
    with pytest.raises(iga.IgaError) as ei:
        sp.check()
    assert ei.value.code == 5


def test_bad_arguments_rejected():
    iga = _gpu()
    w = workloads.make(3, n=6)
    with pytest.raises(iga.IgaError):       # periodic with too few elements (< 2p+1 functions)
        iga.Space.from_workload(workloads.make(3, n=4))
    bad = workloads.make(1, n=4)
    bad.knots[0] = bad.knots[0][::-1].copy()   # decreasing knots
    with pytest.raises(iga.IgaError) as ei:
        iga.Space.from_workload(bad)
    assert ei.value.code == 2
    ring = workloads.make(7, n=6)
    ring.ctrl = ring.ctrl.copy()
    ring.ctrl[:, 0, 1] += 0.01                 # clamped net no longer C^1 periodic (Alg. 2 check)
    with pytest.raises(iga.IgaError) as ei:
        iga.Space.from_workload(ring)
    assert ei.value.code == 2
    sp = iga.Space.from_workload(w)
    U = torch.zeros(sp.ndof, dtype=torch.float64, device="cuda")
    with pytest.raises(iga.IgaError):       # NEOHOOKE needs dof 3 / dim 3
        sp.form_residual(iga.make_phys(2, [1.0, 1.0]), U)


@pytest.mark.parametrize("cid,n", [(3, 40), (5, 9), (8, 12), (4, 8)])
def test_rerun_spread_bounded(cid, n):
    """The CSR values are summed with fp64 red.add in arrival order (reading A-18), so
    reruns may differ in the last bits.  Bound that spread: five reruns of the same call agree
    within 1e-14 of each row's max |entry| (1000x inside the 1e-11 parity bar), and the pattern
    and residual are unchanged."""
    iga = _gpu()
    w = workloads.make(cid, n=n)
    sp = iga.Space.from_workload(w)
    dev = torch.device("cuda", 0)
    U = torch.from_numpy(w.U).to(dev)
    Ud = torch.from_numpy(w.Udot).to(dev)
    rp, _ = sp.csr_pattern()
    ph = iga.make_phys(w.phys, w.params)
    runs = []
    for _ in range(5):
        vals, F = sp.form_jacobian(ph, w.a, w.b, U, Ud, want_F=True)
        runs.append((vals.clone(), F.clone()))
    sp.check()
    rpn = rp.cpu().numpy()
    v0 = runs[0][0].cpu().numpy()
    for vals, F in runs[1:]:
        assert rowmax_rel_err(rpn, v0, vals.cpu().numpy()) <= 1e-14
        assert vec_rel_err(runs[0][1].cpu().numpy(), F.cpu().numpy()) <= 1e-14


@pytest.mark.parametrize("cid,n,offset", [(5, 7, 1), (5, 7, 2), (8, 6, 1)])
def test_unaligned_values_buffer(cid, n, offset):
    """The caller's CSR value buffer may start at any 8-byte boundary (iga.h: plain double
    pointer): a view `offset` doubles into a larger allocation gives the same values as the
    oracle, and nothing outside the view is written (the scatter's red.add needs only 8-byte
    alignment; a 16-byte bulk-reduction scatter was tried and would need a fallback here)."""
    iga = _gpu()
    w = workloads.make(cid, n=n)
    sp = iga.Space.from_workload(w)
    dev = torch.device("cuda", 0)
    ph = iga.make_phys(w.phys, w.params)
    big = torch.full((sp.nnz + 4,), float("nan"), dtype=torch.float64, device=dev)
    view = big[offset:offset + sp.nnz]
    assert view.data_ptr() % 16 == (8 if offset % 2 else 0)
    sp.form_jacobian(ph, w.a, w.b, torch.from_numpy(w.U).to(dev), torch.from_numpy(w.Udot).to(dev), vals=view)
    sp.check()
    torch.cuda.synchronize()
    osp = oracle.Space.from_workload(w)
    K, T, _ = osp.assemble_dense(w.phys, w.params, w.a, w.b, w.U, w.Udot)
    orp, _, ovals = oracle.dense_to_csr(K, T)
    assert rowmax_rel_err(orp, ovals, view.cpu().numpy()) <= ROW_TOL
    assert torch.isnan(big[:offset]).all() and torch.isnan(big[offset + sp.nnz:]).all()   # nothing outside
