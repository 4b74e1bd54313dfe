"""Helpers shared by the GPU parity tests (comparison rules of the north star / DESIGN.md)."""
import numpy as np

# north_star: values within 1e-11 relative to the row's max |entry| (fp64, differing order)
ROW_TOL = 1e-11


def rowmax_rel_err(rowptr, ref_vals, got_vals):
    """max over rows of max|got-ref| / max|ref| (rows whose ref is all-zero use an absolute 1e-300 floor)."""
    rp = np.asarray(rowptr)
    ref = np.asarray(ref_vals)
    got = np.asarray(got_vals)
    diff = np.abs(got - ref)
    worst = 0.0
    nrows = len(rp) - 1
    # vectorised per-row maxima
    lens = np.diff(rp)
    if len(ref) == 0:
        return 0.0
    row_id = np.repeat(np.arange(nrows), lens)
    rmax = np.zeros(nrows)
    np.maximum.at(rmax, row_id, np.abs(ref))
    dmax = np.zeros(nrows)
    np.maximum.at(dmax, row_id, diff)
    rel = dmax / np.maximum(rmax, 1e-300)
    worst = float(rel.max()) if nrows else 0.0
    return worst


def vec_rel_err(ref, got):
    ref = np.asarray(ref)
    got = np.asarray(got)
    scale = max(np.abs(ref).max(), 1e-300)
    return float(np.abs(got - ref).max() / scale)


def gather_rows(rowptr, cols, vals, rows):
    """Extract CSR rows `rows` -> (rowptr_sub, cols_sub, vals_sub)."""
    rp = np.asarray(rowptr)
    starts = rp[rows]
    ends = rp[np.asarray(rows) + 1]
    lens = ends - starts
    idx = np.concatenate([np.arange(s, e) for s, e in zip(starts, ends)]) if len(rows) else np.zeros(0, np.int64)
    sub_rp = np.zeros(len(rows) + 1, np.int64)
    sub_rp[1:] = np.cumsum(lens)
    return sub_rp, np.asarray(cols)[idx], (None if vals is None else np.asarray(vals)[idx])


def oracle_rows_parallel(osp, w, rows, threads=None, **kw):
    """The oracle's row-subset assembly (complete rows) on host threads: the sorted rows are cut
    into contiguous chunks, each assembled by the unchanged oracle call (ctypes releases the GIL),
    and the per-chunk CSR pieces are concatenated."""
    import concurrent.futures as cf
    import os
    T = threads or max(1, len(os.sched_getaffinity(0)))
    chunks = [c for c in np.array_split(np.asarray(rows, np.int64), T) if len(c)]
    with cf.ThreadPoolExecutor(max_workers=len(chunks)) as ex:
        parts = list(ex.map(lambda c: osp.assemble_rows(w.phys, w.params, w.a, w.b, w.U, c, Udot=w.Udot, **kw),
                            chunks))
    rp = [np.zeros(1, np.int64)]
    off = 0
    for p in parts:
        rp.append(p["rowptr"][1:] + off)
        off += p["rowptr"][-1]
    return dict(rowptr=np.concatenate(rp), cols=np.concatenate([p["cols"] for p in parts]),
                vals=np.concatenate([p["vals"] for p in parts]), F=np.concatenate([p["F"] for p in parts]),
                touched=np.concatenate([p["touched"] for p in parts]),
                nvisited=sum(p["nvisited"] for p in parts))
