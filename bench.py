#!/usr/bin/env python
"""bench.py -- Jacobian-assembly throughput of libiga on B200 (BASELINE.json metric).

One "step" = one iga_form_jacobian(a, b) call on the configured state that also forms the
residual F in the same pass (every §8(a) hot-path row: basis tables are resident, the call does
tensor product -> rational -> push-forward -> fields -> integrand -> element contraction ->
CSR / F scatter).  Pattern build and space creation are setup, outside the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl iga|reference]

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "Jacobian assembly quadrature points/sec (fp64)"
UNIT = "qpts/s"
DEFAULT_CONFIG = 5          # BASELINE.json configs[4]: the largest single-GPU config (the headline)
# Algorithmic model:
#   F_J  = min over rank / test-side sum-factorised / sum-factorised contraction flops per qpt
#   F_R  = residual rank-form flops per qpt;  B = CSR values written once + vectors, bytes per qpt
F_J = {1: 72.0, 2: 672.0, 3: 738.0, 4: 9477.0, 5: 40986.0, 7: 324.0, 8: 4428.0}
F_R = {1: 108.0, 2: 192.0, 3: 198.0, 4: 972.0, 5: 2376.0, 7: 108.0, 8: 702.0}
B_QP = {1: 25.6, 2: 25.8, 3: 24.9, 4: 348.0, 5: 596.0, 7: 25.6, 8: 37.5}
# config 7 (the Alg. 2 ring, not a BASELINE config): 2D p = 2 NURBS Laplace + mass, R' = 3, nnzD' = 9,
# symmetric: tsf = sf = 324 flop/qpt (Appendix B with n1 = q1 = 3, C_tsf = 54, C_sf = 324).
# config 8 (3D CH, §8(f) rank 3): ESTIMATE -- Appendix B's tsf with n1 = q1 = 3, C_tsf = 243,
# R' = 7 separable test kinds and nnzD' = 19 (config 3's 11 extended to d = 3; T = 1 + 3d + 2d^2)
# FP64 peak from unit counts and clock: 148 SMs x 64 DFMA/clk x 2 flop x 1.965 GHz
P64_NOMINAL_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


class ClockSampler:
    """SM clock and throttle reasons sampled with NVML (every ~1 ms) during the timed region.

    The GPU is found by PCI bus id (CUDA and NVML orderings can differ).  At least one sample is
    always taken (at exit) so that short regions still report a clock."""

    BAD = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
           "sw_power_cap": 0x4, "hw_power_brake": 0x80}

    def __init__(self, cuda_index: int):
        self.idx = cuda_index
        self.samples, self.reasons, self.mx = [], set(), None
        self._stop = threading.Event()
        self.h = None

    def _sample(self, nv):
        self.samples.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        for nm, bit in self.BAD.items():
            if r & bit:
                self.reasons.add(nm)

    def _loop(self, nv):
        while not self._stop.is_set():
            try:
                self._sample(nv)
            except Exception:
                return
            time.sleep(0.001)

    def __enter__(self):
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            self.nv = nv
            try:
                p = torch.cuda.get_device_properties(self.idx)
                bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
                self.h = nv.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = nv.nvmlDeviceGetHandleByIndex(self.idx)
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._loop, args=(nv,), daemon=True)
            self.t.start()
        except Exception:
            self.h = None
        return self

    def __exit__(self, *a):
        if self.h is not None:
            self._stop.set()
            self.t.join(timeout=2)
            try:
                self._sample(self.nv)
            except Exception:
                pass

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml"}


def box_procs(n: int, dim: int):
    """ranks per axis for n GPUs: split the largest factor 2 first over the leading axes"""
    procs = [1] * dim
    k, a = n, 0
    while k > 1:
        f = 2 if k % 2 == 0 else k
        procs[a % dim] *= f
        k //= f
        a += 1
    return procs


def owned_rows(w, sp):
    """global dof indices of the space's owned node box (node-major, dof innermost)"""
    idx = np.zeros(1, dtype=np.int64)
    for a in range(w.dim):
        g = np.arange(sp.owned_lo[a], sp.owned_hi[a], dtype=np.int64)
        idx = (idx[:, None] * w.nfun[a] + g[None, :]).reshape(-1)
    return (idx[:, None] * w.dof + np.arange(w.dof)[None, :]).reshape(-1)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------------------------------
# reference arm: the CPU oracle (as it stands) on a bounded sample of the same workload
# ------------------------------------------------------------------------------------------
def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_rows_threads(osp, w, rows, nthreads):
    """The oracle's row-subset assembly on `nthreads` host threads: the sorted rows are cut into
    contiguous chunks, each assembled by the unchanged oracle call (ctypes releases the GIL), so
    elements at chunk seams are integrated once per chunk.  Returns the element count visited."""
    import concurrent.futures as cf
    chunks = [c for c in np.array_split(rows, nthreads) if len(c)]
    with cf.ThreadPoolExecutor(max_workers=len(chunks)) as ex:
        res = list(ex.map(lambda c: osp.assemble_rows(w.phys, w.params, w.a, w.b, w.U, c, Udot=w.Udot), chunks))
    return sum(r["nvisited"] for r in res)


class OracleSlab:
    """CPU baseline: the oracle, as it stands, assembling the COMPLETE rows (all dofs,
    Jacobian + residual) of a slab of consecutive node rows of the workload -- whole node layers
    along axis 0 when they fit the time budget (config 5: the 128 x 128 node layers of the periodic
    box), else a run of consecutive rows inside one layer -- on all host cores (row chunks on
    threads).  The full assembly time is extrapolated linearly in the row count (every slab of a
    uniform periodic box costs the same; open boxes to within their boundary layers):
        value = nqp_total * (rows_in_slab / rows_total) / t_slab   [qpts/s, labelled extrapolation]
    The slab is sized from a one-pencil calibration so that one timed pass takes ~target_s."""

    def __init__(self, w, target_s: float, threads: int):
        import oracle
        self.w, self.T = w, threads
        self.osp = oracle.Space.from_workload(w)
        self.nrows = self.osp.ndof
        nf = w.nfun
        self.layer = int(np.prod(nf[1:])) * w.dof            # rows of one node layer along axis 0
        mid = (nf[0] // 2) * self.layer
        # calibration: one pencil (the last axis) of rows, all dofs, single pass on all threads
        pen = nf[-1] * w.dof
        rows = np.arange(mid, mid + pen, dtype=np.int64)
        t0 = time.perf_counter()
        oracle_rows_threads(self.osp, w, rows, threads)
        per_row = (time.perf_counter() - t0) / pen
        self.target, self.grown = target_s, False
        self._size(max(pen, int(target_s / max(per_row, 1e-12))))

    def _size(self, want):
        w, nf = self.w, self.w.nfun
        pen = nf[-1] * w.dof
        mid = (nf[0] // 2) * self.layer
        if want >= self.layer:
            nl = max(1, min(nf[0], want // self.layer))
            lo = max(0, nf[0] // 2 - nl // 2) * self.layer
            self.rows = np.arange(lo, lo + nl * self.layer, dtype=np.int64)
            self.desc = f"{nl} node layer(s) along axis 0 ({len(self.rows)} rows)"
        else:
            n = max(pen, (want // pen) * pen)
            self.rows = np.arange(mid, mid + n, dtype=np.int64)
            self.desc = f"{n // pen} pencil(s) of node rows inside one axis-0 layer ({len(self.rows)} rows)"

    def run(self):
        """One timed pass; returns (seconds, extrapolated qpts/s).  A pass much shorter than the
        target (the one-pencil calibration overestimates the per-row cost: its row chunks are tiny)
        grows the slab for the next pass."""
        t0 = time.perf_counter()
        oracle_rows_threads(self.osp, self.w, self.rows, self.T)
        dt = time.perf_counter() - t0
        rate = self.w.nqp * (len(self.rows) / self.nrows) / dt
        if dt < 0.5 * self.target and not self.grown:
            self.grown = True
            self._size(int(len(self.rows) * min(8.0, self.target / max(dt, 1e-3))))
        return dt, rate

    def sample_text(self):
        return (f"complete Jacobian + residual rows (all {self.w.dof} dofs) of {self.desc} of {self.w.name}, "
                f"C oracle on {self.T} host threads (row chunks); full-assembly rate extrapolated linearly in the "
                f"row count: nqp_total x rows_sample / rows_total / t_sample")


def run_reference(args, w, ws, rank):
    """Reference arm of this tier: the CPU oracle (as it stands) on the host cores, same workload,
    metric and unit as the product arm; each step is one bounded slab sample (OracleSlab) so that
    the whole --steps K --warmup W run ends within a few minutes.  Rank 0 alone runs it."""
    if rank != 0:
        return 0
    import oracle  # noqa: F401  (test infrastructure, allowed for the reference arm)
    budget = 150.0
    per_step = max(2.0, min(20.0, budget / max(1, args.steps + args.warmup)))
    T = host_cores()
    slab = OracleSlab(w, per_step, T)
    times, vals = [], []
    for it in range(args.warmup + args.steps):
        dt, v = slab.run()
        if it >= args.warmup:
            times.append(dt)
            vals.append(v)
    value = len(vals) / sum(1.0 / v for v in vals)          # = total qpts-equivalent / total time
    ms = 1e3 * w.nqp / value
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": w.name, "nqp": w.nqp, "l2": "host",
                      "sample_seconds_per_step": sum(times) / len(times)},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": T, "kind": "oracle", "sample": slab.sample_text()},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ------------------------------------------------------------------------------------------
# product arm
# ------------------------------------------------------------------------------------------
def run_iga(args, w, ws, rank, local):
    import torch
    import paper_1305_4452_b200 as iga

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    procs = None
    if ws > 1:
        # box decomposition of the element grid; libiga's own NCCL communicator
        # carries the ghost-U and halo-row exchanges, torch.distributed only ships its unique id
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        procs = box_procs(ws, w.dim)
        obj = [iga.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        sp = iga.Space.from_workload(w, device=local, dist={"rank": rank, "nranks": ws, "procs": procs,
                                                            "transport": iga.XPORT_NCCL, "nccl_id": obj[0]})
    else:
        sp = iga.Space.from_workload(w, device=local)
    for kv in args.opt:
        k, v = kv.split("=")
        sp.set_option(k, int(v))
    stream = torch.cuda.current_stream()
    own = owned_rows(w, sp)
    U = torch.from_numpy(w.U[own]).to(dev)
    Ud = torch.from_numpy(w.Udot[own]).to(dev)
    rp, ci = sp.csr_pattern()
    vals = torch.empty(sp.nnz, dtype=torch.float64, device=dev)
    F = torch.empty(sp.nrows, dtype=torch.float64, device=dev)
    ph = iga.make_phys(w.phys, w.params)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # 512 MiB > 126 MB L2

    def step():
        sp.form_jacobian(ph, w.a, w.b, U, Ud, vals=vals, F=F)

    experiment = any(kv.startswith("dbg=") and kv != "dbg=0" for kv in args.opt)   # phase-skip A/B: results invalid

    def check():
        if experiment:
            try:
                sp.check()
            except iga.IgaError:
                pass
        else:
            sp.check()

    for _ in range(args.warmup):
        flush.zero_()
        step()
    check()
    torch.cuda.synchronize()
    launches_per_step = sp.last_launch_count()

    def timed_region(nsteps, profile=False):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nsteps)]
        if profile:
            sp.profile(True)
            sp.profile_reset()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        for i in range(nsteps):
            flush.zero_()                       # L2 flush between timed iterations (not timed)
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        prof = sp.profile_read() if profile else None
        if profile:
            sp.profile(False)
        return [a.elapsed_time(b) for a, b in evs], prof

    with ClockSampler(local) as clk:
        ms, _ = timed_region(args.steps)
    check()
    step_ms = sum(ms) / len(ms)
    nqp_total = sp.nqp
    if ws > 1:
        t = torch.tensor([step_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        step_ms = float(t.item())
        q = torch.tensor([float(sp.nqp)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(q)
        nqp_total = int(q.item())
    value = nqp_total / (step_ms * 1e-3)

    # per-kernel device times (second pass with the kernel timing hook on)
    _, prof = timed_region(args.steps, profile=True)

    # end to end from pinned host buffers: single rank through the host-buffer C-ABI call
    # (iga_form_jacobian_host); multi-rank through the device call with the owned-vector H2D and
    # the owned values / residual D2H copies inside the timed region (max over ranks)
    Uh = torch.from_numpy(w.U[own]).pin_memory()
    Udh = torch.from_numpy(w.Udot[own]).pin_memory()
    vh = torch.empty(sp.nnz, dtype=torch.float64).pin_memory()
    fh = torch.empty(sp.nrows, dtype=torch.float64).pin_memory()
    e2e_steps = max(3, min(args.steps, 10))

    def e2e_step():
        if ws == 1:
            sp.form_jacobian_host(ph, w.a, w.b, Uh, Udh, vh, fh)
        else:
            U.copy_(Uh, non_blocking=True)
            Ud.copy_(Udh, non_blocking=True)
            step()
            vh.copy_(vals, non_blocking=True)
            fh.copy_(F, non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    e2e_ms = []
    for _ in range(e2e_steps):
        flush.zero_()
        if ws > 1:
            torch.distributed.barrier()
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_ev.record(stream)
        e2e_step()
        b_ev.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(a_ev.elapsed_time(b_ev))
    e2e_t = statistics.mean(e2e_ms)
    if ws > 1:
        t = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e_val = nqp_total / (e2e_t * 1e-3)

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return 0
    peaks = load_peaks()
    # dominant kernel and its roofline (FP64-ALU bound)
    kern = {k: v for k, v in prof.items()}
    dom = max(kern, key=lambda k: kern[k][1])
    n_l, tot_ms = kern[dom]
    avg_ms = tot_ms / n_l
    cid = w.cid
    # the assembly kernels (fused 2D / 3D, or the split contraction) carry the whole element
    # contraction: FP64-ALU bound; their algorithmic flops per launch are
    # (F_J + F_R) x the quadrature points that launch integrates
    ASSEMBLY = ("k_fused2d", "k_fused3d", "k_contract")
    if dom in ASSEMBLY:
        dom_per_step = max(1.0, kern[dom][0] / args.steps)
        nqp_launch = sp.nqp / dom_per_step
        alg = (F_J[cid] + F_R[cid]) * nqp_launch
        bound, unit, peak = "alu", "TFLOP/s", P64_NOMINAL_TFLOPS
        achieved = alg / (avg_ms * 1e-3) / 1e12
    elif dom == "k_point":
        # pointwise stage of the split path: no algorithmic flops in the model
        alg = None
        bound, unit, peak = "alu", "TFLOP/s", P64_NOMINAL_TFLOPS
        achieved = 0.0
    else:
        alg = 8.0 * sp.nnz
        bound, unit, peak = "hbm", "GB/s", peaks.get("hbm_gbs", 6650.0)
        achieved = alg / (avg_ms * 1e-3) / 1e9
    traffic, ncu_k = None, {}
    summ = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(summ):
        try:
            ncu_k = json.load(open(summ)).get(w.name, {}).get(dom, {})
            traffic = ncu_k.get("dram_bytes_per_launch")
        except Exception:
            ncu_k = {}
    # executed FP64 work of the same kernel (ncu op counters, profiles/ncu_summary.json): exposes
    # redundant work against the algorithmic model
    executed = None
    if ncu_k.get("exec_fp64_flop_per_launch") and dom in ASSEMBLY:
        ef = float(ncu_k["exec_fp64_flop_per_launch"])
        executed = {"flop_per_qpt": ef / nqp_launch, "model_flop_per_qpt": F_J[cid] + F_R[cid],
                    "executed_over_model": ef / alg, "tflops_at_bench_time": ef / (avg_ms * 1e-3) / 1e12,
                    "fp64_pipe_pct_ncu": ncu_k.get("fp64_pipe_pct"), "source": ncu_k.get("source")}
    t_roof = max((F_J[cid] + F_R[cid]) * sp.nqp / (P64_NOMINAL_TFLOPS * 1e12),
                 B_QP[cid] * sp.nqp / (peaks.get("hbm_gbs", 6650.0) * 1e9))
    clocks = clk.summary()

    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        import oracle  # noqa: F401  (bench's cpu_baseline leg may execute the oracle)
        T = host_cores()
        slab = OracleSlab(w, 15.0, T)
        slab.run()                              # sizes the slab (grows it if the calibration overshot)
        dt, vT = slab.run()
        cpu = {"value": vT, "unit": UNIT, "cores": T, "kind": "oracle", "sample": slab.sample_text(),
               "sample_seconds": dt}

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "nqp": sp.nqp, "nelem": w.nelem, "ndof": sp.ndof, "nnz": sp.nnz,
                   "degree": w.degree[0], "dof_per_node": w.dof, "l2": "flushed (512 MiB write) between steps",
                   "step": "iga_form_jacobian(a,b) with residual F fused",
                   "parallelism": f"box {'x'.join(map(str, procs))} over {ws} GPUs (NCCL ghost/halo exchange)"
                   if ws > 1 else "1 GPU"},
        "roofline": {"bound": bound, "kernel": dom, "achieved": achieved, "peak": peak, "unit": unit,
                     "frac": achieved / peak if peak else None, "traffic": traffic,
                     "peak_source": "148 SM x 64 DFMA/clk x 2 x 1.965 GHz (B200 unit counts, DESIGN.md)"
                     if unit == "TFLOP/s" else "MEASURED_PEAKS.json hbm_gbs",
                     "kernel_ms": {k: v[1] / v[0] for k, v in kern.items()},
                     "kernel_launches_per_step": {k: v[0] / args.steps for k, v in kern.items()},
                     "step_roofline_ms": t_roof * 1e3, "step_frac": t_roof * 1e3 / step_ms,
                     "executed": executed},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(2 * 8 * sp.nrows * ws),
                "d2h_bytes_per_step": int(8 * (sp.nnz + sp.nrows) * ws), "ms_per_step": e2e_t},
        "gpu_launches": int(sum(v[0] for v in kern.values())) if kern else int(launches_per_step * args.steps),
        "clocks": clocks,
    }
    print(json.dumps(out), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def run_basis3(args, w, local):
    """Secondary measurement: iga_basis_eval, all spatial derivatives up to
    third order of every local basis function at every Gauss point.  HBM-write-bound: the
    algorithmic bytes are the output tensor (8 B x nen x ncomp x nqp)."""
    import torch
    import paper_1305_4452_b200 as iga
    torch.cuda.set_device(local)
    sp = iga.Space.from_workload(w, device=local)
    out = sp.basis_eval(3)
    sp.check()
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=out.device)
    for _ in range(args.warmup):
        sp.basis_eval(3, out=out)
    ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            sp.basis_eval(3, out=out)
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
    sp.check()
    t = statistics.mean(ms)
    nbytes = out.numel() * 8
    peaks = load_peaks()
    bw = peaks.get("hbm_gbs", 6650.0)
    achieved = nbytes / (t * 1e-3) / 1e9
    print(json.dumps({
        "metric": "third-order basis evaluation quadrature points/sec (fp64)", "value": sp.nqp / (t * 1e-3),
        "unit": "qpts/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t,
        "higher_is_better": True, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "op": "iga_basis_eval(order=3)", "out_shape": list(out.shape),
                   "l2": "flushed (512 MiB write) between steps"},
        "roofline": {"bound": "hbm", "kernel": "k_basis3", "achieved": achieved, "peak": bw, "unit": "GB/s",
                     "frac": achieved / bw, "traffic": None, "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
        "clocks": clk.summary()}), flush=True)
    return 0


def run_residual(args, w, local):
    """Secondary measurement: the residual call alone, iga_form_residual."""
    import torch
    import paper_1305_4452_b200 as iga
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sp = iga.Space.from_workload(w, device=local)
    U, Ud = torch.from_numpy(w.U).to(dev), torch.from_numpy(w.Udot).to(dev)
    F = torch.empty(sp.nrows, dtype=torch.float64, device=dev)
    ph = iga.make_phys(w.phys, w.params)
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        sp.form_residual(ph, U, Ud, F=F)
    sp.check()
    ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            sp.form_residual(ph, U, Ud, F=F)
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
    sp.check()
    t = statistics.mean(ms)
    cid = w.cid
    t_roof = max(F_R[cid] * sp.nqp / (P64_NOMINAL_TFLOPS * 1e12),
                 (3 * 8.0 * sp.nrows) / (load_peaks().get("hbm_gbs", 6650.0) * 1e9))
    print(json.dumps({
        "metric": "Residual assembly quadrature points/sec (fp64)", "value": sp.nqp / (t * 1e-3), "unit": "qpts/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t, "higher_is_better": True,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "op": "iga_form_residual", "l2": "flushed (512 MiB write) between steps"},
        "roofline": {"bound": "alu", "achieved": F_R[cid] * sp.nqp / (t * 1e-3) / 1e12, "peak": P64_NOMINAL_TFLOPS,
                     "unit": "TFLOP/s", "frac": t_roof / (t * 1e-3), "model": "F_R rank-form flops/qpt (SURVEY §8(d))"},
        "clocks": clk.summary()}), flush=True)
    return 0


def run_protocol(args, w, ws, rank, local):
    """Secondary measurement: the paper's §5 fixed-budget protocol
     -- generalized-alpha steps (rho_inf = 0.5, the workloads' (a, b)), each 2 Newton
    iterations of {Jacobian + residual assembly, 30 GMRES iterations with block-Jacobi ILU(0)}:
    iga_alpha_step.  A step = one time step.  The GMRES iteration is HBM-bound; its algorithmic
    bytes (SpMV nnz*12 + 4n*8, one Gram-Schmidt pass (2j+5) n*8 averaged over j < 30,
    preconditioner vectors 3n*8) give the roofline line."""
    import torch
    import paper_1305_4452_b200 as iga
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        # one process per GPU over the box decomposition: distributed assembly (libiga's NCCL
        # communicator) and distributed GMRES; torch.distributed ships the NCCL id and the max-time
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        obj = [iga.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        sp = iga.Space.from_workload(w, device=local, dist={"rank": rank, "nranks": ws, "procs": box_procs(ws, w.dim),
                                                            "transport": iga.XPORT_NCCL, "nccl_id": obj[0]})
    else:
        sp = iga.Space.from_workload(w, device=local)
    rp, ci = sp.csr_pattern()
    val = torch.empty(ci.numel(), dtype=torch.float64, device=dev)
    ph = iga.make_phys(w.phys, w.params)
    rho, dt = 0.5, w.b * 9.0 / 4.0          # (a, b) = (5/6, 4/9 dt) <=> rho_inf = 0.5
    own = owned_rows(w, sp)
    U, Ud = torch.from_numpy(w.U[own]).to(dev), torch.from_numpy(w.Udot[own]).to(dev)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        sp.alpha_step(ph, U, Ud, rp, ci, val, rho, dt)
    sp.check()
    ms, stats = [], None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            stats = sp.alpha_step(ph, U, Ud, rp, ci, val, rho, dt)
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
    launches = sp.last_launch_count()
    sp.check()
    if ws > 1:
        import torch.distributed as dist
        tm = torch.tensor(ms, dtype=torch.float64, device=dev)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)          # device-timed, max over ranks
        ms = tm.cpu().tolist()
    # breakdown: one Jacobian + residual assembly, one 30-iteration solve (same buffers)
    F = torch.empty(sp.nrows, dtype=torch.float64, device=dev)
    x = torch.zeros_like(F)

    def timed(fn, reps=3):
        out = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            out.append(a.elapsed_time(b))
        return statistics.median(out)
    t_asm = timed(lambda: sp.form_jacobian(ph, w.a, w.b, U, Ud, vals=val, F=F, want_F=True))
    t_g0 = timed(lambda: sp.gmres(rp, ci, val, F, x=x.zero_(), maxit=0, rtol=0.0))
    t_g1 = timed(lambda: sp.gmres(rp, ci, val, F, x=x.zero_(), maxit=1, rtol=0.0))
    t_g30 = timed(lambda: sp.gmres(rp, ci, val, F, x=x.zero_(), maxit=30, rtol=0.0))
    t_it = (t_g30 - t_g1) / 29.0
    n, nnz = sp.nrows, ci.numel()
    bytes_it = nnz * 12 + 4 * n * 8 + (2 * 14.5 + 5) * n * 8 + 3 * n * 8
    bw = load_peaks().get("hbm_gbs", 6650.0)
    achieved = bytes_it / (t_it * 1e-3) / 1e9
    t = statistics.mean(ms)
    if rank != 0:
        return 0
    print(json.dumps({
        "metric": "generalized-alpha time steps/sec (2 Newton x (assembly + 30 GMRES), fp64)", "value": 1e3 / t,
        "unit": "steps/s", "n_gpus": ws, "scaling": "weak", "steps": args.steps, "warmup": args.warmup, "ms_per_step": t,
        "higher_is_better": True, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "op": "iga_alpha_step", "rho_inf": rho, "dt": dt, "newton_its": 2,
                   "gmres": "GMRES(30), 30 iterations, block-Jacobi ILU(0), 32-row blocks",
                   "l2": "inputs larger than L2 (matrix)"},
        "breakdown_ms": {"assembly_jacobian_and_residual": t_asm, "gmres_setup_and_residual": t_g0,
                         "gmres_per_iteration": t_it, "gmres_30_iterations": t_g30},
        "newton": stats,
        "roofline": {"bound": "hbm", "kernel": "GMRES iteration (k_spmv_sw + k_ell_solve + Gram-Schmidt)",
                     "achieved": achieved, "peak": bw, "unit": "GB/s", "frac": achieved / bw, "traffic": None,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
        "gpu_launches": int(launches * args.steps),
        "clocks": clk.summary()}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--op", default="jacobian", choices=["jacobian", "residual", "basis3", "protocol"],
                    help="jacobian: the headline assembly step; residual: the residual call alone; "
                         "basis3: third-order basis evaluation; protocol: the paper's generalized-alpha "
                         "step with 2 Newton x 30 GMRES")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--n", type=int, default=None, help="elements per axis (default: BASELINE size)")
    ap.add_argument("--impl", default="iga", choices=["iga", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--opt", action="append", default=[], help="libiga option key=value (experiments)")
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="--gpus N > 1: strong = the named mesh is split N ways (default for the 3D configs, "
                         "incl. the headline config 5: the north star's 8-GPU target is config-5 strong "
                         "scaling); weak = every GPU keeps the named config's element count (default for 2D)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup) if args.impl == "iga" else args.warmup
    if args.scaling is None:
        args.scaling = "strong" if args.config in (4, 5, 8) else "weak"
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torch.distributed.run (127.0.0.1)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    ws, rank, local = dist_env()
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; launch with torch.distributed.run "
              f"--nproc-per-node {args.gpus} (or without WORLD_SIZE to let bench.py launch the ranks)",
              file=sys.stderr)
        return 2
    if args.impl == "iga":
        import torch
        if torch.cuda.device_count() < ws:
            print(f"bench.py: {ws} ranks but only {torch.cuda.device_count()} CUDA device(s) visible", file=sys.stderr)
            return 2
    n = args.n
    if ws > 1 and args.scaling == "weak":
        dim = workloads.make(args.config, n=6).dim
        base = n if n is not None else workloads.FULL_N[args.config]
        n = [base * f for f in box_procs(ws, dim)]
    w = workloads.make(args.config, n=n)
    if args.impl == "reference":
        return run_reference(args, w, ws, rank)
    if args.op == "basis3":
        return run_basis3(args, w, local)
    if args.op == "residual":
        return run_residual(args, w, local)
    if args.op == "protocol":
        return run_protocol(args, w, ws, rank, local)
    return run_iga(args, w, ws, rank, local)


if __name__ == "__main__":
    sys.exit(main())
