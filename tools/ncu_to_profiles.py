"""Summarise ncu reports from gpurun_out/ into profiles/: per-report text summary and the
profiles/ncu_summary.json that bench.py reads for roofline.traffic (dram bytes per launch).
usage: python tools/ncu_to_profiles.py TAG"""
import csv, glob, json, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
sys.path.insert(0, ROOT)
import workloads  # noqa: E402

summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
for rep in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "**", f"{tag}_c*_k_*.ncu-rep"), recursive=True)):
    m = re.search(r"_c(\d)_(k_\w+)\.ncu-rep", rep)
    cid, kern = int(m.group(1)), m.group(2)
    name = workloads.make(cid, n=4).name.rsplit("_", 1)[0]
    wname = workloads.make(cid).name
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                         capture_output=True, text=True).stdout
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_c{cid}_{kern}.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none, one launch of {kern}, bench.py --config {cid} ({wname})\n")
        f.write(out)
    vals = {}
    for ln in out.splitlines():
        p = ln.split()
        if len(p) >= 2:
            vals[p[0]] = (p[1], p[2] if len(p) > 2 else "")
    def tobytes(v):
        x, u = float(v[0]), v[1].lower()
        return x * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
    def toms(v):
        x, u = float(v[0]), v[1].lower()
        return x * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1, "s": 1e3, "second": 1e3}.get(u, 1)
    rd, wr = tobytes(vals["dram__bytes_read.sum"]), tobytes(vals["dram__bytes_write.sum"])

    def cnt(k):
        try:
            return float(vals[k][0])
        except (KeyError, ValueError):
            return float("nan")
    # executed FP64 flops of the launch: 2 x DFMA + DADD + DMUL thread-instructions
    # (ncu reports them as rates per elapsed cycle summed over SMSPs; x the elapsed SMSP cycles)
    pc = "smsp__sass_thread_inst_executed_op_{}_pred_on.sum.per_cycle_elapsed"
    exec_flop = (2 * cnt(pc.format("dfma")) + cnt(pc.format("dadd")) + cnt(pc.format("dmul"))) * \
        cnt("smsp__cycles_elapsed.avg")
    summ.setdefault(wname, {})[kern] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                                        "ncu_ms": toms(vals["gpu__time_duration.sum"]),
                                        "fp64_pipe_pct": float(vals.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", ("nan",))[0]),
                                        "exec_fp64_flop_per_launch": exec_flop,
                                        "source": os.path.basename(rep), "tag": tag}
json.dump(summ, open(summ_path, "w"), indent=1)
print(json.dumps(summ, indent=1))
