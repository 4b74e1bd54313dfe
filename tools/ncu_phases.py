"""Stall samples / executed warp-instructions of k_fused3d per phase, from an ncu source page
(--print-source cuda,sass).  SASS rows are attributed to the CUDA line printed above them; rows
of inlined helpers (static_for, physics, atomics) are attributed to the enclosing phase by
address order.  usage: python tools/ncu_phases.py x.csv 'name:lo-hi,...'"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "Line No")
iS, iI = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
phases = [(p.split(":")[0], *map(int, p.split(":")[1].split("-"))) for p in sys.argv[2].split(",")]
sass = []   # (address, line, samples, instrs)
line = None
for r in rows:
    if not r:
        continue
    if r[0].isdigit():
        line = int(r[0])
    elif r[0] == "" and len(r) > 5 and r[2].startswith("0x"):
        try:
            sass.append((int(r[2], 16), line, float(r[4]), float(r[7])))
        except ValueError:
            pass
sass.sort()
out, cur = {}, "other"
for addr, ln, s, n in sass:
    for name, lo, hi in phases:
        if lo <= ln <= hi:
            cur = name
            break
    o = out.setdefault(cur, [0.0, 0.0, 0])
    o[0] += s; o[1] += n; o[2] += 1
ts = sum(v[0] for v in out.values()); tn = sum(v[1] for v in out.values())
for k, (s, n, c) in sorted(out.items(), key=lambda x: -x[1][0]):
    print(f"{k:10s} samples {100*s/ts:5.1f}%  instr {100*n/tn:5.1f}%  sass {c}")
