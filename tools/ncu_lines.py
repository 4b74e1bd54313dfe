"""Aggregate an ncu source page (--print-source cuda,sass --csv) by CUDA source line.
usage: ncu -i REP --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "Line No")
iS, iI = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_")]
lines = []
for r in rows:
    if r and r[0].isdigit():
        try:
            s, n = float(r[iS]), float(r[iI])
        except ValueError:
            continue
        st = sorted(((float(r[i]) if r[i] not in ("", "-") else 0.0, h[6:]) for i, h in stall_cols), reverse=True)[:3]
        lines.append((s, n, int(r[0]), r[1].strip()[:70], st))
tot = sum(l[0] for l in lines) or 1
totn = sum(l[1] for l in lines) or 1
print(f"total samples {tot:.0f}, warp-instr {totn:.3e}")
for s, n, ln, src, st in sorted(lines, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100*s/tot:5.1f}% {100*n/totn:5.1f}%i L{ln:<5} {src:70s} {[(h, int(v)) for v, h in st if v]}")
