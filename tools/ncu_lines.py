"""Aggregate an ncu source (SASS) page by CUDA source line.
usage: python tools/ncu_lines.py REPORT.ncu-rep OBJ.o KERNEL_MANGLED_SUBSTR [topN]"""
import collections, csv, re, subprocess, sys, tempfile, os, glob
rep, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(csvtxt.splitlines()))
h = rows[1]
ai, ii, si = h.index('Address'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
recs = []
for r in rows[2:]:
    try:
        recs.append((int(r[ai], 16), float(r[ii] or 0), float(r[si] or 0), r[h.index('Source')]))
    except Exception:
        pass
base = min(a for a, *_ in recs)
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = glob.glob(os.path.join(d, "*.cubin"))[0]
sass = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout.split("\n")
a2l, cur, inside = {}, None, False
for l in sass:
    if l.startswith(".text."):
        inside = kname in l
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
    m2 = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m2 and cur:
        a2l[int(m2.group(1), 16)] = cur
agg, st = collections.Counter(), collections.Counter()
for a, n, s_, _ in recs:
    k = a2l.get(a - base, ('?', 0))
    agg[k] += n
    st[k] += s_
T, S = sum(agg.values()), sum(st.values())
print(f"total warp-instructions {T:.4g}, stall samples {S:.4g}")
for k, v in sorted(agg.items(), key=lambda kv: -st[kv[0]])[:top]:
    print(f"{k[0]}:{k[1]:<5d} inst {100*v/T:5.1f}%  stall {100*st[k]/S:5.1f}%")
