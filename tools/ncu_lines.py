"""Scratch: per-source-line executed instructions of a capture (cuda,sass view); optional address window.
  python tools/ncu_lines.py rep.ncu-rep [lo_off hi_off]   (offsets relative to the kernel's first address)
"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
src = ",".join(["/root/repo/paper_2309_07270_b200/csrc/xdrop_kernels.cuh", "/root/repo/paper_2309_07270_b200/csrc/xdrop_pk16.cuh"])
import os
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if not os.environ.get("NO_RESOLVE"):
    cmd += ["--resolve-source-file", src]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
fname, line = "?", "?"
rows = []
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    if r[0]:
        line = r[0]; text = r[1]
        continue
    if r[2].startswith("0x"):
        rows.append((int(r[2], 16), fname, int(line), text, int(r[7]) if r[7] not in ("-", "") else 0, r[3].strip()))
base = min(a for a, *_ in rows)
lo, hi = (int(sys.argv[2], 16), int(sys.argv[3], 16)) if len(sys.argv) > 3 else (0, 1 << 40)
agg = collections.defaultdict(lambda: [0, 0, ""])
for a, f, l, t, e, s in rows:
    if lo <= a - base <= hi:
        k = (f, l); agg[k][0] += e; agg[k][1] += 1; agg[k][2] = t
tot = sum(v[0] for v in agg.values())
for (f, l), (e, n, t) in sorted(agg.items(), key=lambda x: -x[1][0])[:400]:
    print(f"{f}:{l:5d} exec {e/ max(tot,1)*100:5.1f}% ({e:.2e}) n_sass {n:4d}  {t.strip()[:90]}")
