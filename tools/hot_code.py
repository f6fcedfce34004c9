"""Scratch: hot-code footprint of a kernel from an ncu --set full capture (SASS page).

  python tools/hot_code.py rep.ncu-rep [gap]
Clusters executed instructions into contiguous address regions (gap in bytes), prints each region's
size, executed warp-instructions and stall samples, and the footprint covering 99% of executions.
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
gap = int(sys.argv[2]) if len(sys.argv) > 2 else 256
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ai, ei, si = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ins = []
for r in rows[2:]:
    if len(r) < len(hdr) - 2:
        continue
    try:
        ins.append((int(r[ai], 16), int(r[ei]), int(r[si]), r[1].strip()))
    except ValueError:
        pass
ins.sort()
base = ins[0][0]
tot = sum(e for _, e, _, _ in ins)
print(f"{len(ins)} instructions ({len(ins) * 16 / 1024:.0f} KB), {tot:.3e} warp-instr executed")
# footprint covering 99% of executions
srt = sorted(ins, key=lambda x: -x[1])
acc = 0
for n, (_, e, _, _) in enumerate(srt, 1):
    acc += e
    if acc >= 0.99 * tot:
        print(f"99% of executions in {n} instructions = {n * 16 / 1024:.1f} KB"); break
regs = []
cur = None
for a, e, s, t in ins:
    if e == 0:
        continue
    if cur and a - cur[1] <= gap:
        cur[1] = a; cur[2] += e; cur[3] += s; cur[4] += 1
    else:
        if cur: regs.append(cur)
        cur = [a, a, e, s, 1]
regs.append(cur)
regs.sort(key=lambda r: -r[2])
for r in regs[:25]:
    print(f"  0x{r[0]-base:06x}-0x{r[1]-base:06x} {((r[1]-r[0])//16+1)*16/1024:6.1f} KB  exec {r[2]/tot*100:5.1f}%  stall-samples {r[3]}  n_exec_instr {r[4]}")
