"""Scratch: warp-stall samples of an ncu --set full capture per CUDA source line, by joining the
capture's SASS view (per-address samples) with the line table of a cubin of the same sources
(nvdisasm --print-line-info).  python tools/stall_lines.py rep.ncu-rep lib.cubin kernel_substring [n]"""
import collections, csv, io, re, subprocess, sys

rep, cubin, kern = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
dis = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
cur = fn = None
amap = {}
for l in dis.splitlines():
    m = re.search(r"\.section\s+\.text\.([^,\s]+)", l)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r'## File "(.*?)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m and fn and kern in fn:
        amap[int(m.group(1), 16)] = cur
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
ai, wi = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
base = min(int(r[ai], 16) for r in rows[2:] if len(r) >= len(hdr))    # absolute -> function-relative
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
tot = collections.Counter()
by = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    a = int(r[ai], 16) - base
    line = amap.get(a)
    s = int(r[wi] or 0)
    tot["all"] += s
    by[line]["all"] += s
    for c in cols:
        v = int(r[hdr.index(c)] or 0)
        tot[c] += v
        by[line][c] += v
print(f"samples {tot['all']}, mapped addresses {len(amap)}")
print("share of all samples per reason:", {c: round(100 * tot[c] / tot['all'], 2) for c in cols if tot[c]})
for c in ("all", "stall_long_sb"):
    print(f"-- top lines by {c}")
    for line, cnt in sorted(by.items(), key=lambda kv: -kv[1][c])[:top]:
        if cnt[c]:
            print(f"  {100 * cnt[c] / tot['all']:6.2f}%  {line}")
