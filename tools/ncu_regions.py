"""Executed-instruction regions of one kernel in an ncu report (runs of SASS with equal execution counts),
largest first, plus the run's stall samples.  python tools/ncu_regions.py REPORT [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
k = [i for i, r in enumerate(rows[:5]) if "Source" in r][0]
hdr = rows[k]; ie = hdr.index("Instructions Executed"); si = hdr.index("Source")
ss = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[k + 1:]:
    try:
        data.append((int(r[0], 16), float(r[ie] or 0), float(r[ss] or 0), r[si].strip()))
    except (ValueError, IndexError):
        pass
segs, cur = [], None
for a, c, st, s in data:
    if cur and cur[1] == c:
        cur[2] += 1; cur[3] += st; cur[5] = s
    else:
        cur = [a, c, 1, st, s, s]; segs.append(cur)
tot = sum(d[1] for d in data) or 1; tst = sum(d[2] for d in data) or 1
print(f"total warp-instructions {tot:.0f}, stall samples {tst:.0f}")
for a, c, n, st, s0, s1 in sorted(segs, key=lambda x: -(x[1] * x[2] + x[3] * tot / tst))[:top]:
    print(f"{hex(a)[-5:]} exec {c:9.0f} x {n:3d} = {c * n / tot:6.1%} instr, {st / tst:6.1%} stalls | {s0[:46]} .. {s1[:36]}")
