"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
si, ai = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((float(r[ai] or 0), r[0], r[si].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
for d in sorted(data, reverse=True)[:top]:
    print(f"{d[0] / tot:6.1%}  {d[1][-5:]}  {d[2][:100]}")
