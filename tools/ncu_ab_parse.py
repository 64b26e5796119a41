"""Split an ncu launch CSV (tools/conv_ncu_ab.py) at the marker fill kernels: per variant the kernels and
the median duration of the REPS launches.  python tools/ncu_ab_parse.py launches.csv order.json"""
import csv, json, statistics, sys
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
seq = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
order = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
groups, cur = [], None
for name, t in seq:
    if "fill" in name.lower() and "xtc" not in name.lower():
        cur = []
        groups.append(cur)
    elif cur is not None:
        cur.append((name, t))
import os
REPS = int(os.environ.get("REPS", "3"))
for label, g in zip(order, groups):
    # the variant's own REPS launches: cuDNN's first REPS kernels, ours the first REPS xtc kernels (the
    # group also holds the next layer's setup kernels up to the next marker)
    mine = [(n, t) for n, t in g if ("xtc" in n) != label.endswith(":cudnn")][:REPS]
    ts = sorted(t for _, t in mine)
    print(f"{label:28s} {ts[len(ts) // 2] / 1e3:8.2f} us (median of {len(ts)})  {sorted({n[:70] for n, _ in mine})}")
