"""Summarise XTC_TRACE output: per CTA, load latency (producer issue -> MMA sees data),
MMA inter-stage gaps, epilogue durations.  All times in microseconds."""
import json, statistics, sys
for ln in (open(sys.argv[1]) if len(sys.argv) < 3 else []):
    d = json.loads(ln)
    S, kK, kT = d["slots"], d["kK"], d["kT"]
    t = d["t"]
    print(f"M={d['M']} N={d['N']} K={d['K']} tile_n={d['tile_n']} tile_k={d['tile_k']} stages={d['stages']} "
          f"cg={d['cta_group']} grid={d['grid']} tiles={d['num_tiles']} kb/split={d['kb_per_split']}")
    for c in range(len(t) // S):
        r = t[c * S:(c + 1) * S]
        if not r[0]:
            continue
        t0 = r[0]
        prod = [x for x in r[8:8 + kK] if x]
        mma = [x for x in r[8 + kK:8 + 2 * kK] if x]
        epi = r[8 + 2 * kK:8 + 2 * kK + 2 * kT]
        n = min(len(prod), len(mma))
        lat = [(mma[i] - prod[i]) / 1e3 for i in range(n)]
        gaps = [(mma[i + 1] - mma[i]) / 1e3 for i in range(len(mma) - 1)]
        tiles = [((epi[2 * j] - t0) / 1e3, (epi[2 * j + 1] - epi[2 * j]) / 1e3) for j in range(kT) if epi[2 * j]]
        print(f"  cta{c}: setup {(r[1] - t0) / 1e3:.2f}  first issue {(prod[0] - t0) / 1e3 if prod else -1:.2f}  "
              f"first data {(mma[0] - t0) / 1e3 if mma else -1:.2f}  "
              f"issue->data med {statistics.median(lat) if lat else -1:.2f} max {max(lat) if lat else -1:.2f}  "
              f"mma gap med {statistics.median(gaps) if gaps else -1:.3f}")
        print("        epilogue (start, dur): " + " ".join(f"({a:.2f},{b:.2f})" for a, b in tiles[:8]))


def grid_summary(path):
    """Whole-grid view: CTA start/end spread, tiles per CTA, per-tile time."""
    for ln in open(path):
        d = json.loads(ln)
        S, kK, kT = d["slots"], d["kK"], d["kT"]
        t = d["t"]
        rows = [t[c * S:(c + 1) * S] for c in range(len(t) // S)]
        rows = [r for r in rows if r[0]]
        t0 = min(r[0] for r in rows)
        starts = [(r[0] - t0) / 1e3 for r in rows]
        ends = [(r[2] - t0) / 1e3 for r in rows if r[2]]
        ntiles = [sum(1 for j in range(kT) if r[8 + 2 * kK + 2 * j]) for r in rows]
        print(f"grid: {len(rows)} CTAs traced; start spread {min(starts):.2f}..{max(starts):.2f} us; "
              f"end min/med/max {min(ends):.2f}/{statistics.median(ends):.2f}/{max(ends):.2f} us; "
              f"tiles/CTA min/max {min(ntiles)}/{max(ntiles)}")
        slow = sorted(range(len(rows)), key=lambda c: -(rows[c][2] - rows[c][0]))[:3]
        for c in slow:
            r = rows[c]
            ep = [((r[8 + 2 * kK + 2 * j] - t0) / 1e3) for j in range(kT) if r[8 + 2 * kK + 2 * j]]
            print(f"  slow cta{c}: start {(r[0] - t0) / 1e3:.2f} end {(r[2] - t0) / 1e3:.2f} epilogue starts "
                  + " ".join(f"{x:.2f}" for x in ep))


if __name__ == "__main__" and len(sys.argv) > 2 and sys.argv[2] == "grid":
    grid_summary(sys.argv[1])
