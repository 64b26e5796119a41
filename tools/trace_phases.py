"""Per-tile phase totals (XTC_TRACE) of a conv_halo trace: python tools/trace_phases.py TRACE.jsonl"""
import json, statistics, sys
for ln in open(sys.argv[1]):
    d = json.loads(ln)
S, kK, kT = d["slots"], d["kK"], d["kT"]; t = d["t"]; PH = 8 + 2 * kK + 2 * kT
r = t[0:S]; t0 = r[0]; f = lambda x: round((x - t0) / 1e3, 2) if x else None
print(" mma starts", [f(x) for x in r[8 + kK:8 + 2 * kK] if x][:8])
print(" epilogues ", [(f(r[8 + 2 * kK + 2 * j]), f(r[8 + 2 * kK + 2 * j + 1])) for j in range(kT) if r[8 + 2 * kK + 2 * j]][:8],
      "TMEM free", f(r[7]))
rows = [t[c * S:(c + 1) * S] for c in range(len(t) // S)]
rows = [x for x in rows if x[0] and x[PH + 5]]
names = ["tfull wait", "decode", "tmem ld(+fold)", "staging wait", "stage+store+tail"]
print(" epilogue cycles/tile:", {n: int(statistics.median([x[PH + k] / x[PH + 5] for x in rows])) for k, n in enumerate(names)})
print(" MMA warp cycles/tile: wait", int(statistics.median([x[PH + 6] / x[PH + 5] for x in rows])),
      "issue", int(statistics.median([x[PH + 7] / x[PH + 5] for x in rows])))
