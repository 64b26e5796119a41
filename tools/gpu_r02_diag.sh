L56='{"engine":1,"tile_m":128,"tile_k":64,"swizzle":128,"pack_halo":1,"buffer_c":1,"acc_buffers":2,"persistent":1,"tile_m":128,"tile_n":64,"stages":2,"b_resident":1}'
for m in 0 8192; do
XTC_DEBUG_SKIP=$m RUN_ONE_WARM=100 XTC_TRACE=gpurun_out/trb$m.jsonl timeout 120 python tools/run_one.py conv 1 56 56 64 64 bf16 bf16 "$L56" 1 > /dev/null 2>&1
python - >> gpurun_out/trb.txt 2>&1 <<PY
import json
d = json.loads(open("gpurun_out/trb$m.jsonl").readline()); S = d["slots"]; kK = d["kK"]; t = d["t"]
rows = [t[c*S:(c+1)*S] for c in range(len(t)//S)]
rows = [r for r in rows if r[0]]
t0 = min(r[0] for r in rows)
f = lambda x: round((x - t0)/1e3, 2) if x else None
print("mask $m")
for c in (0, 1):
    r = rows[c]
    print("  cta", c, "entry", f(r[0]), "setup", f(r[1]), "thread0 at", f(r[3]), "count", r[4], "thread0 past final barrier", f(r[2]), "warp4 past", f(r[5]), "stores done", f(r[6]), "tmem freed", f(r[7]))
PY
done
