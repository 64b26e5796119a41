mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "halo" > gpurun_out/pytest_halo.log 2>&1; echo rc=$? >> gpurun_out/pytest_halo.log
timeout 300 python - > gpurun_out/halo_sk.log 2>&1 <<'PY'
import sys, json
sys.path.insert(0, ".")
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import _best, HALO, CONV_SCHEDS
for name, (h, c) in {"L14": (14, 256), "L56": (56, 64)}.items():
    for nb in (1, 2, 4, 8, 16, 32):
        tn = min(c, 128)
        cands = list(CONV_SCHEDS[name]) + [dict(HALO, tile_n=tn, stages=4, split_k=sk, buffer_c=0, acc_buffers=1) for sk in (2, 3, 4, 6, 9)]
        if name == "L56":
            cands += [dict(HALO, tile_n=64, stages=2, split_k=sk, buffer_c=0, b_resident=1, acc_buffers=1) for sk in (3, 9)]
        d = xtc.conv2d_desc(nb, h, h, c, c, 3, 3, 1, 1, "bf16", "bf16")
        r = _best(xtc, torch, torch.device("cuda:0"), d, cands, [(nb, h, h, c), (3, 3, c, c)], 1701.1)
        print(name, nb, json.dumps({"best_us": round(r.get("t_med_us", 0), 2), "tflops": round(r.get("tflops_med", 0), 1), "sched": r.get("schedule")}), flush=True)
PY
echo done
