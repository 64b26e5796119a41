mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "halo" > gpurun_out/pytest_halo.log 2>&1; echo rc=$? >> gpurun_out/pytest_halo.log
timeout 300 python - > gpurun_out/halo_mc.log 2>&1 <<'PY'
import os, sys, json
sys.path.insert(0, ".")
import torch
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.bench_extras import _best, HALO
cands = [dict(HALO, tile_n=128, tile_k=128, stages=3), dict(HALO, cluster_m=2, tile_n=128, tile_k=128, stages=3),
         dict(HALO, cluster_m=2, tile_n=128, tile_k=64, stages=4), dict(HALO, cluster_m=2, tile_n=256, tile_k=64, stages=3, acc_buffers=1),
         dict(HALO, cluster_m=2, tile_n=128, tile_k=128, stages=3, buffer_c=0), dict(HALO, cluster_m=2, tile_n=128, tile_k=64, stages=4, persistent=0)]
for nb in (32, 8, 1):
    d = xtc.conv2d_desc(nb, 14, 14, 256, 256, 3, 3, 1, 1, "bf16", "bf16")
    r = _best(xtc, torch, torch.device("cuda:0"), d, cands, [(nb, 14, 14, 256), (3, 3, 256, 256)], 1701.1)
    print("L14 n%d" % nb, json.dumps({"best_us": r.get("t_med_us"), "tflops": r.get("tflops_med"), "sched": r.get("schedule"), "tried": r.get("tried")}), flush=True)
PY
echo done
