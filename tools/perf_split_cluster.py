"""A/B: split_k_mode 2 (K segments of a tile = one cluster's CTAs, in-kernel ordered reduction)
against the best round-1 schedules on the parallelism-bound BASELINE configs (512^3 / 1024^3 bf16,
conv L14 / L56 at small batch).  Same protocol as bench.py extras: validated on chip, L2 flushed,
median of 20 event-timed reps.  Prints one JSON object per config."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_16512_b200 as xtc  # noqa: E402
from paper_2512_16512_b200 import bench_extras as bx  # noqa: E402

CL = xtc.XTC_SPLITK_CLUSTER
TC = dict(engine=1, tile_m=128, swizzle=128, buffer_c=0, acc_buffers=1, split_k_mode=CL)


def mm_cands(n):
    out = []
    for tn in (64, 128):
        for tk in (64, 128):
            kb = n // tk
            for sk in (2, 3, 4, 6, 8, 12, 16):
                if sk > kb or (sk - 1) * -(-kb // sk) >= kb:
                    continue
                if (n // 128) * (n // tn) * sk > 148 * 2:
                    continue
                out.append(dict(TC, tile_n=tn, tile_k=tk, stages=4 if tk == 64 else 3, split_k=sk))
        for tk in (64, 128):
            out.append(dict(TC, tile_n=tn, tile_k=tk, stages=4, buffer_c=1, acc_buffers=2, persistent=1,
                            split_k_mode=xtc.XTC_SPLITK_STREAM))
    return out


SKM = xtc.XTC_SPLITK_STREAM


def conv_cands(name, nb):
    halo = dict(TC, pack_halo=1, acc_buffers=2)
    out = []
    # stream-K over the persistent grid: the same schedules as the data-parallel best, split points from the grid
    if name == "L56":
        out += [dict(halo, tile_n=64, tile_k=64, stages=2, buffer_c=1, b_resident=1, persistent=1, split_k_mode=SKM),
                dict(halo, tile_n=64, tile_k=64, stages=2, buffer_c=1, persistent=1, split_k_mode=SKM)]
    else:
        out += [dict(halo, tile_n=128, tile_k=128, stages=3, buffer_c=1, persistent=1, split_k_mode=SKM),
                dict(halo, tile_n=64, tile_k=128, stages=3, buffer_c=1, persistent=1, split_k_mode=SKM)]
    if name == "L14":
        for tn in (64, 128):
            for sk in (2, 3, 6, 9, 18):
                out.append(dict(halo, tile_n=tn, tile_k=128, stages=3, split_k=sk))
        for sk in (2, 4, 8, 12, 16):
            out.append(dict(TC, tile_n=128, tile_k=128, stages=3, split_k=sk))
    else:
        for sk in (2, 3, 9):
            out.append(dict(halo, tile_n=64, tile_k=64, stages=3, split_k=sk))
    return out


def main():
    dev = torch.device("cuda:0")
    peak = 1638.9
    only = sys.argv[1:]
    for n in (512, 1024):
        if only and f"mm{n}" not in only:
            continue
        d = xtc.matmul_desc(n, n, n, "bf16", "bf16")
        cands = bx.MATMUL_SCHEDS[n] + mm_cands(n)
        r = bx._best(xtc, torch, dev, d, cands, [(n, n), (n, n)], peak)
        r["tried"] = [dict(row, sched=c) for row, c in zip(r.get("tried", []), cands)]
        print(json.dumps({"config": f"matmul_{n}_bf16", **r}), flush=True)
    for name, (h, c) in {"L14": (14, 256), "L56": (56, 64)}.items():
        for nb in (1, 8, 32):
            if only and f"{name}n{nb}" not in only:
                continue
            d = xtc.conv2d_desc(nb, h, h, c, c, 3, 3, 1, 1, "bf16", "bf16")
            cands = list(bx.CONV_SCHEDS[name]) + conv_cands(name, nb)
            r = bx._best(xtc, torch, dev, d, cands, [(nb, h, h, c), (3, 3, c, c)], peak)
            r["tried"] = [dict(row, sched=c) for row, c in zip(r.get("tried", []), cands)]
            print(json.dumps({"config": f"conv_{name}_n{nb}", **r}), flush=True)


if __name__ == "__main__":
    main()
