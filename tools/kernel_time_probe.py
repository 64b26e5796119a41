"""Runs a list of (config, schedule) pairs a few times each, for an ncu launch list
(gpu__time_duration per kernel, no launch overhead) next to the event-timed protocol.

  ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/kernel_time_probe.py
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_16512_b200 as xtc  # noqa: E402

CL = xtc.XTC_SPLITK_CLUSTER
TC = dict(engine=1, tile_m=128, swizzle=128)
HALO = dict(TC, pack_halo=1, acc_buffers=2, persistent=1)
CASES = [
    ("mm512", (512, 512, 512), dict(TC, tile_n=64, tile_k=128, stages=4, buffer_c=1, acc_buffers=1, pack_warps=2)),
    ("mm512", (512, 512, 512), dict(TC, tile_n=64, tile_k=64, stages=4, buffer_c=0, acc_buffers=1, split_k=4,
                                    split_k_mode=CL)),
    ("mm512", (512, 512, 512), dict(TC, tile_n=64, tile_k=64, stages=4, buffer_c=0, acc_buffers=1, split_k=8,
                                    split_k_mode=CL)),
    ("mm512", (512, 512, 512), dict(TC, tile_n=64, tile_k=64, stages=4, buffer_c=1, acc_buffers=1, split_k=4,
                                    split_k_mode=CL)),
    ("mm1024", (1024, 1024, 1024), dict(TC, tile_n=64, tile_k=128, stages=4, buffer_c=1, acc_buffers=2,
                                        raster_group=8, pack_warps=2)),
    ("L14n1", (1, 14, 256), dict(HALO, tile_n=128, tile_k=128, stages=3, buffer_c=1)),
    ("L14n1", (1, 14, 256), dict(HALO, tile_n=64, tile_k=128, stages=3, buffer_c=0, split_k=6, split_k_mode=CL)),
    ("L14n1", (1, 14, 256), dict(HALO, tile_n=128, tile_k=128, stages=3, buffer_c=0, split_k=9, split_k_mode=CL)),
    ("L14n32", (32, 14, 256), dict(HALO, tile_n=128, tile_k=128, stages=3, buffer_c=1)),
    ("L56n1", (1, 56, 64), dict(HALO, tile_n=64, tile_k=64, stages=2, buffer_c=1, b_resident=1)),
    ("L56n32", (32, 56, 64), dict(HALO, tile_n=64, tile_k=64, stages=2, buffer_c=1, b_resident=1)),
    ("L56n32", (32, 56, 64), dict(HALO, tile_n=64, tile_k=64, stages=2, buffer_c=1, b_resident=1, split_k_mode=3)),
    ("mm1024", (1024, 1024, 1024), dict(TC, tile_n=64, tile_k=128, stages=4, buffer_c=1, acc_buffers=2,
                                        persistent=1, split_k_mode=3)),
]


def main():
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = []
    pick = [int(x) for x in sys.argv[1:]]
    for i, (name, shape, sch) in enumerate(CASES):
        if pick and i not in pick:
            continue
        if name.startswith("mm"):
            M, N, K = shape
            d = xtc.matmul_desc(M, N, K, "bf16", "bf16")
            a = torch.empty((M, K), dtype=torch.bfloat16, device=dev)
            b = torch.empty((K, N), dtype=torch.bfloat16, device=dev)
        else:
            n, h, c = shape
            d = xtc.conv2d_desc(n, h, h, c, c, 3, 3, 1, 1, "bf16", "bf16")
            M, N, K = xtc.gemm_view(d)
            a = torch.empty((n, h, h, c), dtype=torch.bfloat16, device=dev)
            b = torch.empty((3, 3, c, c), dtype=torch.bfloat16, device=dev)
        c_ = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        xtc.xtc_fill(a.data_ptr(), a.numel(), xtc.XTC_BF16, 1, 0, 0, st)
        xtc.xtc_fill(b.data_ptr(), b.numel(), xtc.XTC_BF16, 2, 0, 0, st)
        op = xtc.Op(d).apply(xtc.schedule(**sch))
        for _ in range(4):
            flush.add_(1)                      # L2 cold, like the bench's flushed protocol
            op.run(a, b, c_)
        m = op.measure(a, b, c_, xtc.measure_cfg(warmup=2, repeats=20, flush_l2=1, validate=1, reuse_reference=0))
        out.append({"case": name, "sched": sch, "t_med_us": m.t_med_ns / 1e3, "valid": int(m.valid)})
        torch.cuda.synchronize()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
