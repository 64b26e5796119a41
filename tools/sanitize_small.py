"""Small-shape runs of every kernel variant, for compute-sanitizer (racecheck / synccheck /
memcheck).  Each case runs once through the C-ABI (xtc_run) with several tiles per persistent
CTA where the variant supports it (grid_sms), so the cross-tile paths are exercised too.

  compute-sanitizer --tool racecheck python tools/sanitize_small.py [case ...]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_16512_b200 as xtc  # noqa: E402
from seeded_inputs import MODE_INT  # noqa: E402

TC = dict(engine=1, swizzle=128, buffer_c=1)
CASES = {
    "tc_1cta": ("mm", (256, 256, 256), dict(TC, tile_m=128, tile_n=128, tile_k=64, stages=3, acc_buffers=2,
                                            persistent=1, grid_sms=2)),
    "tc_direct": ("mm", (256, 192, 256), dict(engine=1, tile_m=128, tile_n=64, tile_k=64, stages=2, acc_buffers=2,
                                              persistent=1, grid_sms=2)),
    "tc_pair": ("mm", (512, 512, 256), dict(TC, tile_m=256, tile_n=256, tile_k=64, stages=3, acc_buffers=2,
                                            cluster_m=2, persistent=1, grid_sms=2)),
    "tc_headline": ("mm", (1024, 512, 256), dict(TC, tile_m=512, tile_n=256, tile_k=64, stages=3, acc_buffers=1,
                                                 cluster_m=2, persistent=1, grid_sms=2)),
    "tc_cluster_n": ("mm", (256, 512, 256), dict(TC, tile_m=128, tile_n=128, tile_k=64, stages=3, acc_buffers=2,
                                                 cluster_n=2, persistent=1, grid_sms=2)),
    "tc_splitk": ("mm", (256, 256, 512), dict(engine=1, tile_m=128, tile_n=128, tile_k=64, stages=3, split_k=2,
                                              acc_buffers=1)),
    "tc_splitk_cluster": ("mm", (384, 256, 512), dict(engine=1, tile_m=128, tile_n=128, tile_k=64, stages=3,
                                                      split_k=4, split_k_mode=2, acc_buffers=2, persistent=1,
                                                      grid_sms=8)),
    "conv_halo_splitk_cluster": ("conv", (2, 14, 14, 64, 64), dict(engine=1, tile_m=128, tile_n=64, tile_k=64,
                                                                   stages=3, pack_halo=1, split_k=3, split_k_mode=2,
                                                                   acc_buffers=2)),
    "tc_stream_k": ("mm", (384, 256, 512), dict(engine=1, tile_m=128, tile_n=128, tile_k=64, stages=3, buffer_c=1,
                                                acc_buffers=2, persistent=1, grid_sms=7, split_k_mode=3)),
    "conv_halo_stream_k": ("conv", (2, 14, 14, 64, 64), dict(engine=1, tile_m=128, tile_n=64, tile_k=64, stages=3,
                                                            pack_halo=1, buffer_c=1, acc_buffers=2, persistent=1,
                                                            grid_sms=5, split_k_mode=3)),
    "conv_mma_stem": ("stem", (1, 64, 64, 3, 16), dict(engine=2, tile_m=128, tile_n=16, tile_k=32)),
    "conv_mma_patch_tma": ("stem", (2, 64, 64, 3, 16), dict(engine=2, tile_m=64, tile_n=16, tile_k=16, pack_halo=1,
                                                           persistent=1, grid_sms=3)),
    "conv_mma_patch_threads": ("stem", (2, 64, 64, 3, 16), dict(engine=2, tile_m=64, tile_n=16, tile_k=16,
                                                               pack_halo=2, persistent=1, grid_sms=3)),
    "conv_halo_sfold": ("conv", (2, 56, 56, 64, 64), dict(engine=1, tile_m=128, tile_n=64, tile_k=64, stages=2,
                                                         pack_halo=1, b_resident=1, inner_n=192, acc_buffers=2,
                                                         persistent=1, grid_sms=4)),
    "conv_halo_compact": ("conv", (2, 56, 56, 64, 64), dict(engine=1, tile_m=128, tile_n=64, tile_k=64, stages=2,
                                                           pack_halo=2, buffer_c=0, b_resident=1, acc_buffers=2,
                                                           persistent=1, grid_sms=4)),
    "conv_halo_compact_ring": ("conv", (2, 17, 39, 64, 128), dict(engine=1, tile_m=256, tile_n=128, tile_k=64,
                                                                  stages=3, pack_halo=2, buffer_c=0, acc_buffers=2,
                                                                  persistent=1, grid_sms=3)),
    "conv_halo_lean": ("conv", (2, 56, 56, 64, 64), dict(engine=1, tile_m=128, tile_n=64, tile_k=64, stages=2,
                                                        pack_halo=1, b_resident=1, acc_buffers=2, persistent=1,
                                                        grid_sms=4)),
    "tc_3xtf32": ("mm32", (256, 256, 256), dict(TC, tile_m=128, tile_n=128, tile_k=32, stages=3, acc_buffers=2,
                                                persistent=1, grid_sms=2)),
    "conv_im2col": ("conv", (2, 14, 14, 64, 64), dict(TC, tile_m=128, tile_n=64, tile_k=64, stages=3, acc_buffers=2,
                                                      persistent=1, grid_sms=2)),
    "conv_halo": ("conv", (2, 14, 14, 64, 64), dict(TC, tile_m=128, tile_n=64, tile_k=64, stages=2, acc_buffers=2,
                                                    pack_halo=1, persistent=1, grid_sms=2)),
    "simt": ("mm32", (128, 128, 64), dict(engine=0, tile_m=64, tile_n=64, tile_k=16, inner_m=4, inner_n=4,
                                          stages=2, swizzle=4)),
}


def run(name):
    kind, shape, sch = CASES[name]
    st = torch.cuda.current_stream().cuda_stream
    if kind in ("conv", "stem"):
        n, h, w, c, f = shape
        r, sd, pd = (7, 2, 3) if kind == "stem" else (3, 1, 1)
        d = xtc.conv2d_desc(n, h, w, c, f, r, r, sd, pd, "bf16", "bf16")
        M, N, K = xtc.gemm_view(d)
        a = torch.empty((n, h, w, c), dtype=torch.bfloat16, device="cuda")
        b = torch.empty((r, r, c, f), dtype=torch.bfloat16, device="cuda")
        out = torch.bfloat16
    else:
        M, N, K = shape
        dt = "bf16" if kind == "mm" else "f32"
        d = xtc.matmul_desc(M, N, K, dt, dt)
        tdt = torch.bfloat16 if dt == "bf16" else torch.float32
        a = torch.empty((M, K), dtype=tdt, device="cuda")
        b = torch.empty((K, N), dtype=tdt, device="cuda")
        out = tdt
    c = torch.empty((M, N), dtype=out, device="cuda")
    for t, s in ((a, 1), (b, 2)):
        xtc.xtc_fill(t.data_ptr(), t.numel(), xtc.XTC_BF16 if t.dtype == torch.bfloat16 else xtc.XTC_F32, s,
                     MODE_INT, 0, st)
    op = xtc.Op(d).apply(xtc.schedule(**sch))
    op.run(a, b, c)
    torch.cuda.synchronize()
    print(f"{name}: ok ({op.launches()} launches)", flush=True)


if __name__ == "__main__":
    for n in (sys.argv[1:] or list(CASES)):
        run(n)
