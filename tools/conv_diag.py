"""Conv vs same-shape GEMM: isolates the cost of TMA im2col addressing."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16512_b200 as xtc

def bench(desc, shapes, sch, reps=30):
    M, N, K = xtc.gemm_view(desc)
    a = torch.empty(shapes[0], dtype=torch.bfloat16, device="cuda"); b = torch.empty(shapes[1], dtype=torch.bfloat16, device="cuda")
    c = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    xtc.xtc_fill(a.data_ptr(), a.numel(), xtc.XTC_BF16, 1, 0, 0, st); xtc.xtc_fill(b.data_ptr(), b.numel(), xtc.XTC_BF16, 2, 0, 0, st)
    op = xtc.Op(desc)
    try:
        op.apply(xtc.schedule(**sch))
    except Exception as e:
        return str(e)[:60]
    out = {}
    for flush in (0, 1):
        m = op.measure(a, b, c, xtc.measure_cfg(warmup=3, repeats=reps, flush_l2=flush, validate=1, reuse_reference=1))
        out["cold" if flush else "warm"] = (round(m.tflops_med, 1), round(m.t_med_ns / 1e3, 2), m.valid)
    return out

TC = dict(engine=1, tile_m=128, tile_k=64, swizzle=128, buffer_c=1)
P2 = dict(TC, tile_m=256, cluster_m=2)
if __name__ == "__main__":
  for name, (B, H, C, F) in {"L56": (32, 56, 64, 64), "L14": (32, 14, 256, 256)}.items():
      d = xtc.conv2d_desc(B, H, H, C, F)
      M, N, K = xtc.gemm_view(d)
      dm = xtc.matmul_desc(M, N, K, "bf16", "bf16")
      scheds = [dict(TC, tile_n=min(F, 256), stages=8 if F == 64 else 4, acc_buffers=2, persistent=1, raster_group=8),
                dict(TC, tile_n=min(F, 256), stages=6, acc_buffers=2, persistent=0),
                dict(TC, tile_n=min(F, 256), tile_k=128, stages=4 if F == 64 else 2, acc_buffers=2, persistent=1)]
      if F >= 128:
          scheds += [dict(P2, tile_n=256, tile_k=128, stages=3, acc_buffers=2, persistent=1, split_k=s) for s in (1, 2, 3)]
          scheds += [dict(TC, tile_n=256, stages=4, acc_buffers=1, split_k=3), dict(TC, tile_n=128, stages=6, acc_buffers=2, split_k=2, persistent=1)]
      for s in scheds:
          print(json.dumps({"layer": name, "sch": {k: v for k, v in s.items() if k not in ("engine", "swizzle")},
                            "conv": bench(d, [(B, H, H, C), (3, 3, C, F)], s), "gemm_same_shape": bench(dm, [(M, K), (K, N)], s)}), flush=True)
