"""Quick perf probe of a few schedules (development aid; bench.py is the contract)."""
import json
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16512_b200 as xtc

def probe(M, N, K, in_dt, out_dt, scheds, validate=0, repeats=10):
    desc = xtc.matmul_desc(M, N, K, in_dt, out_dt)
    tdt = torch.bfloat16 if in_dt == "bf16" else torch.float32
    odt = torch.bfloat16 if out_dt == "bf16" else torch.float32
    a = torch.empty((M, K), dtype=tdt, device="cuda:0"); b = torch.empty((K, N), dtype=tdt, device="cuda:0")
    c = torch.empty((M, N), dtype=odt, device="cuda:0")
    st = torch.cuda.current_stream().cuda_stream
    xtc.xtc_fill(a.data_ptr(), M * K, xtc.DTYPES[in_dt], 1, 0, 0, st)
    xtc.xtc_fill(b.data_ptr(), K * N, xtc.DTYPES[in_dt], 2, 0, 0, st)
    op = xtc.Op(desc)
    for s in scheds:
        sch = xtc.schedule(**s)
        try:
            op.apply(sch)
            m = op.measure(a, b, c, xtc.measure_cfg(warmup=3, repeats=repeats, validate=validate, reuse_reference=1,
                                                    peak_tflops=1701.1))
            print(json.dumps({"shape": [M, N, K, in_dt, out_dt], "sch": s, "tflops_med": round(m.tflops_med, 1),
                              "t_med_us": round(m.t_med_ns / 1e3, 2), "valid": m.valid,
                              "err": m.max_norm_err, "clk": m.sm_clock_mhz}), flush=True)
        except Exception as e:
            print(json.dumps({"shape": [M, N, K], "sch": s, "error": str(e)}), flush=True)
    # torch reference point (cuBLAS) for context
    if in_dt == "bf16":
        for _ in range(3): torch.matmul(a, b)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10): torch.matmul(a, b)
        e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 10 * 1e-3
        print(json.dumps({"shape": [M, N, K], "cublas_tflops": round(2 * M * N * K / t / 1e12, 1)}), flush=True)

TC = dict(engine=1, tile_m=128, tile_k=64, swizzle=128, buffer_c=1)
if __name__ == "__main__":
    big = [dict(TC, tile_n=256, stages=4, acc_buffers=2, persistent=1, raster_group=8),
           dict(TC, tile_n=256, stages=4, acc_buffers=2, persistent=1, raster_group=16),
           dict(TC, tile_n=256, stages=4, acc_buffers=1, persistent=0),
           dict(TC, tile_n=128, stages=6, acc_buffers=2, persistent=1, raster_group=8),
           dict(TC, tile_n=256, tile_k=128, stages=2, acc_buffers=2, persistent=1, raster_group=8)]
    probe(8192, 8192, 8192, "bf16", "bf16", big, validate=int(os.environ.get("VAL", "0")))
    probe(1024, 1024, 1024, "bf16", "bf16", [dict(TC, tile_n=128, stages=4, acc_buffers=2, persistent=1),
                                              dict(TC, tile_n=64, stages=4, acc_buffers=2, persistent=1),
                                              dict(TC, tile_n=128, stages=4, split_k=2, persistent=1)], validate=1)
    probe(1024, 1024, 1024, "f32", "f32", [dict(engine=0, tile_m=128, tile_n=128, tile_k=16, inner_m=8, inner_n=8,
                                                 unroll_k=4, vector_n=4, stages=2, swizzle=4),
                                            dict(engine=0, tile_m=64, tile_n=64, tile_k=16, inner_m=4, inner_n=4,
                                                 unroll_k=4, vector_n=4, stages=2, swizzle=4)], validate=1)
