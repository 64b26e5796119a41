"""Quick perf probe of a few schedules (development aid; bench.py is the contract).

Sustained GEMM load drives the B200 into its power cap (SM clock 1.9 -> 1.2 GHz
over a few hundred ms), so a single pass over a candidate list is biased
toward the first candidates.  probe() therefore interleaves `rounds` passes
over the list, idles `cool_s` between measurements and reports, per schedule,
the best and the median of its per-round medians (and the NVML clock seen)."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_16512_b200 as xtc


def probe(M, N, K, in_dt, out_dt, scheds, validate=0, repeats=10, rounds=3, cool_s=0.3, cublas=True):
    desc = xtc.matmul_desc(M, N, K, in_dt, out_dt)
    tdt = torch.bfloat16 if in_dt == "bf16" else torch.float32
    odt = torch.bfloat16 if out_dt == "bf16" else torch.float32
    a = torch.empty((M, K), dtype=tdt, device="cuda:0")
    b = torch.empty((K, N), dtype=tdt, device="cuda:0")
    c = torch.empty((M, N), dtype=odt, device="cuda:0")
    st = torch.cuda.current_stream().cuda_stream
    xtc.xtc_fill(a.data_ptr(), M * K, xtc.DTYPES[in_dt], 1, 0, 0, st)
    xtc.xtc_fill(b.data_ptr(), K * N, xtc.DTYPES[in_dt], 2, 0, 0, st)
    op = xtc.Op(desc)
    res = {i: {"tf": [], "clk": [], "valid": None, "err": None} for i in range(len(scheds))}
    for r in range(rounds):
        for i, s in enumerate(scheds):
            if res[i]["err"]:
                continue
            try:
                op.apply(xtc.schedule(**s))
                m = op.measure(a, b, c, xtc.measure_cfg(warmup=3, repeats=repeats, validate=validate if r == 0 else 0,
                                                        reuse_reference=1, peak_tflops=1701.1))
                res[i]["tf"].append(m.tflops_med)
                res[i]["clk"].append(m.sm_clock_mhz)
                if r == 0:
                    res[i]["valid"] = m.valid
            except Exception as e:
                res[i]["err"] = str(e)
            time.sleep(cool_s)
    for i, s in enumerate(scheds):
        rec = res[i]
        if rec["err"]:
            print(json.dumps({"shape": [M, N, K, in_dt, out_dt], "sch": s, "error": rec["err"]}), flush=True)
            continue
        print(json.dumps({"shape": [M, N, K, in_dt, out_dt], "sch": s, "tflops_med": round(statistics.median(rec["tf"]), 1),
                          "tflops_best": round(max(rec["tf"]), 1), "rounds": [round(x, 1) for x in rec["tf"]],
                          "valid": rec["valid"], "clk": rec["clk"]}), flush=True)
    if cublas and in_dt == "bf16":
        for _ in range(3):
            torch.matmul(a, b)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10):
            torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 10 * 1e-3
        print(json.dumps({"shape": [M, N, K], "cublas_tflops": round(2 * M * N * K / t / 1e12, 1)}), flush=True)


TC = dict(engine=1, tile_m=128, tile_k=64, swizzle=128, buffer_c=1)

if __name__ == "__main__":
    P = dict(TC, tile_m=256, cluster_m=2, tile_n=256, tile_k=128, stages=3, acc_buffers=2, persistent=1)
    probe(8192, 8192, 8192, "bf16", "bf16", [dict(P, raster_group=16), dict(P, raster_group=6)], validate=1)
