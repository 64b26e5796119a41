"""N3 model study: the traffic model (paper_2512_16512_b200/model.py) against
hardware counters collected through xtc_measure(counters=...) (CUPTI range profiler) over
GpuStrategy samples of the paper's 1024^2 x 1024^2 matmul (bf16), as the paper's §VI-C does
for its cache model (Table II: Pearson 0.534, Spearman 0.492).
Usage: python tools/model_study.py [n_samples] [out.json]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from scipy import stats
import paper_2512_16512_b200 as xtc
from paper_2512_16512_b200.model import predicted_l2_bytes
from paper_2512_16512_b200.strategy import GpuStrategy

n = int(sys.argv[1]) if len(sys.argv) > 1 else 192
out_path = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/model_study.json"
N = 1024
d = xtc.matmul_desc(N, N, N, "bf16", "bf16")
st = GpuStrategy(d)
samples = st.sample(n, seed=0)
a = torch.empty((N, N), dtype=torch.bfloat16, device="cuda"); b = torch.empty_like(a); c = torch.empty_like(a)
s0 = torch.cuda.current_stream().cuda_stream
xtc.xtc_fill(a.data_ptr(), a.numel(), xtc.XTC_BF16, 1, 0, 0, s0); xtc.xtc_fill(b.data_ptr(), b.numel(), xtc.XTC_BF16, 2, 0, 0, s0)
names = ["gpu.lts__t_bytes.sum", "gpu.lts__t_sectors_srcunit_tex.sum", "gpu.dram__bytes_read.sum",
         "gpu.sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]
op = xtc.Op(d)
# keep the metric names this CUPTI/driver knows (an unknown name makes the whole pass unavailable)
op.apply(st.generate(samples[0]))
for cand in (names, [names[0], names[2], names[3]], [names[0]]):
    m = op.measure(a, b, c, xtc.measure_cfg(warmup=0, repeats=1, validate=0, counters=cand))
    if m.n_counters > 0:
        names = cand
        break
    print("counter set unavailable:", cand, xtc.xtc_last_error())
rows = []
for i, smp in enumerate(samples):
    s = st.generate(smp)
    op.apply(s)
    m = op.measure(a, b, c, xtc.measure_cfg(warmup=1, repeats=5, validate=0, counters=names))
    cv = m.counter_values(names)
    if not cv:
        print("counters unavailable:", xtc.xtc_last_error()); sys.exit(1)
    pred = predicted_l2_bytes(d, s)
    rows.append({"id": i, "schedule": s.as_dict(), "pred": pred, "counters": cv, "t_med_us": m.t_med_ns / 1e3,
                 "tflops": m.tflops_med})
P = np.array([r["pred"]["total"] for r in rows])
res = {"shape": [N, N, N], "dtype": "bf16", "samples": len(rows), "strategy": "GpuStrategy(TC_SLOTS), seed 0",
       "paper_table_ii": {"pearson": 0.534, "spearman": 0.492, "what": "L1 misses vs fully associative cache model, M4 Max"}}
for name in [x for x in names if "pct" not in x]:
    Y = np.array([r["counters"][name] * (32.0 if "sectors" in name else 1.0) for r in rows])
    res[name] = {"pearson": float(stats.pearsonr(P, Y)[0]), "spearman": float(stats.spearmanr(P, Y)[0]),
                 "measured_over_predicted_median": float(np.median(Y / P))}
T = np.array([r["t_med_us"] for r in rows])
res["time_vs_predicted_traffic"] = {"pearson": float(stats.pearsonr(P, T)[0]), "spearman": float(stats.spearmanr(P, T)[0])}
res["rows"] = rows
json.dump(res, open(out_path, "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "rows"}, indent=1))
