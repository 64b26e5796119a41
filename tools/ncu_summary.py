"""Summarise an ncu report (.ncu-rep) and a launch list (.csv) into profiles/.

  python tools/ncu_summary.py REPORT.ncu-rep LAUNCHES.csv OUT_PREFIX [algorithmic_flops] [algorithmic_bytes]
Writes OUT_PREFIX.txt (human) and updates profiles/ncu_summary.json (read by bench.py for `traffic`)."""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "sm__warps_active.avg.per_cycle_active"]

UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            d[h] = (v, u)
        kernels.append(d)
    return kernels


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = {}
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        t = float(r[vi].replace(",", ""))
        n, s = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, s + t)
    return agg


def main():
    rep, lcsv, prefix = sys.argv[1], sys.argv[2], sys.argv[3]
    flops = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
    abytes = float(sys.argv[5]) if len(sys.argv) > 5 else 0.0
    ks = raw(rep)
    lines = [f"ncu --set full summary of {os.path.basename(rep)}"]
    summ = {}
    for i, k in enumerate(ks):
        name = k.get("Kernel Name", ("?", ""))[0]
        lines.append(f"[{i}] {name}")
        rec = {}
        for key in KEYS:
            if key in k:
                v, u = k[key]
                lines.append(f"    {key:70s} {v} {u}")
                rec[key] = (v, u)
        rb = float(k["dram__bytes_read.sum"][0].replace(",", "")) * UNIT.get(k["dram__bytes_read.sum"][1], 1)
        wb = float(k["dram__bytes_write.sum"][0].replace(",", "")) * UNIT.get(k["dram__bytes_write.sum"][1], 1)
        t_us = float(k["gpu__time_duration.sum"][0].replace(",", ""))
        lines.append(f"    dram traffic per launch = {rb + wb:.4g} B (algorithmic {abytes:.4g} B, ratio "
                     f"{(rb + wb) / abytes if abytes else float('nan'):.2f})")
        if flops:
            lines.append(f"    achieved under ncu = {flops / (t_us * 1e-6) / 1e12:.1f} TFLOP/s")
        summ = {"kernel": name, "dram_bytes_per_launch": rb + wb, "dram_read": rb, "dram_write": wb,
                "duration_us_under_ncu": t_us, "algorithmic_bytes": abytes, "algorithmic_flops": flops,
                "tensor_active_pct_elapsed": float(k.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", ("nan", ""))[0]),
                "report": os.path.basename(rep)}
    if lcsv and os.path.exists(lcsv):
        agg = launches(lcsv)
        tot = sum(s for _, s in agg.values())
        lines.append("launch list (ncu --metrics gpu__time_duration.sum, cold/serialised):")
        for name, (n, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"    {name:40s} launches={n:4d} total_ns={s:14.0f} share={s / tot:6.1%}")
    open(prefix + ".txt", "w").write("\n".join(lines) + "\n")
    js = os.path.join(os.path.dirname(prefix), "ncu_summary.json")
    allj = json.load(open(js)) if os.path.exists(js) else {}
    allj[os.path.basename(prefix)] = summ
    if "headline" in os.path.basename(prefix):
        allj["headline_kernel"] = summ
    json.dump(allj, open(js, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
