"""Summarise an ncu launch list (gpu__time_duration) and an ncu --set full report
into a markdown table + traffic.json (per-launch DRAM bytes) under profiles/."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.append((d["Kernel Name"].split("(")[0].replace("void ", ""), float(d["Metric Value"])))
    return out


def full(rep):
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    want = {"Kernel Name": "kernel", "gpu__time_duration.sum": "time",
            "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
            "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
            "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pct2",
            "dram__bytes_read.sum.pct_of_peak_sustained_elapsed": "dram_read_pct",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
            "launch__registers_per_thread": "regs"}
    idx = {v: (h.index(k), u[h.index(k)]) for k, v in want.items() if k in h}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ms": 1e-3, "us": 1e-6,
             "ns": 1e-9, "s": 1}
    res = []
    for r in rows[2:]:
        d = {}
        for k, (i, unit) in idx.items():
            v = r[i]
            if k == "kernel":
                d[k] = v.split("(")[0].replace("void ", "")
                continue
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                x = None
            if x is not None and unit in scale:
                x *= scale[unit]
            d[k] = x
        res.append(d)
    return res


if __name__ == "__main__":
    lpath, rep, md, tj, label = sys.argv[1:6]
    L = launches(lpath)
    tot = sum(v for _, v in L)
    agg, cnt = defaultdict(float), defaultdict(int)
    for n, v in L:
        agg[n] += v
        cnt[n] += 1
    F = full(rep)
    lines = [f"# ncu summary — {label}", "",
             "One kvtc_compress + kvtc_decompress of the bench workload (Llama-3.1-8B shape, 32768 tokens, CR 16),",
             "scripts/profile_run.py under ncu (--clock-control none).  Launch list: cold-cache, serialised",
             "(compare SHARES).  Source: " + lpath + ", " + rep, "",
             "## Launch list (gpu__time_duration.sum)", "", "| kernel | launches | ms | share |", "|---|---|---|---|"]
    for n, v in sorted(agg.items(), key=lambda x: -x[1]):
        lines.append(f"| `{n}` | {cnt[n]} | {v / 1e6:.3f} | {100 * v / tot:.1f} % |")
    lines += [f"| total | {len(L)} | {tot / 1e6:.3f} | |", "", "## ncu --set full, per launch", "",
              "| kernel | time ms | DRAM read GB | DRAM write GB | DRAM read % peak | L2 % | tensor pipe % | SM % | warps active % | regs |",
              "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for d in F:
        tp = d.get("tensor_pct") if d.get("tensor_pct") is not None else d.get("tensor_pct2")
        f = lambda x, s=1, p=3: "-" if x is None else f"{x / s:.{p}f}"
        lines.append(f"| `{d['kernel']}` | {f(d.get('time'), 1e-3)} | {f(d.get('dram_read'), 1e9)} | "
                     f"{f(d.get('dram_write'), 1e9)} | {f(d.get('dram_read_pct'), 1, 1)} | {f(d.get('l2_pct'), 1, 1)} | "
                     f"{f(tp, 1, 1)} | {f(d.get('sm_pct'), 1, 1)} | {f(d.get('occupancy_pct'), 1, 1)} | "
                     f"{f(d.get('regs'), 1, 0)} |")
        kn = d["kernel"].replace(" ", "")
        kn = kn.replace("kvtc::", "")
        key = ("c.project_quant_gemm" if kn.startswith("gemm_kernel<1")
               else "d.reconstruct_gemm" if kn.startswith("gemm_kernel<2") else None)
        if key and key not in traffic and d.get("dram_read") is not None:
            traffic[key] = d["dram_read"] + (d.get("dram_write") or 0)
    open(md, "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tj, "w"), indent=1)
    print("\n".join(lines))
