"""Summarise the ncu evidence of tools/ncu_capture.sh (run here, no GPU):
launch list -> per-kernel device time and DRAM bytes; --set full reports ->
duration, DRAM bytes/throughput, tensor-pipe and SM activity, registers.
Writes profiles/ncu_<config>_<tag>.json and prints it.

    python tools/ncu_summary.py c2 r01
"""
import csv
import io
import json
import os
import statistics
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")

RAW_METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__cluster_dim_x",
    "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_active.avg",
    "gpc__cycles_elapsed.max",
]


def short(name):
    for k in ("ffn_persistent_kernel", "front_kernel", "combine_slots_kernel", "combine_dense_kernel",
              "ep_wait_kernel", "tile_gemm_kernel",
              "fused_route_kernel", "gate_topk_kernel", "coreset_kernel",
              "constrained_route_kernel", "permute_kernel"):
        if k in name:
            return k
    return name[:60]


def launches(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                      hdr.index("Metric Value"), hdr.index("ID"))
    per = defaultdict(dict)
    for r in rows[1:]:
        try:
            per[(int(r[ii]), short(r[ki]))][r[mi]] = float(r[vi].replace(",", ""))
        except (ValueError, IndexError):
            pass
    agg = defaultdict(lambda: defaultdict(list))
    for (_, k), mets in per.items():
        for mname, v in mets.items():
            agg[k][mname].append(v)
    out = {}
    for k, mets in agg.items():
        t = mets.get("gpu__time_duration.sum", [])
        rd = mets.get("dram__bytes_read.sum", [])
        wr = mets.get("dram__bytes_write.sum", [])
        out[k] = {"launches": len(t),
                  "median_us": round(statistics.median(t) / 1e3, 2) if t else None,
                  "mean_dram_read_MB": round(statistics.mean(rd) / 1e6, 2) if rd else None,
                  "mean_dram_write_MB": round(statistics.mean(wr) / 1e6, 2) if wr else None}
    return out


def full_report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return {}
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {"kernel": short(vals[hdr.index("Kernel Name")])}
    for m in RAW_METRICS:
        if m in hdr:
            i = hdr.index(m)
            v = vals[i].replace(",", "")
            try:
                res[m] = float(v)
            except ValueError:
                res[m] = v
            if units[i]:
                res[m + " [unit]"] = units[i]
    return res


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    tag = sys.argv[2] if len(sys.argv) > 2 else "r01"
    summ = {"config": cfg, "tag": tag,
            "source": "tools/ncu_capture.sh under gpurun (B200, --clock-control none)"}
    lp = os.path.join(OUT, f"launches_{cfg}_{tag}.csv")
    if os.path.exists(lp):
        summ["launch_list"] = launches(lp)
    for kern in ("ffn", "front"):
        rp = os.path.join(OUT, f"{kern}_{cfg}_{tag}.ncu-rep")
        if os.path.exists(rp):
            summ[f"{kern}_full"] = full_report(rp)
    ffn = summ.get("ffn_full", {})
    if "dram__bytes_read.sum" in ffn:
        rd = ffn["dram__bytes_read.sum"] * (1e6 if ffn.get("dram__bytes_read.sum [unit]") == "Mbyte"
                                           else 1e3 if ffn.get("dram__bytes_read.sum [unit]") == "Kbyte"
                                           else 1e9 if ffn.get("dram__bytes_read.sum [unit]") == "Gbyte" else 1)
        wr = ffn.get("dram__bytes_write.sum", 0) * (1e6 if ffn.get("dram__bytes_write.sum [unit]") == "Mbyte"
                                                   else 1e3 if ffn.get("dram__bytes_write.sum [unit]") == "Kbyte"
                                                   else 1e9 if ffn.get("dram__bytes_write.sum [unit]") == "Gbyte" else 1)
        summ["ffn_dram_bytes_per_block"] = rd + wr
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    dst = os.path.join(ROOT, "profiles", f"ncu_{cfg}_{tag}.json")
    with open(dst, "w") as f:
        json.dump(summ, f, indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
