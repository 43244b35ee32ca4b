"""Per-source-line warp-stall attribution from an ncu SourceCounters report.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_stalls.py src.csv [--top 40]

SASS rows follow the CUDA line they map to; their per-reason stall samples
are summed under that line (inlined code lands on the callee's line).
"""
import argparse
import collections
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=40)
    args = ap.parse_args()
    rows = list(csv.reader(open(args.csv)))
    hdr = None
    cur_file, cur_line, cur_src = "?", "?", ""
    agg = collections.defaultdict(collections.Counter)
    src = {}
    total = collections.Counter()
    for r in rows:
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            reasons = [h for h in r if h.startswith("stall_") and "(Not" not in h]
            continue
        if hdr is None:
            continue
        if r[0]:  # a CUDA source line
            cur_line, cur_src = r[0], r[1]
            continue
        if len(r) < len(hdr):
            continue
        key = (cur_file, cur_line)
        src[key] = cur_src.strip()
        for h in reasons:
            try:
                v = float(r[hdr[h]] or 0)
            except ValueError:
                continue
            agg[key][h] += v
            total[h] += v
    s = sum(total.values()) or 1.0
    print("total samples", int(s))
    print("  ".join(f"{h[6:]}={100 * v / s:.1f}%" for h, v in total.most_common(10)))
    lines = sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))
    for key, c in lines[: args.top]:
        t = sum(c.values())
        top = ", ".join(f"{h[6:]}:{int(v)}" for h, v in c.most_common(3) if v)
        print(f"{100 * t / s:5.1f}% {key[0]}:{key[1]:<5} {src[key][:58]:58s} {top}")


if __name__ == "__main__":
    main()
