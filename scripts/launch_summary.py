"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel:
python scripts/launch_summary.py gpurun_out/launches.csv > profiles/<round>_launches_summary.csv"""

import csv
import sys
from collections import defaultdict


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    head = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[head]
    k, m, v, u = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[head + 1:]:
        if len(r) <= v or r[m] != "gpu__time_duration.sum":
            continue
        val = float(r[v].replace(",", ""))
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[u], 1e-6)
        name = r[k].split("(")[0]
        tot[name] += val * scale
        cnt[name] += 1
    total = sum(tot.values())
    print(f"# total device time {total:.1f} ms over {sum(cnt.values())} launches")
    print("kernel,launches,total_ms,share")
    for name, t in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{name},{cnt[name]},{t:.3f},{t / total:.4f}")


if __name__ == "__main__":
    main(sys.argv[1])
