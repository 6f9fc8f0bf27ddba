"""Summarise one kernel of an ncu --set full report into the JSON bench.py
reads for roofline.traffic (profiles/<kernel>_ncu_summary.json):
python scripts/ncu_summary.py REPORT.ncu-rep KERNEL_REGEX NOTE SOURCE > profiles/x.json"""

import csv
import io
import json
import re
import subprocess
import sys


def main(rep, regex, note, source):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        if not re.search(regex, name):
            continue

        def g(key, scale=1.0):
            i = hdr.index(key)
            u = units[i]
            v = float(r[i].replace(",", ""))
            mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "Tbyte": 1e12, "byte": 1.0, "msecond": 1.0,
                    "usecond": 1e-3, "nsecond": 1e-6, "second": 1e3}.get(u, 1.0)
            return v * mult * scale

        rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
        res = {
            "kernel": name, "duration_ms": g("gpu__time_duration.sum"),
            "dram_read": rd, "dram_write": wr, "dram_bytes_per_launch": rd + wr,
            "xu_pipe_pct": g("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
            "tensor_pipe_pct": g("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
            "shared_pipe_pct": g("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": g("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "fma_pipe_pct": g("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": g("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
            "registers_per_thread": g("launch__registers_per_thread"),
            "threads_per_cta": g("launch__block_size"),
            "sm_clock_ghz_under_ncu": g("sm__cycles_elapsed.avg.per_second"),
            "note": note, "source": source,
        }
        print(json.dumps(res, indent=1))
        return
    sys.exit(f"no kernel matching {regex}")


if __name__ == "__main__":
    main(*sys.argv[1:5])
