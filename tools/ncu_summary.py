"""Summarise an `ncu --set full` report: per captured kernel the duration,
DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum), DRAM / SM
throughput and issue statistics.

usage: python tools/ncu_summary.py REPORT.ncu-rep [--json]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
           "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size"]


def main():
    path = sys.argv[1]
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")][:60]}
        for m in METRICS:
            if m in hdr:
                k = hdr.index(m)
                v = r[k].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                d[m] = v
                d[m + ".unit"] = units[k]
        res.append(d)
    if "--json" in sys.argv:
        print(json.dumps(res, indent=1))
        return
    for d in res:
        t = d.get("gpu__time_duration.sum")
        tu = d.get("gpu__time_duration.sum.unit")
        rb = d.get("dram__bytes_read.sum", 0)
        wb = d.get("dram__bytes_write.sum", 0)
        ub = d.get("dram__bytes_read.sum.unit")
        print(f"{d['kernel']:60s} t={t} {tu}  dram_rd={rb} {ub} dram_wr={wb} {d.get('dram__bytes_write.sum.unit')}  "
              f"dram%={d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')}  "
              f"sm%={d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed')}  "
              f"dmma_inst%={d.get('sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active')}  "
              f"tensor_active%={d.get('TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed')}  "
              f"regs={d.get('launch__registers_per_thread')}")


if __name__ == "__main__":
    main()
