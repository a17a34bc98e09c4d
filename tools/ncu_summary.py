"""Summarise ncu reports / launch lists into the numbers profiles/ records.

  python tools/ncu_summary.py rep <file.ncu-rep>       per-kernel key metrics (one line per launch)
  python tools/ncu_summary.py launches <launches.csv>  per-kernel share of device time
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("time_us", "gpu__time_duration.sum"),
    ("dram_rd_MB", "dram__bytes_read.sum"),
    ("dram_wr_MB", "dram__bytes_write.sum"),
    ("tensor_pct", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("tcgen05_bf16_pct", "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed"),
    ("hmma_pct", "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("lts_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("issue_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("warps_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("regs", "launch__registers_per_thread"),
    ("smem_KB", "launch__shared_mem_per_block_dynamic"),
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:60], "grid": r[hdr.index("Grid Size")]}
        for k, m in KEYS:
            if m in hdr:
                d[k] = r[hdr.index(m)]
                d[k + "_unit"] = units[hdr.index(m)]
        res.append(d)
    return res


def launches(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    tot = collections.Counter()
    n = collections.Counter()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v / 1000.0 if unit == "ns" else v * (1000.0 if unit == "ms" else 1.0)
        tot[name] += v
        n[name] += 1
    s = sum(tot.values())
    return [(k, n[k], round(v, 1), round(100 * v / s, 1)) for k, v in tot.most_common()]


if __name__ == "__main__":
    if sys.argv[1] == "rep":
        for d in rep(sys.argv[2]):
            print({k: v for k, v in d.items() if not k.endswith("_unit")})
    else:
        print("kernel, launches, total_us, share_%")
        for row in launches(sys.argv[2]):
            print(row)
