"""Summarise ncu output brought back in gpurun_out/ into a committed text file.

    python tools/ncu_summary.py launches <launches.csv>          # per-kernel share
    python tools/ncu_summary.py report <file.ncu-rep> [regex]    # key metrics of a --set full capture
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_read.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sectors_srcunit_tex_op_read.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]

_US = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * _US.get(d["Metric Unit"], 1.0)
        name = re.sub(r"^.*::", "", d["Kernel Name"].split("(")[0])
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    out = [f"{'kernel':40s} {'launches':>8s} {'total us':>12s} {'mean us':>10s} {'share':>7s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{k:40s} {cnt[k]:8d} {v:12.1f} {v / cnt[k]:10.1f} {100 * v / s:6.1f}%")
    return "\n".join(out)


def report(path, regex=None):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?")
        if regex and not re.search(regex, name):
            continue
        out.append(f"kernel: {name[:120]}")
        for k in KEYS:
            if k in d:
                out.append(f"  {k:70s} {d[k]:>16s} {units[hdr.index(k)]}")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        print(report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None))
