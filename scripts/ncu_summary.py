"""Summarise ncu captures for profiles/ (run in the build container).

usage: python scripts/ncu_summary.py <report.ncu-rep> ...        -> key metrics
       python scripts/ncu_summary.py --launches <launches.csv>     -> per-kernel time shares
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__cycles_elapsed.avg.per_second",
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"== {path}")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"kernel: {name}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:70s} {r[i]:>16s} {units[i]}")
        # tensor-pipe metrics differ across ncu versions: print any present
        for i, h in enumerate(hdr):
            if "pipe_tensor" in h and h not in KEYS and r[i] not in ("", "0"):
                print(f"  {h:70s} {r[i]:>16s} {units[i]}")


def launches(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        name = r[ik].split("(")[0][:90]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    print(f"== {path}: {sum(cnt.values())} launches, total {T / 1e3:.1f} us (ncu serialised, cold)")
    for name in sorted(tot, key=lambda n: -tot[n]):
        print(f"  {tot[name] / T * 100:6.2f}%  {cnt[name]:6d} x  avg {tot[name] / cnt[name] / 1e3:9.3f} us  {name}")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        for p in sys.argv[2:]:
            launches(p)
    else:
        for p in sys.argv[1:]:
            report(p)
