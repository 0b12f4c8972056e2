"""DRAM traffic of the bench step's GEMMs from an ncu launch list (build container).

The GPU side runs (scripts/round_measure.sh):
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none -k regex:w4a8_gemm --csv --log-file gpurun_out/traffic.csv \
        python scripts/quick_bench.py --profile --ms 1,2,4,8,16,32,64,128,256,512,1024
quick_bench --profile launches every (shape, M) point 4 times (2 cold replicas x 2) in
shape-major, M-minor order; ncu flushes the caches before each launch, so each
launch reads its weights from HBM like the bench's rotated cold replicas.

usage: python scripts/traffic_summary.py gpurun_out/traffic.csv > profiles/r01_traffic.json
"""
import csv
import io
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench as B  # noqa: E402

PER_POINT = 4


def main(path):
    text = open(path).read()
    text = text[text.index('"ID"'):]
    launches = defaultdict(dict)
    names = {}
    for r in csv.DictReader(io.StringIO(text)):
        i = int(r["ID"])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1,
                 "msecond": 1e3}.get(unit, 1)
        launches[i][r["Metric Name"]] = v * scale
        names[i] = r["Kernel Name"]
    ids = sorted(launches)
    pts = [(k, n, m) for (k, n) in B.SHAPES_C2 for m in B.MS_C2]
    if len(ids) != PER_POINT * len(pts):
        raise SystemExit(f"expected {PER_POINT * len(pts)} GEMM launches, found {len(ids)}")
    out, tot_dram, tot_alg = [], 0.0, 0.0
    for j, (k, n, m) in enumerate(pts):
        ls = [launches[i] for i in ids[PER_POINT * j: PER_POINT * (j + 1)]]
        dram = sum(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in ls) / len(ls)
        us = sum(x["gpu__time_duration.sum"] for x in ls) / len(ls)
        alg = B.alg_bytes(m, k, n, "per-group")
        tot_dram += dram
        tot_alg += alg
        out.append(dict(shape=f"{k}x{n}", M=m, kernel=names[ids[PER_POINT * j]].split("(")[0],
                        dram_bytes=round(dram), alg_bytes=round(alg), ratio=round(dram / alg, 3),
                        ncu_us=round(us, 3)))
    print(json.dumps(dict(source=os.path.basename(path), note="ncu dram__bytes_read.sum + dram__bytes_write.sum "
                          "per GEMM launch (mean of 4 cold launches per point); step = the bench's 33 GEMMs",
                          step_dram_bytes=round(tot_dram), step_alg_bytes=round(tot_alg),
                          step_ratio=round(tot_dram / tot_alg, 3), points=out), indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
