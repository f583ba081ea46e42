"""Parse an ncu CSV (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum)
of a bench.py run and write profiles/traffic_<workload>_p<N>.json with the DRAM bytes per GEMM
launch (the bench's roofline `traffic`), plus the per-kernel launch list summary.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/ncu_c2.csv \
        python bench.py --steps 2 --warmup 3 --eager --no-e2e --no-cpu-baseline
    python tools/ncu_traffic.py gpurun_out/ncu_c2.csv c2 1
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    path, workload, world = sys.argv[1], sys.argv[2], int(sys.argv[3])
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    iid, ik, im, iv, iu = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value",
                                                  "Metric Unit"))
    per = {}
    for r in rows[1:]:
        d = per.setdefault(r[iid], {"kernel": r[ik]})
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(r[iu], 1)
        d[r[im]] = float(r[iv].replace(",", "")) * scale
    gemms = [d for d in per.values() if "gemm_tc" in d["kernel"]]
    if not gemms:
        raise SystemExit("no GEMM launches in the capture")
    # skip warm-up launches: keep the last steps' worth (6 GEMMs per step for two layers)
    gemms = gemms[-12:]
    by = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in gemms)
    t = sum(d.get("gpu__time_duration.sum", 0) for d in gemms)
    allk = list(per.values())[-(len(gemms) * 2 + 8):]
    out = {"workload": workload, "n_gpus": world, "gemm_launches": len(gemms),
           "dram_bytes_per_gemm_launch": int(by / len(gemms)),
           "gemm_ns_per_launch_cold": int(t / len(gemms)),
           "source": os.path.basename(path) + " (ncu --clock-control none, cold-cache replay)",
           "launches": [{"kernel": d["kernel"][:90], "ns": int(d.get("gpu__time_duration.sum", 0)),
                         "dram_bytes": int(d.get("dram__bytes_read.sum", 0) +
                                           d.get("dram__bytes_write.sum", 0))} for d in allk]}
    dst = os.path.join(ROOT, "profiles", f"traffic_{workload}_p{world}.json")
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(dst, out["dram_bytes_per_gemm_launch"], out["gemm_ns_per_launch_cold"])


if __name__ == "__main__":
    main()
