"""Summarise an ncu --set full report of tools/ncu_shapes.py (one capture per GEMM shape) as a
markdown table: duration, SM clock, achieved TFLOP/s and its fraction of the clock-scaled dense
bf16 peak, tensor-pipe utilisation, DRAM bytes against the algorithmic operand + output bytes.

    python tools/ncu_summary.py gpurun_out/ncu_shapes.ncu-rep gpurun_out/ncu_shapes.log > profiles/...md

Algorithmic bytes per launch: each operand read once and the output written once, bf16:
2 (M K + K N + M N). Peak at the measured SM clock f: 148 SMs x 8192 dense bf16 flop/clk x f
(the per-clock rate behind the nominal 2.25 PFLOP/s, which it reaches at 1.856 GHz); the
burst column scales MEASURED_PEAKS.json's bf16_tflops from the 1.965 GHz it was measured at.
"tensor %" = sm__mem_tensor_cycles_active (tcgen05 / TMEM datapath busy, % of elapsed).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COLS = {
    "dur": "gpu__time_duration.sum",
    "clk": "sm__cycles_elapsed.avg.per_second",
    "tc": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "rd": "dram__bytes_read.sum",
    "wr": "dram__bytes_write.sum",
    "grid": "launch__grid_size",
    "name": "Kernel Name",
}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, data = r[0], r[1], r[2:]
    idx = {k: hdr.index(v) for k, v in COLS.items() if v in hdr}
    res = []
    for d in data:
        item = {}
        for k, i in idx.items():
            v, u = d[i], units[i]
            if k in ("name",):
                item[k] = v
                continue
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                x = float("nan")
            scale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
                     "msecond": 1e-3, "s": 1.0, "second": 1.0,
                     "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                     "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1,
                     "cycle/nsecond": 1e9, "cycle/usecond": 1e6}.get(u, 1)
            item[k] = x * scale
        res.append(item)
    return res


def shapes(log):
    out = []
    for line in open(log):
        m = re.match(r"(\w+): M=(\d+) K=(\d+) N=(\d+) ta=(\d) tb=(\d)", line)
        if m:
            out.append((m.group(1), *map(int, m.groups()[1:])))
    return out


def main():
    rep, log = sys.argv[1], sys.argv[2]
    R = [r for r in rows(rep) if "gemm" in r.get("name", "")]
    S = shapes(log)
    try:
        burst = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    except (OSError, KeyError, ValueError):
        burst = None
    print("| shape | m x k x n (op) | kernel | grid | us | SM GHz | TFLOP/s | frac peak@clk | "
          "frac burst@clk | tensor % | DRAM MB | alg MB | DRAM/alg |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    reps = len(R) // max(len(S), 1)
    for i, (name, M, K, N, ta, tb) in enumerate(S):
        r = R[i * reps + reps - 1]  # last launch of the shape
        fl = 2.0 * M * N * K
        t = r["dur"]
        tf = fl / t / 1e12
        ghz = r["clk"] / 1e9
        nom = 148 * 8192 * ghz * 1e9 / 1e12
        alg = 2.0 * (M * K + K * N + M * N)
        dram = r["rd"] + r["wr"]
        op = ("T" if ta else "N") + ("T" if tb else "N")
        kern = re.sub(r"\(.*", "", r["name"]).replace("(anonymous namespace)::", "")
        frac_b = f"{tf / (burst * ghz / 1.965):.3f}" if burst else "-"
        print(f"| {name} | {M}x{K}x{N} ({op}) | {kern} | {int(r['grid'])} | {t * 1e6:.1f} | {ghz:.2f} | "
              f"{tf:.0f} | {tf / nom:.3f} | {frac_b} | {r['tc']:.1f} | {dram / 1e6:.1f} | "
              f"{alg / 1e6:.1f} | {dram / alg:.2f} |")


if __name__ == "__main__":
    main()
