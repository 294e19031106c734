#!/usr/bin/env python3
"""Markdown result tables from bench lines (README): one row per config.

  python tools/results_tables.py [profiles/r02]
"""
import json
import os
import sys

NAMES = {"C1": "C1", "C2": "C2", "C3": "C3", "C4": "C4", "C5": "C5", "LAP": "LAP (Tensor 2)",
         "P6W": "P6W (weak-scaling shape, p = 1)", "P6S": "P6S (strong-scaling tensor, 125 GB)"}


def line(path):
    with open(path) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def fmt_us(v):
    return f"{v / 1000:.1f} ms" if v > 10000 else f"{v:.0f} µs"


def main():
    d = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02"
    print("| cfg | sweeps/s | ms per 20-sweep run | phase mix dt / build / pp | DT sweep | PP build | "
          "PP middle | dominant kernel (roofline) | oracle |")
    print("|---|---|---|---|---|---|---|---|---|")
    for c, name in NAMES.items():
        p = os.path.join(d, f"bench_{c}.json")
        if not os.path.exists(p):
            continue
        b = line(p)
        ph = b.get("phase_us", {})
        mix = " / ".join(str(int(ph.get(k, {}).get("count_per_step", 0))) for k in ("dt", "pp-build", "pp-approx"))
        cell = [fmt_us(ph[k]["median"]) if k in ph else "—" for k in ("dt", "pp-build", "pp-approx")]
        r = b["roofline"]
        if c == "C1":
            roof = "latency-bound (solve chain)"
        elif r["unit"] == "TFLOP/s":
            roof = f"TTM {r['achieved']:.1f} TF/s = {r['frac']:.3f} of DMMA peak"
        else:
            roof = f"TTM {r['achieved'] / 1000:.2f} TB/s = {r['frac']:.3f} of HBM"
        cpu = b.get("cpu_baseline") or {}
        oracle = f"{cpu['value']:.4g} sweeps/s" if cpu else "—"
        print(f"| {name} | {b['value']:.5g} | {b['ms_per_step']:.4g} | {mix} | {cell[0]} | {cell[1]} | "
              f"{cell[2]} | {roof} | {oracle} |")


if __name__ == "__main__":
    main()
