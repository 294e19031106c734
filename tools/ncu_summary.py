#!/usr/bin/env python3
"""Summarise ncu outputs into profiles/: per-kernel launch shares from a
`--metrics gpu__time_duration.sum --csv` launch list, and the key counters of `--set full`
captures (.ncu-rep, read with `ncu -i ... --page raw --csv`).

  python tools/ncu_summary.py launches <launches.csv>           -> markdown table on stdout
  python tools/ncu_summary.py full <a.ncu-rep> [<b.ncu-rep> ...] -> JSON list on stdout
  python tools/ncu_summary.py traffic <a.ncu-rep> <class> [...]  -> {"class": bytes/launch}
"""
import collections
import csv
import io
import json
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smsp__inst_executed.sum",
]


def short(name):
    n = name.split("(")[0]
    n = n.replace("void ", "").replace("(anonymous namespace)::", "").replace("cppp::", "")
    return n.split("::")[-1].strip()


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        a = agg[short(r[ki])]
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {k} | {n} | {t:.1f} | {t / n:.2f} | {t / tot:.3f} |")
    return "\n".join(out)


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for m in FULL_METRICS:
            if m in h:
                d[m] = f"{r[h.index(m)]} {units[h.index(m)]}".strip()
        res.append(d)
    return res


def num(s):
    v, u = s.split(" ", 1) if " " in s else (s, "")
    v = float(v.replace(",", ""))
    return v * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}.get(u.strip(), 1.0)


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        print(launches(sys.argv[2]))
    elif mode == "full":
        out = []
        for rep in sys.argv[2:]:
            out += raw(rep)
        print(json.dumps(out, indent=1))
    elif mode == "traffic":
        rep, cls = sys.argv[2], sys.argv[3]
        ks = raw(rep)
        b = [num(k["dram__bytes_read.sum"]) + num(k["dram__bytes_write.sum"]) for k in ks]
        print(json.dumps({cls: sum(b) / len(b)}))
