#!/usr/bin/env python
"""Summarise ncu output brought back in gpurun_out/ into text files kept under profiles/.

    python profiles/summarize.py launches <launches.csv> > profiles/<tag>_launch_summary.txt
    python profiles/summarize.py full <prof.ncu-rep>     > profiles/<tag>_<kernel>_ncu_summary.txt

`launches`: per-kernel count, total/mean device time and share of the profiled
launches (cold-cache, serialised: compare SHARES with bench.py, not absolutes).
`full`: the metrics the roofline needs (duration, DRAM bytes, tensor-pipe activity,
occupancy, registers) plus the top SASS stall sites.
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def launches(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)  # -> us
        a = agg.setdefault(name, [0, 0.0, r["Grid Size"], r["Block Size"]])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"# {path}: {sum(a[0] for a in agg.values())} launches, {tot / 1e3:.3f} ms total (ncu, serialised)")
    print(f"{'kernel':24s} {'n':>4s} {'total_us':>12s} {'mean_us':>12s} {'share':>7s}  grid / block")
    for k, (n, t, g, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:24s} {n:4d} {t:12.1f} {t / n:12.1f} {t / tot:7.3f}  {g} / {b}")


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        print(f"# kernel: {vals[hdr.index('Kernel Name')] if 'Kernel Name' in hdr else '?'}")
        for k in KEYS:
            for i, h in enumerate(hdr):
                if h == k:
                    print(f"{k:90s} {vals[i]:>16s} {units[i]}")
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    # one section per kernel: a "Kernel Name" row, a header row, then instruction rows
    sections, cur = [], None
    for r in srows:
        if r and r[0] == "Kernel Name":
            cur = [r[1] if len(r) > 1 else "?", None, []]
            sections.append(cur)
        elif cur is not None and cur[1] is None:
            cur[1] = r
        elif cur is not None:
            cur[2].append(r)
    for name, h, data in sections:
        if not h or "Warp Stall Sampling (All Samples)" not in h:
            continue
        i_s = h.index("Warp Stall Sampling (All Samples)")
        i_src = h.index("Source")
        stall = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
        num = lambda v: float(v) if v not in ("", None) else 0.0
        tot = sum(num(r[i_s]) for r in data) or 1.0
        print(f"\n# {name}: top SASS stall sites (share of warp-stall samples)")
        for r in sorted(data, key=lambda r: -num(r[i_s]))[:15]:
            top = sorted(((num(r[i]), h[i]) for i in stall), reverse=True)[:2]
            print(f"{num(r[i_s]) / tot * 100:5.1f}%  {r[i_src][:58]:58s} {', '.join(f'{n}={int(v)}' for v, n in top)}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
