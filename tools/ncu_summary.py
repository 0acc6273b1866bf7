"""Summarize ncu output for profiles/ (committed evidence).

  python tools/ncu_summary.py launches <launches.csv>            -> per-kernel time shares
  python tools/ncu_summary.py report <prof.ncu-rep> [--json out]  -> key metrics + stall mix per kernel
"""
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("smsp__cycles_active.avg", "smsp_active_cycles_avg"),
    ("smsp__cycles_active.max", "smsp_active_cycles_max"),
    ("sm__cycles_elapsed.avg", "sm_elapsed_cycles"),
    ("smsp__inst_executed.sum", "warp_instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads_per_instr"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_throughput_%"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1_lsu_wavefronts_%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1_throughput_%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_throughput_%"),
    ("sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "fp64_pipe_%"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in data:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ms": 1e3, "us": 1.0, "ns": 1e-3, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3}.get(r[ui], 1.0)
        name = r[ki].replace("(bool)", "").replace("(int)", "")
        agg[name.split("(")[0].replace("void ", "").replace("gmaco::", "").strip()].append(v)
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | mean us | total us | share |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.2f} | {sum(v):.1f} | {sum(v) / tot:.3f} |")
    return "\n".join(out)


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for row in rows[2:]:
        k = {"kernel": row[hdr.index("Kernel Name")]}
        for m, name in METRICS:
            hits = [j for j, x in enumerate(hdr) if x == m] + [j for j, x in enumerate(hdr) if x.endswith("." + m)]
            hits = [j for j in hits if row[j] not in ("", "no data")]
            if hits:
                i = hits[0]
                k[name] = f"{row[i]} {units[i]}".strip()
        kernels.append(k)
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    secs = [i for i, r in enumerate(srows) if r and r[0] == "Kernel Name"]
    for si, i0 in enumerate(secs):
        end = secs[si + 1] if si + 1 < len(secs) else len(srows)
        name = srows[i0][1]
        h = srows[i0 + 1]
        data = [r for r in srows[i0 + 2:end] if len(r) == len(h)]
        reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
        tot = {x: sum(float(r[h.index(x)] or 0) for r in data) for x in reasons}
        s = sum(tot.values()) or 1.0
        short = name.replace("(bool)", "").replace("(int)", "").split("(")[0].replace("void ", "").replace("gmaco::", "")
        for k in kernels:
            kk = k["kernel"].replace("(bool)", "").replace("(int)", "").split("(")[0].replace("void ", "")
            if kk.replace(" ", "") == short.replace(" ", "") and "stalls_%" not in k:
                k["stalls_%"] = {r[6:]: round(v / s * 100, 1)
                                 for r, v in sorted(tot.items(), key=lambda kv: -kv[1])[:6]}
                break
    return kernels


def main():
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        ks = report(sys.argv[2])
        if "--json" in sys.argv:
            json.dump(ks, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
        for k in ks:
            print(f"### `{k['kernel']}`")
            for key, val in k.items():
                if key != "kernel":
                    print(f"- {key}: {val}")
            print()


if __name__ == "__main__":
    main()
