"""Summarise ncu captures into the markdown tables kept under profiles/.

  python profiles/summarize.py full  <report.ncu-rep>   # --set full capture
  python profiles/summarize.py launches <launches.csv>  # gpu__time_duration list

Only reads existing reports (ncu -i); never profiles anything itself.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

FULL = [
    ("time_us", "gpu__time_duration.sum", 1e-3),
    ("dram_rd_MB", "dram__bytes_read.sum", 1.0),
    ("dram_wr_MB", "dram__bytes_write.sum", 1.0),
    ("sm_thru_%", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("dram_%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("fp64_pipe_%", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1.0),
    ("warps_active_%", "sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    ("ipc", "sm__inst_executed.avg.per_cycle_active", 1.0),
    ("regs", "launch__registers_per_thread", 1.0),
]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def to_mb(v, unit):
    x = float(v)
    return x / 1e6 if unit == "byte" else x / 1e3 if unit == "Kbyte" else x if unit == "Mbyte" \
        else x * 1e3 if unit == "Gbyte" else x


def full(path):
    hdr, units, data = raw(path)
    ix = {h: i for i, h in enumerate(hdr)}
    groups = defaultdict(list)
    for r in data:
        name = r[ix["Kernel Name"]].split("(")[0].split("::")[-1]
        groups[name].append(r)
    print("| kernel | n | " + " | ".join(k for k, _, _ in FULL) + " | top stalls |")
    print("|---" * (len(FULL) + 3) + "|")
    for name, rs in groups.items():
        vals = []
        for key, metric, scale in FULL:
            if metric not in ix:
                vals.append("?")
                continue
            xs = []
            for r in rs:
                v = r[ix[metric]].replace(",", "")
                try:
                    x = to_mb(v, units[ix[metric]]) if "bytes" in metric else float(v)
                except ValueError:
                    continue
                xs.append(x * scale if key == "time_us" and units[ix[metric]] in ("nsecond", "ns")
                          else x)
            u = units[ix[metric]]
            if key == "time_us" and u in ("msecond", "ms"):
                xs = [x * 1e3 for x in xs]
            # "usecond"/"us": already microseconds
            vals.append(f"{sum(xs) / len(xs):.4g}" if xs else "?")
        st = {}
        for h, i in ix.items():
            if h.startswith(STALLS) and not h.endswith("not_issued") and h.endswith(".sum") is False:
                pass
        for h, i in ix.items():
            if h.startswith(STALLS) and "not_issued" not in h:
                try:
                    st[h[len(STALLS):]] = sum(float(r[i] or 0) for r in rs)
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        stalls = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top)
        print(f"| {name} | {len(rs)} | " + " | ".join(vals) + f" | {stalls} |")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0].split("::")[-1]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        us = v / 1e3 if unit in ("nsecond", "ns") else v if unit in ("usecond", "us") else v * 1e3
        tot[name] += us
        cnt[name] += 1
    s = sum(tot.values())
    print("| kernel | launches | total us | share |")
    print("|---|---|---|---|")
    for n, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| {n} | {cnt[n]} | {t:.1f} | {100 * t / s:.1f}% |")
    print(f"| **all** | {sum(cnt.values())} | {s:.1f} | 100% |")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
