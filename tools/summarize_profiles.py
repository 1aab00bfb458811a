"""Summarise ncu outputs into profiles/ (tracked).

  launch list (gpu__time_duration per launch) -> share of step time per kernel
  --set full report                           -> per-launch duration, DRAM bytes,
                                                 throughput, occupancy
"""
import collections
import csv
import io
import subprocess
import sys


def launch_share(path, marker="k_apply", last=None):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    idx = [i for i, r in enumerate(rows) if marker in r["Kernel Name"]]
    seg = rows[idx[-(last + 1)] + 1: idx[-1] + 1] if last else rows
    tot, cnt = collections.Counter(), collections.Counter()
    for r in seg:
        k = r["Kernel Name"].split("(")[0][:110]
        tot[k] += float(r["Metric Value"])
        cnt[k] += 1
    T = sum(tot.values())
    out = [f"# {len(seg)} launches, {T/1e3:.1f} us serialized (ncu, cold cache: compare SHARES)",
           "share%   total_us   n   kernel"]
    ours = 0.0
    for k, v in tot.most_common():
        mine = k.startswith(("k_apply", "void k_apply", "k_snapshot", "void k_average", "k_accum"))
        if mine:
            ours += v
        out.append(f"{100*v/T:6.2f} {v/1e3:10.1f} {cnt[k]:5d}  {'[ours] ' if mine else ''}{k}")
    out.insert(1, f"# our kernels (K1-K4): {100*ours/T:.2f}% of the serialized step time")
    return "\n".join(out)


def kernel_table(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    want = ["Kernel Name", "launch__grid_size", "launch__registers_per_thread", "gpu__time_duration.sum",
            "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active"]
    ix = [hdr.index(w) for w in want]
    out = ["kernel | grid | regs | us | dram_read_MB | dram_write_MB | dram_%peak | warps_active_%"]
    for r in rows[2:]:
        out.append(" | ".join([r[ix[0]].split("(")[0]] + [r[i] for i in ix[1:]]))
    return "\n".join(out)


def traffic_json(rep):
    """Per-launch duration and DRAM bytes (read + write) -> the JSON bench.py
    reads for roofline.traffic."""
    import json

    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {w: hdr.index(w) for w in ("Kernel Name", "launch__grid_size", "gpu__time_duration.sum",
                                      "dram__bytes_read.sum", "dram__bytes_write.sum")}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tscale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
    out = []
    for r in rows[2:]:
        by = sum(float(r[col[k]]) * scale[units[col[k]]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        us = float(r[col["gpu__time_duration.sum"]]) * tscale[units[col["gpu__time_duration.sum"]]]
        out.append({"kernel": r[col["Kernel Name"]].split("(")[0], "grid": int(r[col["launch__grid_size"]]),
                    "us": us, "dram_bytes": by})
    return json.dumps({"source": "ncu --set full, tools/profile_kernels.py (L2 flushed before each launch)",
                       "launches": out}, indent=1)


if __name__ == "__main__":
    kind, src = sys.argv[1], sys.argv[2]
    if kind == "launches":
        print(launch_share(src, last=int(sys.argv[3]) if len(sys.argv) > 3 else None))
    elif kind == "traffic":
        print(traffic_json(src))
    else:
        print(kernel_table(src))
