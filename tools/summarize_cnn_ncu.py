"""gpurun_out/cnn_full_raw.csv.gz (tools/ncu_cnn.sh) -> profiles/r2_cnn_kernels_ncu.txt"""
import collections
import csv
import gzip
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/cnn_full_raw.csv.gz"
dst = sys.argv[2] if len(sys.argv) > 2 else "profiles/r2_cnn_kernels_ncu.txt"
rows = list(csv.reader(gzip.open(src, "rt")))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def g(r, m):
    try:
        return float(r[ix[m]].replace(",", "")) * scale.get(units[ix[m]], 1)
    except (KeyError, ValueError):
        return float("nan")


agg = collections.OrderedDict()
for r in data:
    name = r[ix["Kernel Name"]].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").split("(")[0]
    agg.setdefault(name[5:] if name.startswith("void ") else name, []).append(r)
lines = ["# fp32 CNN kernels (csrc/conv_f32.cu), ncu --set full --clock-control none, one fwd+bwd of each",
         "# ResNet-20 basic-block shape at B = 128 (tools/profile_cnn_kernels.py via tools/ncu_cnn.sh; cold caches,",
         "# serialised; forward convolutions carry their fused BatchNorm statistics and 8-CTA clusters; FMAs as FFMA2).",
         "# Columns: launches, mean duration, FMA-pipe and issue activity (% of active cycles), DRAM bytes per launch",
         "# (read + write) and the rate they imply, achieved warps per SM, grid x block.",
         f"{'kernel':50s} {'n':>2s} {'us':>7s} {'fma%':>6s} {'issue%':>6s} {'dram MB':>8s} {'GB/s':>6s} {'warps':>6s}  grid x block"]
for k, v in agg.items():
    def m(key):
        return sum(g(r, key) for r in v) / len(v)
    dram = m("dram__bytes_read.sum") + m("dram__bytes_write.sum")
    t = m("gpu__time_duration.sum") / 1e3 if units[ix["gpu__time_duration.sum"]] == "ns" else m("gpu__time_duration.sum")
    lines.append(f"{k[:50]:50s} {len(v):2d} {t:7.2f} {m('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):6.1f} "
                 f"{m('smsp__issue_active.avg.pct_of_peak_sustained_active'):6.1f} {dram / 1e6:8.2f} "
                 f"{dram / (t * 1e-6) / 1e9:6.0f} {m('sm__warps_active.avg.per_cycle_active'):6.1f}  "
                 f"{v[0][ix['Grid Size']]} x {v[0][ix['Block Size']]}")
open(dst, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[5:]))
