"""Complete kernel launch list of the bench's timed region (ResNet-20
LPP-SGD, U=4, native loop) from a CUPTI activity trace (torch.profiler):
every kernel of K steps, concurrent (not serialised like ncu), with its
duration — the full-coverage complement of the ncu launch list, which
cannot finish the whole bench under replay in reasonable time."""
import collections, csv, json, sys
from pathlib import Path
import torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
from paper_2203_06638_b200.engine import Trainer
from paper_2203_06638_b200.objectives import ResNetObjective

torch.backends.cudnn.benchmark = True
torch.backends.cudnn.allow_tf32 = False        # the bench's fp32 headline
torch.backends.cuda.matmul.allow_tf32 = False
K, W, U = 20, 5, 4
args = [a for a in sys.argv[1:] if not a.startswith("--")]
out_dir = Path(args[0] if args else "gpurun_out")
obj = ResNetObjective("resnet20", n_samples=50_000, seed=0, data="device",
                      autocast=None if "--bf16" not in sys.argv else "bf16")
cfg = bench.build_cfg(obj, (K + W) * U)
tr = Trainer(cfg)
tr.run(W * U, evaluate=False)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    res = tr.run(K * U, evaluate=False)
    torch.cuda.synchronize()
rows = []
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA and ev.name and not ev.name.startswith("Memcpy") \
            and not ev.name.startswith("Memset"):
        rows.append((ev.name, ev.time_range.start, ev.time_range.end - ev.time_range.start))
rows.sort(key=lambda r: r[1])
with open(out_dir / "trace_launches.csv", "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["kernel", "start_us", "dur_us"])
    t0 = rows[0][1] if rows else 0
    for n, s, d in rows:
        w.writerow([n, s - t0, d])
tot, cnt = collections.Counter(), collections.Counter()
for n, _, d in rows:
    k = n.replace("(anonymous namespace)::", "").split("(")[0][:110]
    tot[k] += d
    cnt[k] += 1
T = sum(tot.values())
OURS = ("k_apply", "k_snapshot", "k_average", "k_accum", "k_gather", "k_publish", "k_set_i64",
        "k_classify", "k_sample", "k_conv3x3", "k_wgrad3x3", "k_wgrad_reduce", "k_conv1x1s2",
        "k_fma_probe", "k_bn_apply", "k_bn_bwd", "k_stem", "k_w_tapmajor")


def is_ours(k):
    base = k[5:] if k.startswith("void ") else k
    base = base.replace("(anonymous namespace)::", "")
    return base.startswith(OURS)


mine = sum(v for k, v in tot.items() if is_ours(k))
span = (rows[-1][1] + rows[-1][2] - rows[0][1]) if rows else 0
lines = [f"# {len(rows)} kernels in the timed region of {K * U + U} minibatches "
         f"(ResNet-20 LPP-SGD U=4 B=128, {'bf16' if '--bf16' in sys.argv else 'fp32'} convolutions, "
         f"native loop); summed kernel time {T / 1e3:.1f} ms "
         f"over a {span / 1e3:.1f} ms span (4 streams overlap)",
         f"# our kernels (K1-K5, in-graph sampler, fp32 convolutions, fused BatchNorm): {100 * mine / T:.2f}% of "
         f"summed kernel time",
         "share%   total_us   n   kernel"]
for k, v in tot.most_common():
    tag = "[ours] " if is_ours(k) else ""
    lines.append(f"{100 * v / T:6.2f} {v:10.1f} {cnt[k]:5d}  {tag}{k}")
(out_dir / "trace_share.txt").write_text("\n".join(lines) + "\n")
print("\n".join(lines[:30]))
tr.close()
