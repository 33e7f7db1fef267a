"""Summarise ncu outputs from gpurun_out/ into profiles/ (tracked).

  python scripts/summarize_ncu.py <tag>
reads gpurun_out/launches_<tag>.csv (gpu__time_duration.sum launch list) and
gpurun_out/decode_attn_<tag>.ncu-rep (--set full capture), writes
profiles/<tag>_launches.txt, profiles/<tag>_decode_attn_ncu.txt and
profiles/decode_attn_traffic.json (read by bench.py for roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)

# ---- launch list (when this tag has one)
path = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
if os.path.exists(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        t = float(r[vi].replace(",", "")) * scale
        c = agg.setdefault(name, [0, 0.0])
        c[0] += 1
        c[1] += t
    STEP = ("decode_attn_v2", "decode_attn_kernel", "decode_merge", "decode_snapshot")
    ROWS = ("prefill_attn", "decode_gqa_tc")
    with open(os.path.join(out_dir, f"{tag}_launches.txt"), "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none of: python bench.py --steps 2 --warmup 1"
                f" --no-cpu-baseline\n# per-launch times are serialised/cold-cache: compare shares, not absolutes\n")
        for title, sel in (("decode-step kernels (the timed region)", lambda k: any(x in k for x in STEP)),
                           ("tensor-core rows beside the headline (prefill attention, GQA decode tile)",
                            lambda k: any(x in k for x in ROWS)),
                           ("setup kernels (prefill offload, synthetic data, verification)",
                            lambda k: not any(x in k for x in STEP + ROWS))):
            part = {k: v for k, v in agg.items() if sel(k)}
            total = sum(v[1] for v in part.values()) or 1.0
            f.write(f"\n## {title}\n{'kernel':50s} {'launches':>9s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}\n")
            for k, (n, t) in sorted(part.items(), key=lambda kv: -kv[1][1]):
                f.write(f"{k[:50]:50s} {n:9d} {t:12.1f} {t / n:10.2f} {100 * t / total:6.2f}%\n")
    print(open(os.path.join(out_dir, f"{tag}_launches.txt")).read())


# ---- full captures of the tensor-core kernels (prefill attention, GQA decode tile)
TC_KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
           "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
           "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
           "smsp__warp_issue_stalled_wait_per_warp_active.pct",
           "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "sm__issue_active.avg.pct_of_peak_sustained_elapsed"]
for cap in ("prefill_attn", "prefill_attn2", "decode_gqa_tc"):
    rep = os.path.join(ROOT, "gpurun_out", f"{cap}_{tag}.ncu-rep")
    if not os.path.exists(rep):
        continue
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, units = rr[0], rr[1]
    lines = [f"# ncu --set full --clock-control none -k regex:{cap} (scripts/*_micro.py), tag {tag}"]
    for r in rr[2:]:
        for k in TC_KEYS + [x for x in h if "tensor" in x and "pct" in x and x not in TC_KEYS][:6]:
            if k in h:
                i = h.index(k)
                lines.append(f"{k:70s} {r[i]} {units[i]}")
        lines.append("")
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    ops = collections.Counter()
    for ln in sass.splitlines():
        for m in ("UTCHMMA", "UTCBAR", "UTMALDG", "UBLKCP", "LDTM", "STTM", "MUFU.EX2"):
            if m in ln:
                ops[m] += 1
        if "HMMA" in ln.replace("UTCHMMA", ""):  # legacy mma.sync path (must stay 0)
            ops["HMMA(legacy)"] += 1
    lines.append("# SASS opcodes present (static count in the source page): " +
                 ", ".join(f"{k}={v}" for k, v in sorted(ops.items())))
    with open(os.path.join(out_dir, f"{tag}_{cap}_ncu.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))

# ---- full capture of the decode kernel
rep = os.path.join(ROOT, "gpurun_out", f"decode_attn_{tag}.ncu-rep")
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, units = rr[0], rr[1]
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
            "launch__shared_mem_per_block_static", "launch__shared_mem_per_block_dynamic",
            "smsp__inst_executed.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
            "smsp__average_warp_latency_issue_stalled_long_scoreboard",
            "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
            "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
            "smsp__warp_issue_stalled_wait_per_warp_active.pct"]
    lines = []
    traffic = []
    for r in rr[2:]:
        for k in keys:
            if k in h:
                i = h.index(k)
                lines.append(f"{k:70s} {r[i]} {units[i]}")
        lines.append("")
        try:
            rd = float(r[h.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(r[h.index("dram__bytes_write.sum")].replace(",", ""))
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[h.index("dram__bytes_read.sum")], 1)
            multw = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[h.index("dram__bytes_write.sum")], 1)
            traffic.append(rd * mult + wr * multw)
        except ValueError:
            pass
    with open(os.path.join(out_dir, f"{tag}_decode_attn_ncu.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none -k regex:decode_attn (bench.py default workload), tag {tag}\n")
        f.write("\n".join(lines))
    if traffic:
        with open(os.path.join(out_dir, "decode_attn_traffic.json"), "w") as f:
            json.dump({"tag": tag, "dram_bytes_per_launch": sum(traffic) / len(traffic),
                       "source": f"profiles/{tag}_decode_attn_ncu.txt (dram__bytes_read.sum + dram__bytes_write.sum)"},
                      f, indent=1)
    print("\n".join(lines[:60]))
