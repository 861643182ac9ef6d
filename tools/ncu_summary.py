"""Summarise ncu output into profiles/ (tracked):

    python tools/ncu_summary.py <gpurun_out/tag> <round-tag> [config]

Reads <dir>/launches.csv (the `--metrics gpu__time_duration.sum --clock-control none` launch
list of a bench run) and every <dir>/prof_*.ncu-rep (`--set full` captures), and writes
profiles/<round-tag>_launches.md (per-kernel count / mean / share of our kernels' time),
profiles/<round-tag>_<kernel>.md (selected metrics) and profiles/ncu_traffic_<config>.json
(DRAM bytes per attention launch, read by bench.py for roofline.traffic)."""
import collections
import csv
import glob
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OURS = ("tree_attn", "attn_combine", "tree_accept", "mss_accept", "accept_kernel", "kv_compact", "tree_mask", "kv_pack", "lm_head",
        "greedy_walk", "tree_select")

METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "smsp__sass_inst_executed_op_tmem_ldt.sum", "smsp__sass_inst_executed_op_tmem_stt.sum",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers", "launch__cluster_dim_x",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__cycles_active.avg",
]


def short(name):
    m = re.search(r"(tree_attn_kernel|mss_accept_kernel|attn_combine\w*|tree_accept\w*|accept_kernel\w*|kv_compact\w*|tree_mask\w*|"
                  r"kv_pack\w*)", name)
    return m.group(1) if m else name[:60]


def launches(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"]) / (1e3 if r["Metric Unit"] == "ns" else 1.0)))
    agg = collections.OrderedDict()
    for n, us in rows:
        k = short(n)
        agg.setdefault(k, []).append(us)
    return agg


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = [l for l in out.splitlines() if l.startswith('"')]
    rd = list(csv.reader(lines))
    hdr, units, rows = rd[0], rd[1], rd[2:]
    res = []
    for v in rows:
        d = {"kernel": short(v[hdr.index("Kernel Name")])}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = (v[i], units[i])
        res.append(d)
    return res


def main():
    src, tag = sys.argv[1], sys.argv[2]
    cfg = sys.argv[3] if len(sys.argv) > 3 else "c2"
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    lp = os.path.join(src, "launches.csv")
    if os.path.exists(lp):
        agg = launches(lp)
        ours = {k: v for k, v in agg.items() if any(o in k for o in OURS)}
        tot = sum(sum(v) for v in ours.values())
        with open(os.path.join(prof, f"{tag}_launches.md"), "w") as f:
            f.write(f"# ncu launch list ({cfg}; `--metrics gpu__time_duration.sum --clock-control none`)\n\n")
            f.write("Cold-cache, serialised per-launch times; compare SHARES with bench.py's live timing.\n\n")
            f.write("| kernel | launches | mean us | total us | share of our kernels |\n|---|---|---|---|---|\n")
            for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
                f.write(f"| {k} | {len(v)} | {sum(v) / len(v):.2f} | {sum(v):.1f} | {sum(v) / tot:.3f} |\n")
            other = {k: v for k, v in agg.items() if k not in ours}
            if other:
                f.write("\nOther (torch setup / input generation, outside the timed region): " +
                        ", ".join(f"{k[:40]} x{len(v)}" for k, v in other.items()) + "\n")
        print(open(os.path.join(prof, f"{tag}_launches.md")).read())
    for rep in sorted(glob.glob(os.path.join(src, "prof_*.ncu-rep"))):
        name = os.path.basename(rep)[5:-8]
        res = raw_metrics(rep)
        with open(os.path.join(prof, f"{tag}_ncu_{name}.md"), "w") as f:
            f.write(f"# ncu --set full: {name} ({cfg}), `{os.path.basename(rep)}`\n\n")
            for d in res:
                f.write(f"## {d['kernel']}\n\n| metric | value | unit |\n|---|---|---|\n")
                for m in METRICS:
                    if m in d:
                        f.write(f"| {m} | {d[m][0]} | {d[m][1]} |\n")
                f.write("\n")
        print(open(os.path.join(prof, f"{tag}_ncu_{name}.md")).read())
        if name.startswith("attn"):
            d = res[0]

            def mb(m):
                v, u = d[m]
                v = float(v.replace(",", ""))
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
            traffic = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
            rcfg = name.split("_", 1)[1] if "_" in name else cfg   # prof_attn_<config>.ncu-rep
            json.dump({"dram_bytes_per_launch": int(traffic), "source": f"profiles/{tag}_ncu_{name}.md",
                       "kernel": d["kernel"]}, open(os.path.join(prof, f"ncu_traffic_{rcfg}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
