"""Turn raw ncu outputs into the committed profile summaries.

    python tools/summarize_profiles.py <tag> <ncu-rep of one layer launch> <launch-list csv|-> <cfg> [layer]

Writes profiles/<tag>_ncu_layer200_<cfg>.json (selected metrics of the
`ncu --set full` capture, per launch) and profiles/<tag>_launches_<cfg>_summary.csv
(every kernel's share of GPU time from the `--metrics gpu__time_duration.sum`
launch list) plus the layer kernel's per-launch durations.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
    "launch__block_size", "launch__grid_size", "sm__inst_executed.sum",
]


def main():
    tag, rep, launches, cfg = sys.argv[1:5]
    layer = sys.argv[5] if len(sys.argv) > 5 else "200"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {m: [vals[hdr.index(m)], units[hdr.index(m)]] for m in METRICS if m in hdr}
    stalls = {h.replace("smsp__average_warps_issue_stalled_", "").replace(
        "_per_issue_active.ratio", ""): float(vals[i] or 0)
        for i, h in enumerate(hdr)
        if h.startswith("smsp__average_warps_issue_stalled_") and
        h.endswith("_per_issue_active.ratio")}
    out["stall_per_issued_instruction"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:10])
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_layer{layer}_{cfg}.json"), "w") as f:
        json.dump(out, f, indent=1)
    if launches == "-":
        print(json.dumps({k: out[k] for k in ("gpu__time_duration.sum", "dram__bytes_read.sum",
                                              "dram__bytes_write.sum")}))
        return
    tot, cnt, layer_us = defaultdict(float), defaultdict(int), []
    with open(launches) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit == "ns" else (v if unit == "us" else v * 1e3)
        tot[name] += us
        cnt[name] += 1
        if "layer_kernel" in name:
            layer_us.append(us)
    allt = sum(tot.values())
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches_{cfg}_summary.csv"), "w") as f:
        f.write("kernel,launches,total_ms,share_pct\n")
        for k in sorted(tot, key=lambda k: -tot[k]):
            f.write(f'"{k}",{cnt[k]},{tot[k] / 1e3:.4f},{tot[k] / allt * 100:.2f}\n')
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches_{cfg}_layer_kernel_us.txt"), "w") as f:
        f.write("# ncu gpu__time_duration per layer_kernel launch (us); bench.py --steps 1 "
                "--warmup 0 --cpu-sample 0\n# (cold-cache, serialised: compare shares, not "
                "absolutes)\n")
        f.write("\n".join(f"{u:.2f}" for u in layer_us) + "\n")
    print(json.dumps({k: out[k] for k in ("gpu__time_duration.sum", "dram__bytes_read.sum",
                                          "dram__bytes_write.sum")}))


if __name__ == "__main__":
    main()
