"""Summarise ncu output into profiles/ (committed evidence).

  python tools/ncu_summary.py full  <report.ncu-rep> <out.md> [config] [algorithmic_bytes]
  python tools/ncu_summary.py launches <launches.csv> <out.md>

`full` extracts the metrics the roofline needs (duration, DRAM bytes, DRAM
throughput %, tensor-pipe %, occupancy, bank conflicts, registers) and, with
a config name, records the per-launch DRAM traffic in profiles/ncu_traffic.json
(read by bench.py's roofline.traffic).  `launches` totals the per-kernel device
time of a launch list (cold-cache, serialised: compare shares, not absolutes)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% of nominal peak)"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% of peak)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy (warps)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("smsp__inst_executed.sum", "instructions"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    return hdr, units, vals


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return v * scale.get(unit, 1)


def full(rep, out_md, config=None, algo=None):
    hdr, units, vals = raw_rows(rep)
    lines = [f"# ncu --set full summary: `{os.path.basename(rep)}`", ""]
    traffic = []
    for row in vals:
        name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"## {name[:120]}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        rd = wr = None
        for key, label in FULL_METRICS:
            if key in hdr:
                i = hdr.index(key)
                lines.append(f"| {label} (`{key}`) | {row[i]} {units[i]} |")
                if key == "dram__bytes_read.sum":
                    rd = to_bytes(row[i], units[i])
                if key == "dram__bytes_write.sum":
                    wr = to_bytes(row[i], units[i])
        if rd is not None and wr is not None:
            traffic.append(rd + wr)
            lines.append(f"| DRAM traffic read+write | {(rd + wr) / 1e9:.4f} GB |")
            if algo:
                lines.append(f"| algorithmic bytes per launch | {algo / 1e9:.4f} GB (traffic / algorithmic = "
                             f"{(rd + wr) / algo:.4f}) |")
        lines.append("")
    open(out_md, "w").write("\n".join(lines) + "\n")
    if config and traffic:
        path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        d = json.load(open(path)) if os.path.exists(path) else {}
        d[config] = round(sum(traffic) / len(traffic))
        json.dump(d, open(path, "w"), indent=1, sort_keys=True)
    print(open(out_md).read())


def launches(csv_path, out_md):
    text = open(csv_path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    tot = {}
    n = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"][:100]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(
            r.get("Metric Unit", "us"), 1)
        tot[k] = tot.get(k, 0) + v * scale
        n[k] = n.get(k, 0) + 1
    setup = {k for k in tot if "fill_kv" in k or "fill_q" in k or "values_kernel" in k}
    probe = {k for k in tot if "read_kernel" in k or "FillFunctor" in k}
    all_us = sum(v for k, v in tot.items() if k not in setup and k not in probe) or 1.0
    lines = [f"# ncu launch list: `{os.path.basename(csv_path)}`", "",
             "Per-launch device time with `--metrics gpu__time_duration.sum --clock-control none` "
             "(cold-cache, serialised: compare shares, not absolutes).", "",
             "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k in sorted(tot, key=lambda x: -tot[x]):
        share = ("setup (input generator)" if k in setup else
                 "outside the timed region (bench's read-ceiling probe / torch fills)" if k in probe else
                 f"{100 * tot[k] / all_us:.1f}%")
        lines.append(f"| `{k}` | {n[k]} | {tot[k]:.1f} | {tot[k] / n[k]:.2f} | {share} |")
    open(out_md, "w").write("\n".join(lines) + "\n")
    print(open(out_md).read())


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None,
             float(sys.argv[5]) if len(sys.argv) > 5 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
