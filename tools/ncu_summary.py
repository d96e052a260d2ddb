"""Summarise ncu reports / launch lists into profiles/ (text, committed).

    python tools/ncu_summary.py gpurun_out/prof_pipe_c5.ncu-rep [...] > profiles/<name>.md
    python tools/ncu_summary.py --launches gpurun_out/launches_c5.csv
"""

import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "CTA threads"),
    ("launch__occupancy_limit_shared_mem", "CTAs/SM (smem limit)"),
    ("launch__occupancy_limit_registers", "CTAs/SM (register limit)"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall: long scoreboard"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall: barrier"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall: short scoreboard"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall: lg throttle"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall: mio throttle"),
    ("smsp__inst_executed.sum", "instructions"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 LSU data-pipe wavefronts % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "shared-memory load wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "shared-memory store wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared-memory bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared-memory bank conflicts (loads)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "shared-memory bank conflicts (stores)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ldgsts.sum", "shared-memory bank conflicts (LDGSTS fills)"),
    ("l1tex__t_sector_hit_rate.pct", "L1 sector hit rate"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "global load requests"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "global store requests"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
]


def raw(report: str):
    if report.endswith(".csv"):  # `ncu -i <rep> --page raw --csv` exported on the GPU box
        out = open(report).read()
    else:
        out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def to_bytes(value: str, unit: str) -> float:
    return float((value or "0").replace(",", "")) * SCALE.get(unit.strip(), 1)


def summarise(report: str) -> str:
    data = raw(report)
    if not data:
        return f"## {report}\n(no data)\n"
    lines = []
    for vals, units in data:
        lines.append(f"## {report}\n\nkernel: `{vals.get('Kernel Name', '?')}`\n")
        lines.append("| metric | value |\n|---|---|")
        for key, label in METRICS:
            if key in vals:
                lines.append(f"| {label} (`{key}`) | {vals[key]} {units.get(key, '')} |")
        rd = to_bytes(vals.get("dram__bytes_read.sum", "0"), units.get("dram__bytes_read.sum", "byte"))
        wr = to_bytes(vals.get("dram__bytes_write.sum", "0"), units.get("dram__bytes_write.sum", "byte"))
        lines.append(f"\ntraffic (read+write): {rd + wr:.6g} bytes = {(rd + wr) / 1e9:.4f} GB\n")
    return "\n".join(lines) + "\n"


def launches(path: str) -> str:
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = {}
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        a = agg.setdefault((name, r[im], r[iu]), [0, 0.0])
        a[0] += 1
        a[1] += float(r[iv].replace(",", ""))
    out = [f"## launch list {path}\n", "| kernel | metric | launches | sum over launches (mean for % / ratios) |",
           "|---|---|---|---|"]
    for (name, metric, unit), (cnt, tot) in sorted(agg.items()):
        rate = unit.strip() in ("%", "") or metric.endswith((".pct", ".ratio")) or "pct_of_peak" in metric
        val = f"mean {tot / cnt:.4g}" if rate else f"{tot:.4g}"
        out.append(f"| `{name}` | {metric} | {cnt} | {val} {unit} |")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--launches":
        for p in args[1:]:
            print(launches(p))
    else:
        for p in args:
            print(summarise(p))
