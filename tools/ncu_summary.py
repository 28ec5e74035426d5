"""Summarise an ncu report (``--set full``) into the markdown tables kept
under profiles/: duration, throughput, DRAM traffic, issue efficiency,
instruction mix and the warp-stall breakdown of each captured kernel.

usage: python tools/ncu_summary.py REPORT.ncu-rep [more.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed_pipe_fma.sum", "FMA-pipe warp instr"),
    ("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "FFMA thread instr"),
    ("smsp__inst_executed.sum", "warp instr executed"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_registers", "occ limit (regs)"),
    ("launch__occupancy_limit_shared_mem", "occ limit (smem)"),
]
STALL_PREFIX = "smsp__average_warp_latency_issue_stalled_"
STALL_PREFIX2 = "smsp__average_warps_issue_stalled_"


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def summarise(path):
    head, units, data = rows(path)
    lines = []
    for row in data:
        get = dict(zip(head, row))
        unit = dict(zip(head, units))
        lines.append(f"### `{get.get('Kernel Name', '?')}`\n")
        lines.append(f"report: `{path}`\n")
        lines.append("| metric | value | unit |\n|---|---|---|")
        for k, name in KEYS:
            if k in get:
                lines.append(f"| {name} (`{k}`) | {get[k]} | {unit.get(k, '')} |")
        stalls = []
        for k, v in get.items():
            for pre in (STALL_PREFIX2,):
                if k.startswith(pre) and k.endswith("_per_issue_active.ratio"):
                    try:
                        stalls.append((float(v.replace(",", "")), k[len(pre):-len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
        if stalls:
            stalls.sort(reverse=True)
            lines.append("\nwarp stalls (warps stalled per issue-active cycle), top 10:\n")
            lines.append("| reason | ratio |\n|---|---|")
            for v, name in stalls[:10]:
                lines.append(f"| {name} | {v:.3f} |")
        lines.append("")
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarise(p))
