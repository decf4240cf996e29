"""Summarise an ncu report (--set full) into profiles/: key throughput, pipe, stall and DRAM metrics.

    python tools/ncu_summary.py gpurun_out/r01a/attn_full.ncu-rep profiles/r01_attn_v3.md [--json key]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", "tensor imma subpipe %"),
    ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", "tensor hmma subpipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed"),
]
STALLS = ["barrier", "wait", "short_scoreboard", "long_scoreboard", "math_pipe_throttle", "mio_throttle",
          "not_selected", "selected", "branch_resolving", "dispatch_stall", "no_instruction", "lg_throttle",
          "membar", "sleeping", "tex_throttle", "drain", "misc"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res = []
    for r in rows[2:]:
        res.append({h: (v, u) for h, u, v in zip(rows[0], rows[1], r)})
    return res


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    kernels = raw(rep)
    lines = [f"# ncu summary of `{rep.split('/')[-1]}`", ""]
    js = []
    for k in kernels:
        name = k.get("Kernel Name", ("?", ""))[0]
        lines.append(f"## {name[:160]}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        d = {"kernel": name}
        for key, label in KEYS:
            if key in k:
                v, u = k[key]
                lines.append(f"| {label} (`{key}`) | {v} {u} |")
                d[key] = v + (" " + u if u else "")
        lines.append("")
        lines.append("Warp stall reasons (warps per issued instruction):")
        lines.append("")
        for s in STALLS:
            key = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if key in k:
                lines.append(f"- {s}: {k[key][0]}")
        lines.append("")
        js.append(d)
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
