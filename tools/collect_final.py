"""Copy a tools/gpu_final.sh run (gpurun_out/<tag>) into profiles/r02/final/: bench lines, ncu
summaries, launch list, test logs, and the configs[1] sweep with each line's roofline.traffic filled
from its ncu DRAM counters; updates profiles/attn_ncu_summary.json (read by bench.py) and writes
profiles/r02/final/sweep.md.

    python tools/collect_final.py r02final3
"""
import csv
import glob
import json
import os
import shutil
import sys

tag = sys.argv[1]
SRC = f"gpurun_out/{tag}"
DST = "profiles/r02/final"
os.makedirs(f"{DST}/sweep", exist_ok=True)
for pat in ("bench*.json", "launches.csv", "attn_fp16_summary.md", "attn_fp32_summary.md", "attn_fp16_ophist.txt",
            "attn_fp32_ophist.txt", "prepass_summary.md", "pytest_gpu.log", "smoke.log", "smi.txt", "pipe_bench.txt"):
    for f in glob.glob(f"{SRC}/{pat}"):
        shutil.copy(f, DST)

summ_path = "profiles/attn_ncu_summary.json"
summ = json.load(open(summ_path))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rows_md = []
for f in sorted(glob.glob(f"{SRC}/sweep/bench_*.json")):
    n = os.path.basename(f)[6:-5]
    d = json.load(open(f))
    t = f"{SRC}/sweep/traffic_{n}.csv"
    traffic = None
    if os.path.exists(t):
        rows = list(csv.reader(open(t)))
        hs = [i for i, r in enumerate(rows) if "Kernel Name" in r]
        if hs:
            hdr = rows[hs[0]]
            mi, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
            m = {r[mi]: float(r[vi].replace(",", "")) * scale.get(r[ui], 1) for r in rows[hs[0] + 1:] if len(r) > vi}
            rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
            traffic = int(rd + wr)
            summ[d["config"]["workload"]] = {
                "kernel": "attn_ws_kernel (round 2)",
                "source": f"profiles/r02/final/sweep/traffic_{n}.csv (ncu --metrics dram__bytes_read.sum,"
                          "dram__bytes_write.sum, one launch)",
                "dram_bytes_per_launch": traffic, "dram_read": int(rd), "dram_write": int(wr)}
            shutil.copy(t, f"{DST}/sweep/")
    d["roofline"]["traffic"] = traffic
    json.dump(d, open(f"{DST}/sweep/bench_{n}.json", "w"))
    c = d["config"]
    rows_md.append((c["head_dim"], c["causal"], c["seq_len"], d["value"], d["roofline"]["achieved"], d["roofline"]["frac"],
                    d["prepass"]["ms_per_launch"], d["e2e"]["value"], traffic, d["cpu_baseline"]["value"],
                    c["l2"].startswith("L2 flushed"), (d.get("clocks") or {}).get("sm_mhz")))
json.dump(summ, open(summ_path, "w"), indent=2)
rows_md.sort()
with open(f"{DST}/sweep.md", "w") as fo:
    fo.write("# BASELINE configs[1] sweep through bench.py (B200, round 2 final build)\n\n")
    fo.write("batch 4 x 32 heads, bf16 N(0,1), FP16 PV accumulation; one `python bench.py --seq N --head-dim D "
             "[--causal]` line per row (`sweep/bench_*.json`), attention-kernel DRAM traffic per launch from ncu "
             "(`sweep/traffic_*.csv`).  Step = prepass + attention, device time; e2e = host arrays through the native "
             "host pipeline (PCIe-bound); CPU = the unmodified lpattn on the host cores, rate N-independent.\n\n")
    fo.write("| D | causal | N | step TOPS | attention TOPS | frac of 3,255 | prepass ms | e2e TOPS | DRAM MB/launch "
             "| CPU TOPS | L2 | SM MHz |\n|---|---|---|---|---|---|---|---|---|---|---|---|\n")
    for r in rows_md:
        fo.write(f"| {r[0]} | {'yes' if r[1] else 'no'} | {r[2]} | {r[3]:.1f} | {r[4]:.1f} | {r[5]:.3f} | {r[6]:.3f} "
                 f"| {r[7]:.1f} | {(r[8] or 0) / 1e6:.0f} | {r[9]:.4f} | {'flushed' if r[10] else 'inputs > L2'} "
                 f"| {r[11]} |\n")
print(open(f"{DST}/sweep.md").read())
