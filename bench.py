#!/usr/bin/env python
"""Benchmark of the B200 SageAttention2++ path (BASELINE.json metric: attention TOPS).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--seq 16384] [--causal] [--pv-accum fp16|fp32]

Workload (BASELINE.json configs[1], the headline): kernel bench, batch 4, 32 heads,
head_dim 128, seq 16384, non-causal, bf16 Q/K/V (synthetic N(0,1)).  A step is one
sageattn forward (prepass + attention kernel) over the whole batch.  Metric: attention
TOPS = 4*B*H*N^2*D (x0.5 causal) / time.  Multi-GPU: the 128-row query tiles of all
(batch, head)s are split contiguously across ranks (parallel.TilePlan, balanced to one tile) with
no data-path collective (strong scaling); the long-context config uses the Ulysses all-to-all.
value = all ranks' ops / max-over-ranks device time.  Rank 0 prints ONE JSON line.

--impl reference times the reference's CPU path -- the unmodified lpattn.attention_quantized,
pip-installed into baseline/_ref (falls back to the oracle port in oracle/sage_cpu.py if that
install is absent) -- on all host cores, one head per process, on a bounded sample of the same
workload (its rate is independent of N).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# (batch, q heads, kv heads, seq, head_dim, causal) per BASELINE.json config
WORKLOADS = {
    "kernel": (4, 32, 32, 16384, 128, False),     # configs[1]: kernel bench, the headline
    "cogvideox": (2, 30, 30, 17776, 64, False),   # configs[2]
    "llama": (8, 32, 8, 8192, 128, True),          # configs[3]: GQA 4
    "longctx": (1, 32, 32, 131072, 128, True),     # configs[4]: Ulysses all-to-all when N > 1
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="kernel",
                    help="BASELINE.json configs: kernel (configs[1], the headline), cogvideox, llama, longctx")
    ap.add_argument("--seq", type=int, default=None, help="override the sequence length")
    ap.add_argument("--causal", action="store_true", help="causal variant of the kernel workload")
    ap.add_argument("--head-dim", type=int, default=None, choices=[64, 128], help="override the head dim")
    ap.add_argument("--pv-accum", choices=["fp16", "fp32"], default="fp16")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def ops_of(B, H, N, D, causal):
    return 4.0 * B * H * N * N * D * (0.5 if causal else 1.0)


def resolve(a):
    B, Hq, Hkv, N, D, causal = WORKLOADS[a.workload]
    if a.seq is not None:
        N = a.seq
    if a.head_dim is not None:
        D = a.head_dim
    if a.causal:
        causal = True
    a.batch, a.heads, a.kv_heads, a.seq, a.head_dim, a.causal = B, Hq, Hkv, N, D, causal
    return a


def workload_name(a):
    return (f"{a.workload}_b{a.batch}_h{a.heads}" + (f"kv{a.kv_heads}" if a.kv_heads != a.heads else "")
            + f"_n{a.seq}_d{a.head_dim}_{'causal' if a.causal else 'noncausal'}")


def prepass_bytes(Hq, Hkv, N, D):
    """Algorithmic HBM bytes of the prepass for bf16 inputs: Q read twice (means, codes), K read
    twice, V once, int8/e4m3 codes written once; scales/bias are O(N) and ignored."""
    return N * D * (Hq * (2 * 2 + 1) + Hkv * (2 * 2 + 1 + 2 + 1))


def metric_name():
    return "attention TOPS (hd128, seq 1K-32K, causal/non-causal) vs B200 FP8 peak; cossim/L1"


# ----------------------------------------------------------------------------- CPU reference leg
REF_INSTALL = ROOT / "baseline" / "_ref"  # pip install --target of the unmodified reference (lpattn)


def reference_kind() -> str:
    """'reference' when the unmodified lpattn is installed in baseline/_ref, else 'port' (the
    oracle restatement in oracle/sage_cpu.py, pinned bit-exact to the reference's goldens)."""
    return "reference" if (REF_INSTALL / "lpattn" / "__init__.py").exists() else "port"


def _cpu_head(args):
    seed, n, d, causal = args
    import numpy as np
    rng = np.random.Generator(np.random.Philox(seed))
    q, k, v = (rng.normal(size=(n, d)).astype(np.float32) for _ in range(3))
    if reference_kind() == "reference":
        sys.path.insert(0, str(REF_INSTALL))
        import lpattn as impl  # the reference's own operator, stock code path
    else:
        from oracle import sage_cpu as impl
    cfg = impl.AttentionConfig(seq_len=n, head_dim=d, causal=causal)
    t0 = time.perf_counter()
    impl.attention_quantized(q, k, v, cfg)
    return time.perf_counter() - t0


def cpu_reference_rate(n_sample: int, d: int, causal: bool, procs: int):
    """Reference CPU path on `procs` heads of (n_sample x d) in parallel; returns (TOPS, wall s)."""
    import concurrent.futures as cf
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    t0 = time.perf_counter()
    with cf.ProcessPoolExecutor(procs) as ex:
        list(ex.map(_cpu_head, [(1000 + i, n_sample, d, causal) for i in range(procs)]))
    wall = time.perf_counter() - t0
    return procs * ops_of(1, 1, n_sample, d, causal) / wall / 1e12, wall


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    procs = max(1, os.cpu_count() or 1)
    n_sample = 1024
    vals = []
    for i in range(a.warmup + a.steps):
        v, _ = cpu_reference_rate(n_sample, a.head_dim, a.causal, procs) if i >= a.warmup else (None, None)
        if i >= a.warmup:
            vals.append(v)
        elif i == 0:
            cpu_reference_rate(256, a.head_dim, a.causal, procs)  # warm the pool/imports once
    value = statistics.median(vals)
    kind = reference_kind()
    sample = (f"{procs} heads x seq {n_sample} x d {a.head_dim} "
              f"{'causal' if a.causal else 'non-causal'}, fp32 N(0,1), one head per process, "
              f"{'lpattn.attention_quantized (baseline/_ref)' if kind == 'reference' else 'oracle port'}; "
              f"rate is N-independent (SURVEY A.8), applied to the workload's ops")
    line = {
        "impl": "reference", "metric": metric_name(), "value": value, "unit": "TOPS",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ops_of(1, procs, n_sample, a.head_dim, a.causal) / (value * 1e12) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64 (numpy emulation of int8/e4m3/fp16-acc)", "data": "synthetic",
        "config": {"workload": workload_name(a), "sample": sample},
        "cpu_baseline": {"value": value, "unit": "TOPS", "cores": procs, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU leg
class ClockSampler:
    def __init__(self, idx: int):
        self.idx = idx
        self.proc = None
        self.path = Path(f"/tmp/sa2pp_clocks_{os.getpid()}.csv")

    def __enter__(self):
        if self.proc is not None:  # already sampling (started before the warm-up)
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            import atexit
            atexit.register(self.stop)  # never leave a sampler behind, whatever happens in between
        except Exception:
            self.proc = None
        return self

    def stop(self):
        if self.proc is not None and self.proc.poll() is None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def wait_started(self, timeout: float = 3.0):
        """Block until the sampler has written its first row (so the timed region is covered)."""
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < timeout:
            if self.path.exists() and self.path.stat().st_size > 0:
                return
            time.sleep(0.05)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)  # one more sample after the last timed step
            self.stop()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return None
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                try:
                    rows.append((float(parts[0]), float(parts[1]), parts[4:8]))
                except ValueError:
                    pass
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, x in enumerate(r) if x.lower() == "active"})
        loaded = [c for c, _, _ in rows if c > 500] or [c for c, _, _ in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(m for _, m, _ in rows),
                "reasons": reasons, "samples": len(rows)}


def read_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("bf16_tflops", 1590.0)), "MEASURED_PEAKS.json"
    return 1590.0, "fallback (B200_PROFILING.md)"


def read_fp8_measured():
    """cuBLASLt e4m3 8192^3 on this pool (tools/fp8_peak.py), committed under profiles/."""
    p = ROOT / "profiles" / "r01_fp8_peak.json"
    if not p.exists():
        return None
    try:
        return float(json.loads(p.read_text())["fp8_e4m3_tflops_burst"])
    except (KeyError, ValueError):
        return None


def read_traffic(workload: str):
    p = ROOT / "profiles" / "attn_ncu_summary.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    e = d.get(workload)
    return None if e is None else e.get("dram_bytes_per_launch")


def run_ours(a):
    import torch
    import torch.distributed as dist
    import paper_2505_21136_b200 as sa
    from paper_2505_21136_b200 import api, parallel, _abi as A

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SA2PP_BENCH_SHARE_GPU=1 (tests only): every rank on cuda:0 with gloo collectives on host tensors,
    # so the multi-rank sharding path runs on a one-GPU box; numbers from it are not bench values
    share = os.environ.get("SA2PP_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def max_over_ranks(vals):
        if world == 1:
            return list(vals)
        t = torch.tensor(list(vals), dtype=torch.float64, device="cpu" if share else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    B, H, Hkv, N, D = a.batch, a.heads, a.kv_heads, a.seq, a.head_dim
    group = H // Hkv
    ulysses = a.workload == "longctx" and world > 1 and not share
    if ulysses:
        # sequence-sharded input [1, N/P, H, D] per rank; all-to-all to [1, N, H/P, D] and back
        Ul, Nl = H // world, N // world
    else:
        # 128-row query tiles of all (batch, head)s sharded contiguously across ranks (balanced to one
        # tile); each rank quantizes the heads (whole GQA groups) its range touches; no collective
        plan = parallel.tile_plan(B, H, Hkv, N, world, rank)
        Ul, Nl = plan.local_heads, N
        u0, u1 = plan.local_units
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    rnd = lambda *shape: torch.randn(*shape, device=dev, generator=gen, dtype=torch.float32).bfloat16()  # noqa: E731
    if ulysses:
        xq, xk, xv = rnd(1, Nl, H, D), rnd(1, Nl, H, D), rnd(1, Nl, H, D)
        q = torch.empty(1, N, Ul, D, device=dev, dtype=torch.bfloat16)  # head-sharded buffers (NHD)
        k, v = torch.empty_like(q), torch.empty_like(q)
        layout_strides = lambda t: (t.stride(0), t.stride(2), t.stride(1))  # noqa: E731
    else:
        q = rnd(1, Ul, N, D)
        k, v = rnd(1, Ul // group, N, D), rnd(1, Ul // group, N, D)
        layout_strides = lambda t: (t.stride(0), t.stride(1), t.stride(2))  # noqa: E731
    out = torch.empty_like(q)
    prob = api._problem(1, Ul, Ul // group if not ulysses else Ul, N, D, causal=a.causal, pv_accum=a.pv_accum)
    qt = api.alloc_quant(prob, dev)
    import ctypes
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    ins = A.Inputs(A.SA2PP_BF16, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                   (ctypes.c_int64 * 3)(*layout_strides(q)), (ctypes.c_int64 * 3)(*layout_strides(k)),
                   (ctypes.c_int64 * 3)(*layout_strides(v)))
    o = A.Output(A.SA2PP_BF16, out.data_ptr(), (ctypes.c_int64 * 3)(*layout_strides(out)))
    qs = qt.struct()
    lib = A.lib()

    def exchange_in():
        if ulysses:
            for src, dst in ((xq, q), (xk, k), (xv, v)):
                dst.copy_(parallel.seq_to_head(src, world))

    def exchange_out():
        if ulysses:
            parallel.head_to_seq(out, world)

    def prepass():
        A.check(lib.sa2pp_prepass(ctypes.byref(prob), ctypes.byref(ins), ctypes.byref(qs),
                                  qt.workspace.data_ptr(), qt.workspace.numel(), sp))

    def attn():
        if ulysses:
            A.check(lib.sa2pp_attn_fwd(ctypes.byref(prob), ctypes.byref(qs), ctypes.byref(o), None, sp))
        else:
            A.check(lib.sa2pp_attn_fwd_units(ctypes.byref(prob), ctypes.byref(qs), ctypes.byref(o), None, u0, u1 - u0,
                                             sp))

    launches_per_step = 5  # channel_means, quantize_q, quantize_k, quantize_v, attention
    # inputs + output smaller than twice the 126 MB L2: flush it between timed steps (a 512 MB write,
    # outside the per-step events) so every step reads Q/K/V from HBM
    resident = sum(t.numel() * t.element_size() for t in (q, k, v, out))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if resident < 2 * (126 << 20) else None

    # the clock sampler starts before the warm-up (nvidia-smi needs ~0.3 s to report) and keeps going
    # until the timed steps are done; it must not be the thing that is slow to start
    clk = ClockSampler(local).__enter__()
    clk.wait_started()
    for _ in range(a.warmup):
        exchange_in()
        prepass()
        attn()
        exchange_out()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    with clk:
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for e0, e1, e2 in ev:
            if flush is not None:
                flush.fill_(1)
            exchange_in()
            e0.record(stream)
            prepass()
            e1.record(stream)
            attn()
            e2.record(stream)
            exchange_out()
        t_end.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    total_ms = t_start.elapsed_time(t_end)
    if flush is not None:  # the flushes sit between the timed steps, not in them
        total_ms = sum(e0.elapsed_time(e2) for e0, _, e2 in ev)
    attn_ms = statistics.mean(e1.elapsed_time(e2) for _, e1, e2 in ev)
    pre_ms = statistics.mean(e0.elapsed_time(e1) for e0, e1, _ in ev)
    total_ms, attn_ms, pre_ms = max_over_ranks([total_ms, attn_ms, pre_ms])
    ms_per_step = total_ms / a.steps
    job_ops = ops_of(B, H, N, D, a.causal)  # all ranks together
    value = job_ops / (ms_per_step * 1e-3) / 1e12

    # ---------------- end-to-end through the public API with pinned host buffers
    e2e = None
    if not a.no_e2e:
        src = (xq, xk, xv) if ulysses else (q, k, v)
        hq, hk, hv = (t.cpu().pin_memory() for t in src)
        ho = torch.empty(src[0].shape, dtype=out.dtype, pin_memory=True)
        pipe = None if ulysses else sa.HostPipeline(1, Ul, Ul // group, N, D, torch.bfloat16, dev,
                                                    is_causal=a.causal, pv_accum=a.pv_accum)

        def e2e_step():
            if ulysses:
                dq, dk, dv = (h.to(dev, non_blocking=True) for h in (hq, hk, hv))
                r = parallel.ulysses_sageattn(dq, dk, dv, a.causal, None, pv_accum=a.pv_accum, quant=qt)
                ho.copy_(r, non_blocking=True)
            else:  # public host API: chunked copies in both directions overlapped with the kernels
                pipe(hq, hk, hv, ho)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_e2e = max(1, min(a.steps, 5))
        s0.record(stream)
        for _ in range(n_e2e):
            e2e_step()
        s1.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = s0.elapsed_time(s1) / n_e2e
        e2e_ms = max_over_ranks([e2e_ms])[0]
        e2e = {"value": job_ops / (e2e_ms * 1e-3) / 1e12, "unit": "TOPS",
               "h2d_bytes_per_step": sum(t.numel() * t.element_size() for t in (hq, hk, hv)) * world,
               "d2h_bytes_per_step": ho.numel() * ho.element_size() * world,
               "ms_per_step": e2e_ms}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    bf16_peak, peak_src = read_peaks()
    fp8_peak = 2.0 * bf16_peak  # dense FP8/INT8 tensor rate is 2x dense BF16 on B200
    # the attention launch of rank 0: its share of the query tiles (all of them at world 1)
    attn_ops_per_launch = ops_of(B, H, N, D, a.causal) * ((u1 - u0) / plan.total_units if not ulysses else 1.0 / world)
    achieved = attn_ops_per_launch / (attn_ms * 1e-3) / 1e12
    line = {
        "metric": metric_name(), "value": value, "unit": "TOPS", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int8 QK / e4m3 PV (fp16 acc)" if a.pv_accum == "fp16" else "int8 QK / e4m3 PV (fp32 acc)",
        "data": "synthetic N(0,1) bf16 Q/K/V",
        "config": {"workload": workload_name(a), "batch": B, "heads": H, "kv_heads": Hkv, "seq_len": N,
                   "head_dim": D, "causal": a.causal, "pv_accum": a.pv_accum,
                   "parallelism": (f"ulysses x{world}" if ulysses else f"q-tile shard x{world}"),
                   "l2": ("L2 flushed between steps (512 MB write outside the step events); %.0f MB bf16 Q/K/V"
                          if flush is not None else "inputs larger than L2 (%.0f MB bf16 Q/K/V per GPU)") % (
                       sum(t.numel() for t in (q, k, v)) * 2 / 1e6)},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": fp8_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp8_peak, "traffic": read_traffic(workload_name(a)),
                     "kernel": "attn_ws_kernel", "ops_per_launch": attn_ops_per_launch,
                     "ms_per_launch": attn_ms, "peak_source": f"2 x bf16 {bf16_peak} ({peak_src})",
                     "frac_of_nominal_4500": achieved / 4500.0,
                     "fp8_cublas_measured_tflops": read_fp8_measured()},
        "prepass": {"ms_per_launch": pre_ms, "hbm_bytes": prepass_bytes(Ul, Ul // group if not ulysses else Ul, N, D),
                    "achieved_gbs": prepass_bytes(Ul, Ul // group if not ulysses else Ul, N, D) / (pre_ms * 1e-3) / 1e9},
        "gpu_launches": launches_per_step * a.steps,
        "clocks": clk.summary(),
    }
    if e2e is not None:
        line["e2e"] = e2e
    if not a.no_cpu:
        procs = max(1, os.cpu_count() or 1)
        v_cpu, wall = cpu_reference_rate(1024, D, a.causal, procs)
        line["cpu_baseline"] = {"value": v_cpu, "unit": "TOPS", "cores": procs, "kind": reference_kind(),
                                "sample": f"{procs} heads x seq 1024 x d {D}, one head per process "
                                          f"({wall:.1f} s wall); rate is N-independent (SURVEY A.8)"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = resolve(parse())
    if a.warmup < 3:
        a.warmup = 3
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
