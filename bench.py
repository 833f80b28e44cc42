#!/usr/bin/env python3
"""DynamiQ all-reduce benchmark (B200).  Prints ONE JSON line on rank 0.

Workloads (BASELINE.json configs):
  N = 1 : configs[1] — one B200 runs the full round of n_sim = 4 simulated
          workers (stats, allocation, permuted ring reduce-scatter with leaf
          compress + fused DAR per hop + sink, compressed gather decode) on
          64M-entry synthetic Llama-like (per-super-group log-normal scale,
          sigma_log = 4) fp32 gradients, 4-bit budget.
  N > 1 : configs[2] — one rank per GPU (torchrun), 256M-entry (1 GiB fp32)
          gradient per rank, ring, 4-bit budget; NCCL bf16 all-reduce timed
          beside it.

metric "effective GB/s": fp32 gradient bytes all-reduced per second summed
over workers, (workers x 4 d) / t — whole-job, so weak scaling keeps per-GPU
work fixed.  ``value`` is device-resident (inputs already in HBM); ``e2e`` runs
the same round through the C-ABI from pinned host buffers (H2D of every input
and D2H of the sum inside the timed region).

``--impl reference`` times the reference's own CPU implementation of the path
(oracle/_ref: the reference library compiled from its sources) on this box's
host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np


ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DynamiQ all-reduce effective GB/s (4-bit budget, fp32-equivalent bytes x workers / s)"
UNIT = "GB/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--entries", "--d", dest="d", type=int, default=0,
                   help="entries per worker (default 2^26 at N=1, 2^28 at N>1)")
    p.add_argument("--n-sim", type=int, default=4, help="simulated workers at N=1")
    p.add_argument("--budget", type=float, default=4.0)
    p.add_argument("--topology", default="ring", choices=["ring", "butterfly"])
    p.add_argument("--sigma-log", type=float, default=4.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-sample-d", type=int, default=1 << 22)
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 10:  # sampler is live before timing starts
                time.sleep(0.02)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        time.sleep(0.06)  # one more sample covering the end of the timed region
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def make_inputs(n, d, sigma_log, seed=1, ranks=None):
    """The bench workload's n worker gradients (host fp32): Llama-like heavy-tailed, i.e. a
    per-super-group log-normal scale shared by every worker (the reference generator's
    locality structure, proj/src/synth.cpp:31-54) times per-worker N(0, 1) entries.  Both
    arms (ours and --impl reference) all-reduce exactly these arrays."""
    T = (d + 255) // 256
    rng = np.random.default_rng(seed)
    scale = np.exp(sigma_log * rng.standard_normal(T)).astype(np.float32)
    out = []
    for r in (range(n) if ranks is None else ranks):
        x = np.random.default_rng([seed, 1000 + r]).standard_normal((T, 256), dtype=np.float32)
        x *= scale[:, None]
        out.append(x.reshape(-1)[:d])
    return out


def synth(torch, d, n, sigma_log, seed=1, device="cuda"):
    """Llama-like heavy-tailed gradients: per-super-group log-normal scale shared
    across workers (proj/src/synth.cpp:46-53), entries N(0, sigma_j^2) per worker."""
    g = torch.Generator(device=device).manual_seed(seed)
    T = (d + 255) // 256
    scale = torch.exp(sigma_log * torch.randn(T, device=device, generator=g))
    out = []
    for r in range(n):
        x = torch.randn(T, 256, device=device, generator=g) * scale[:, None]
        out.append(x.reshape(-1)[:d].contiguous())
    return out


# algorithmic bytes per entry of each kernel family (c = compressed bits per
# entry incl. scales): what the engine books per launch (dq_engine.cpp quant_bytes & co.)
FAMILY_BYTES = {"stats": "4 (+ 8/256 per worker row)", "reduce_stats": "8(n+1)/256",
                "quant_leaf": "4 + 8/256 + c/8", "quant_dar": "4 + 8/256 + 2c/8 (+4 output for fused sinks)",
                "decompress_accumulate": "8 + c/8", "decode_out": "c/8 + 4 + 8/256",
                "alloc_search": "8/256 per pass", "alloc_assign": "13/256"}


def roofline_families(prof, peak):
    """Achieved GB/s of every kernel family (algorithmic bytes / live CUDA-event time)."""
    out = {}
    for k, p in prof.items():
        if p["ms"] <= 0 or k == "nccl":
            continue
        gbs = p["bytes"] / (p["ms"] * 1e-3) / 1e9
        out[k] = {"achieved_gbs": round(gbs, 1), "frac": round(gbs / peak, 4), "launches": p["launches"],
                  "avg_launch_ms": round(p["ms"] / max(p["launches"], 1), 5),
                  "bytes_per_entry": FAMILY_BYTES.get(k)}
    return out


def roofline_of(prof, peak, peak_kind, kernel="quant_dar", traffic_ok=True):
    p = prof.get(kernel)
    if not p or p["ms"] <= 0:
        return None
    achieved = p["bytes"] / (p["ms"] * 1e-3) / 1e9
    traffic = traffic_alg = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                nc = json.load(f).get(kernel, {})
            # the capture is of an N=1 bench launch; other configs launch different sizes
            if traffic_ok:
                traffic = nc.get("dram_bytes_per_launch")
                traffic_alg = nc.get("algorithmic_bytes_same_launch")
        except Exception:
            traffic = None
    out = {"bound": "hbm", "kernel": kernel, "achieved": round(achieved, 1), "peak": peak, "peak_source": peak_kind,
           "unit": "GB/s", "frac": round(achieved / peak, 4),
           "algorithmic_bytes_per_launch": p["bytes"] / max(p["launches"], 1),
           "avg_launch_ms": p["ms"] / max(p["launches"], 1), "launches": p["launches"], "traffic": traffic}
    if traffic is not None:
        out["traffic_source"] = {"capture": "profiles/ncu_traffic.json (one N=1 DAR hop launch)",
                                 "algorithmic_bytes_same_launch": traffic_alg}
    else:
        out["traffic_source"] = "null: the committed ncu capture is of the N=1 bench's DAR launch, not this config's"
    # the fused hop is integer-issue-bound: the issue-side numbers of the
    # same kernel from the committed ncu capture
    try:
        with open(tpath) as f:
            nc = json.load(f).get(kernel, {})
        if "ipc" in nc:
            out["issue"] = {"ipc": nc["ipc"], "max_ipc": 4.0, "alu_pipe_pct": nc.get("alu_pipe_pct"),
                            "issue_active_pct": nc.get("issue_active_pct"), "source": "profiles/ncu_traffic.json"}
    except Exception:
        pass
    return out


def cpu_baseline(hw, d_sample, budget, topology, sigma_log, gpu_vnmse_fn=None, steps=1):
    """The reference's own run_round (oracle/_ref) on a bounded sample of the SAME inputs
    (the first d_sample entries of every worker), all chunk threads; with gpu_vnmse_fn the
    device round on that sample too, so both vNMSEs are on identical inputs."""
    from oracle.oracle import Oracle, available
    kind = "reference" if available("reference") else "port"
    ora = Oracle(kind)
    n = len(hw)
    ws = [np.ascontiguousarray(w[:d_sample]) for w in hw]
    threads = min(n, os.cpu_count() or 1) if kind == "reference" else 1
    cfg = ora.round_cfg(n, budget, topology, seed=1, threads=threads)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        res = ora.run_round(ws, cfg)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    out = {"value": round(n * 4 * d_sample / t / 1e9, 6), "unit": UNIT, "cores": threads, "kind": kind,
           "sample": f"run_round n={n} {topology} b={budget} on the first {d_sample} entries of each of the "
                     f"bench's {n} worker gradients (same inputs as the timed arm), median of {steps}",
           "seconds_per_round": round(t, 4), "vnmse": res["vnmse"]}
    if gpu_vnmse_fn is not None:
        out["gpu_vnmse_same_sample"] = gpu_vnmse_fn(ws)
    return out


# --------------------------------------------------------------------- N = 1
def bench_sim(args):
    import torch
    import paper_2602_08923_b200 as dq
    d = args.d or (1 << 26)
    n = args.n_sim
    cfg = dq.PipelineConfig(n_workers=n, budget_bits=args.budget,
                            topology=dq.BUTTERFLY if args.topology == "butterfly" else dq.RING,
                            seed=dq.SharedSeed(1, 0))
    ctx = dq.Context(cfg)
    hw = make_inputs(n, d, args.sigma_log)
    ws = [torch.from_numpy(w).cuda() for w in hw]
    out = torch.empty(d, device="cuda")
    st = torch.cuda.current_stream()
    r = dq.run_round(ws, cfg, out=out, ctx=ctx)  # with metrics (vNMSE vs fp64 sum), untimed
    vnmse = r.vnmse
    for _ in range(args.warmup):
        r = dq.run_round(ws, cfg, out=out, ctx=ctx, metrics=False)
    torch.cuda.synchronize()
    # timed region: K rounds back to back, no per-launch instrumentation (value)
    ctx.profile(False)
    ctx.read_profile(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    per_step = []
    with Clocks(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(args.steps):
            r = dq.run_round(ws, cfg, out=out, ctx=ctx, metrics=False)
            per_step.append(r.info["ms_total"])
        e1.record(st)
        torch.cuda.synchronize()
    launch_counts = ctx.read_profile(reset=True)
    ms = e0.elapsed_time(e1) / args.steps
    # the same K rounds again with CUDA events around every launch (per-kernel times,
    # roofline); the extra event records cost host time, so this region runs slower
    ctx.profile(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(st)
    for _ in range(args.steps):
        dq.run_round(ws, cfg, out=out, ctx=ctx, metrics=False)
    p1.record(st)
    torch.cuda.synchronize()
    prof = ctx.read_profile(reset=True)
    ctx.profile(False)
    prof_ms = p0.elapsed_time(p1) / args.steps
    value = n * 4 * d / (ms * 1e-3) / 1e9
    peak, pk = peaks()
    launches = sum(p["launches"] for p in launch_counts.values())
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 in / u8 codes (bit-exact integer PRNG path)", "data": "synthetic",
        "config": {"workload": f"configs[1]: single-B200 simulated {args.topology} all-reduce round, "
                               f"{n} workers x {d} entries, b={args.budget}, sigma_log={args.sigma_log}",
                   "global_batch": n, "entries_per_worker": d, "parallelism": f"sim{n}",
                   "l2": "inputs larger than L2 (>= 1 GiB resident)"},
        "vnmse": vnmse, "u": r.u, "widths_8_4_2": [r.info["n8"], r.info["n4"], r.info["n2"]],
        "round_device_ms_median": round(statistics.median(per_step), 4),
        "kernels": {k: {"launches": v["launches"], "ms_per_step": round(v["ms"] / args.steps, 4),
                        "GBps": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1)} for k, v in prof.items()},
        "kernels_region": {"steps": args.steps, "ms_per_step": round(prof_ms, 4),
                           "note": "second timed region, CUDA events around every launch"},
        "roofline": roofline_of(prof, peak, pk), "roofline_families": roofline_families(prof, peak),
        "gpu_launches": launches, "clocks": clk.summary(),
    }
    if not args.no_e2e:
        hosts = [torch.empty(d, dtype=torch.float32, pin_memory=True) for _ in range(n)]
        for h, w in zip(hosts, ws):
            h.copy_(w)
        hout = torch.empty(d, dtype=torch.float32, pin_memory=True)
        import ctypes as C
        from paper_2602_08923_b200._lib import RoundInfo, check, lib
        ptrs = (C.c_void_p * n)(*[h.data_ptr() for h in hosts])
        info = RoundInfo()
        sptr = C.c_void_p(st.cuda_stream)
        for _ in range(2):
            check(lib().dq_run_round_host(ctx.h, ptrs, d, C.c_void_p(hout.data_ptr()), C.byref(info), sptr))
        k = max(3, args.steps // 4)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(k):
            check(lib().dq_run_round_host(ctx.h, ptrs, d, C.c_void_p(hout.data_ptr()), C.byref(info), sptr))
        b.record(st)
        torch.cuda.synchronize()
        ems = a.elapsed_time(b) / k
        line["e2e"] = {"value": round(n * 4 * d / (ems * 1e-3) / 1e9, 3), "unit": UNIT, "ms_per_step": round(ems, 3),
                       "h2d_bytes_per_step": n * 4 * d, "d2h_bytes_per_step": 4 * d,
                       "api": "dq_run_round_host (C-ABI, pinned host buffers)"}
    if not args.no_cpu_baseline:
        def gpu_vnmse(sample):
            return dq.run_round([torch.from_numpy(w).cuda() for w in sample], cfg).vnmse
        line["cpu_baseline"] = cpu_baseline(hw, args.cpu_sample_d, args.budget, args.topology, args.sigma_log,
                                            gpu_vnmse)
    return line


# --------------------------------------------------------------------- N > 1
def bench_dist(args):
    import torch
    import torch.distributed as dist
    import paper_2602_08923_b200 as dq
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    d = args.d or (1 << 28)
    cfg = dq.PipelineConfig(n_workers=world, budget_bits=args.budget,
                            topology=dq.BUTTERFLY if args.topology == "butterfly" else dq.RING,
                            seed=dq.SharedSeed(1, 0))
    comm = dq.Communicator(cfg, rank, world)
    # this rank's worker gradient of the shared workload (the same arrays --impl reference reduces)
    x = torch.from_numpy(make_inputs(world, d, args.sigma_log, ranks=[rank])[0]).cuda()
    out = torch.empty_like(x)
    st = torch.cuda.current_stream()
    for _ in range(args.warmup):
        comm.allreduce(x, out, async_op=True)
    torch.cuda.synchronize()
    # accuracy vs exact fp32 sum (outside the timed region)
    truth = x.clone()
    dist.all_reduce(truth)
    err = float(((out.double() - truth.double()) ** 2).sum())
    ref = float((truth.double() ** 2).sum())
    # timed region without per-launch instrumentation (value), then the same K rounds
    # with CUDA events around every launch (per-kernel times, roofline)
    comm.ctx.profile(False)
    comm.ctx.read_profile(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(args.steps):
            comm.allreduce(x, out, async_op=True)
        e1.record(st)
        torch.cuda.synchronize()
        dist.barrier()
    launch_counts = comm.ctx.read_profile(reset=True)
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms)
    comm.ctx.profile(True)
    dist.barrier()
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(st)
    for _ in range(args.steps):
        comm.allreduce(x, out, async_op=True)
    p1.record(st)
    torch.cuda.synchronize()
    prof = comm.ctx.read_profile(reset=True)
    comm.ctx.profile(False)
    prof_ms = torch.tensor([p0.elapsed_time(p1) / args.steps], device="cuda")
    dist.all_reduce(prof_ms, op=dist.ReduceOp.MAX)
    prof_ms = float(prof_ms)
    # NCCL bf16 all-reduce baseline on the same d
    xb = x.to(torch.bfloat16)
    for _ in range(3):
        dist.all_reduce(xb)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(args.steps):
        dist.all_reduce(xb)
    b.record(st)
    torch.cuda.synchronize()
    nms = torch.tensor([a.elapsed_time(b) / args.steps], device="cuda")
    dist.all_reduce(nms, op=dist.ReduceOp.MAX)
    nms = float(nms)
    peak, pk = peaks()
    line = None
    if rank == 0:
        value = world * 4 * d / (ms * 1e-3) / 1e9
        launches = sum(p["launches"] for k, p in launch_counts.items() if k != "nccl")
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 in / u8 codes (bit-exact integer PRNG path)", "data": "synthetic",
            "config": {"workload": f"configs[2]: {args.topology} all-reduce over {world} B200, {d} fp32 entries "
                                   f"per rank, b={args.budget}, sigma_log={args.sigma_log}",
                       "global_batch": world, "entries_per_worker": d, "parallelism": f"dp{world}",
                       "l2": "inputs larger than L2"},
            "algbw_effective_gbs": round(4 * d / (ms * 1e-3) / 1e9, 3),
            "vnmse": err / ref if ref > 0 else 0.0,
            "nccl_bf16": {"ms": round(nms, 4), "effective_gbs": round(4 * d / (nms * 1e-3) / 1e9, 3),
                          "algbw_gbs": round(2 * d / (nms * 1e-3) / 1e9, 3),
                          "busbw_gbs": round(2 * d / (nms * 1e-3) / 1e9 * 2 * (world - 1) / world, 3)},
            "kernels": {k: {"launches": v["launches"], "ms_per_step": round(v["ms"] / args.steps, 4),
                            "GBps": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1)} for k, v in prof.items()},
            "kernels_region": {"steps": args.steps, "ms_per_step": round(prof_ms, 4),
                               "note": "second timed region, CUDA events around every launch"},
            "roofline": roofline_of(prof, peak, pk, traffic_ok=False), "gpu_launches": launches, "clocks": clk.summary(),
        }
    # e2e: pinned host -> device, all-reduce, device -> host
    if not args.no_e2e:
        hx = torch.empty(d, dtype=torch.float32, pin_memory=True)
        hx.copy_(x)
        hy = torch.empty(d, dtype=torch.float32, pin_memory=True)
        dx = torch.empty_like(x)
        k = max(3, args.steps // 4)
        for _ in range(2):
            dx.copy_(hx, non_blocking=True)
            comm.allreduce(dx, out, async_op=True)
            hy.copy_(out, non_blocking=True)
        torch.cuda.synchronize()
        dist.barrier()
        a.record(st)
        for _ in range(k):
            dx.copy_(hx, non_blocking=True)
            comm.allreduce(dx, out, async_op=True)
            hy.copy_(out, non_blocking=True)
        b.record(st)
        torch.cuda.synchronize()
        ems = torch.tensor([a.elapsed_time(b) / k], device="cuda")
        dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        if rank == 0:
            ems = float(ems)
            line["e2e"] = {"value": round(world * 4 * d / (ems * 1e-3) / 1e9, 3), "unit": UNIT,
                           "ms_per_step": round(ems, 3), "h2d_bytes_per_step": 4 * d, "d2h_bytes_per_step": 4 * d,
                           "api": "Communicator.allreduce (dq_allreduce C-ABI) with pinned host copies"}
    dist.barrier()
    dist.destroy_process_group()
    return line


def bench_reference(args):
    """--impl reference: the reference's CPU run_round (oracle/_ref) on the host cores, rank 0
    only, on the SAME inputs as our arm (make_inputs).  Every step is the full workload when
    the whole --steps/--warmup run fits in about five and a half minutes (the warm-up round measures
    it), else the first entries of every worker - stated in config and cpu_baseline."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    n = args.n_sim if args.gpus <= 1 else args.gpus
    d_full = args.d or ((1 << 26) if args.gpus <= 1 else (1 << 28))
    from oracle.oracle import Oracle, available
    kind = "reference" if available("reference") else "port"
    ora = Oracle(kind)
    threads = min(n, os.cpu_count() or 1) if kind == "reference" else 1
    cfg = ora.round_cfg(n, args.budget, args.topology, seed=1, threads=threads)
    steps = max(1, args.steps)
    total = steps + max(0, args.warmup)
    hw = make_inputs(n, d_full, args.sigma_log)
    dsamp = d_full
    # the reference holds ~10 copies of the inputs (grads, normalized, permuted, exact sum, ...)
    if n * d_full * 4 * 10 > 0.6 * _host_ram_bytes():
        dsamp = max(1 << 16, int(0.6 * _host_ram_bytes() / (n * 4 * 10)) // 256 * 256)
    t0 = time.perf_counter()
    res = ora.run_round([np.ascontiguousarray(w[:dsamp]) for w in hw], cfg)  # first warm-up round
    t1 = time.perf_counter() - t0
    if t1 * (total - 1) > 330.0:  # keep the run to a few minutes: a per-step prefix sample
        dsamp = max(1 << 16, int(dsamp * 330.0 / (t1 * max(total - 1, 1))) // 256 * 256)
    ws = [np.ascontiguousarray(w[:dsamp]) for w in hw]
    for _ in range(max(0, args.warmup) - 1):
        ora.run_round(ws, cfg)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        res = ora.run_round(ws, cfg)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    value = n * 4 * dsamp / t / 1e9
    full = dsamp == d_full
    sample = (f"run_round n={n} {args.topology} b={args.budget}, " +
              (f"the full workload ({d_full} entries per worker)" if full else
               f"the first {dsamp} of the {d_full} entries of every worker") +
              f" of the same inputs as our arm, median of {steps}")
    if args.gpus <= 1:
        config = {"workload": f"configs[1]: single-B200 simulated {args.topology} all-reduce round, "
                              f"{n} workers x {d_full} entries, b={args.budget}, sigma_log={args.sigma_log}",
                  "global_batch": n, "entries_per_worker": dsamp, "parallelism": f"sim{n}",
                  "l2": "inputs larger than L2 (>= 1 GiB resident)"}
    else:
        config = {"workload": f"configs[2]: {args.topology} all-reduce over {n} B200, {d_full} fp32 entries "
                              f"per rank, b={args.budget}, sigma_log={args.sigma_log}",
                  "global_batch": n, "entries_per_worker": dsamp, "parallelism": f"dp{n}", "l2": "inputs larger than L2"}
    return {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config, "reference_host_threads": threads,
            "vnmse": res["vnmse"],
            "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": threads, "kind": kind,
                             "sample": sample},
            "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _host_ram_bytes():
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        return 64 << 30


def main():
    args = parse()
    # stdout carries only the JSON line: libraries that print to fd 1 directly (NCCL's
    # version banner under NCCL_DEBUG=VERSION) are sent to stderr for the run.
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    if args.impl == "reference":
        line = bench_reference(args)
    elif int(os.environ.get("WORLD_SIZE", "1")) > 1:
        line = bench_dist(args)
    else:
        line = bench_sim(args)
    if line is not None:
        sys.stdout.flush()
        os.write(json_fd, (json.dumps(line) + "\n").encode())


if __name__ == "__main__":
    main()
