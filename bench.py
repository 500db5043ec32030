#!/usr/bin/env python3
"""bench.py -- headline benchmark of the B200 partition solver.

Workload (BASELINE.json configs[1]): scalar tridiagonal fp64, n = 2^26,
p = 65536 partitions, off-diagonals U[-1,1], diagonal 4+U[0,1], RHS U[-1,1],
seeded SplitMix64 (generated on the device, bit-identical to the CPU oracle).
One step = parallel_factor + solve (the reference's two entry points,
proj/include/parsol/parfact.hpp:52-60) with device-resident inputs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun, one process per GPU): every rank solves its own
independent system of the same size (weak scaling, no data-path collective);
timing is max over ranks of device-event time.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref: the unmodified proj/src compiled here) with all host threads on
a bounded sample of the same workload; only rank 0 runs it.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "solved unknowns/s and % of HBM roofline, fp64 partitioned tridiagonal n=2^26"
UNIT = "unknowns/s"
N_CFG1 = 1 << 26
P_CFG1 = 65536


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref or the oracle port) -- baseline, never the product
# BASELINE.md §3 / SURVEY.md §8(d): all host threads, 1 warm-up + median of 5,
# parallel_factor(A, p_cpu, Lu) + solve with p_cpu = the config's own p for
# config 0 and p_cpu = #threads for configs 1-3 (the reference's dense reduced
# solve needs a dim^2 matrix: 34 GB at config 1's p = 65536); config 4 at
# N = 2^12, p = 64 (the reference's Babd entry access is O(block row), so full
# N takes hours); plus solve_sequential on one thread.
# ---------------------------------------------------------------------------
CPU_CFG = {0: (1 << 20, 1024), 1: (N_CFG1, None), 2: (1 << 20, None), 3: (1 << 24, None), 4: (1 << 12, 64)}


def run_cpu_reference(cfg: int, reps: int = 5, warmup: int = 1, sequential: bool = False):
    import oracle as O

    threads = os.cpu_count() or 1
    size, p = CPU_CFG[cfg]
    A, f = O.generate_config(cfg, size, cfg + 1)
    n = A.n
    times = []
    if O.ref_available():
        kind = "reference"
        cores = 1 if sequential else threads
        O.ref_set_threads(cores)
        p = p or threads
        R = O.RefMatrix(A)
        for it in range(warmup + reps):
            t0 = time.perf_counter()
            if sequential:
                R.solve_sequential(f)
            else:
                F = R.factor(p)
                F.solve(f)
                del F
            if it >= warmup:
                times.append(time.perf_counter() - t0)
        O.ref_set_threads(threads)
    else:  # oracle port (single thread)
        kind, cores, p = "port", 1, p or 64
        for it in range(warmup + reps):
            t0 = time.perf_counter()
            if sequential:
                O.solve_sequential(A, f)
            else:
                O.parallel_solve(A, p, f)
            if it >= warmup:
                times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    what = "solve_sequential (1 thread)" if sequential else f"parallel_factor+solve (Strategy::Lu), p={p}"
    sample = (f"cfg{cfg}, n={n}, {what}, {warmup} warm-up + median of {reps}; "
              f"host: {cpu_model()}, {cores} thread(s)")
    return dict(value=n / med, unit=UNIT, cores=cores, kind=kind, sample=sample, seconds_per_sample=med, n=n,
                p=None if sequential else p), times


def impl_reference(args, rank, world):
    if rank != 0:
        return 0
    steps = max(1, args.steps)
    info, times = run_cpu_reference(1, steps, warmup=max(0, min(args.warmup, 1)))
    ms = 1e3 * sum(times) / len(times)
    line = {
        "metric": METRIC, "value": info["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64, BASELINE cfg1 distribution)",
        "impl": "reference",
        "config": {"workload": "cfg1: tridiagonal fp64 n=2^26, factor+solve per step (the unmodified reference, "
                               "oracle/_ref, all host threads)",
                   "n": info["n"], "p": info["p"], "threads": info["cores"],
                   "p_note": "p = #threads: the reference's reduced solve is a dense dim^2 LU (34 GB at the "
                             "config's p = 65536, SURVEY.md §0.3); p is the paper's processor count"},
        "cpu_baseline": {k: info[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": info["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# multi-rank aggregation: max over ranks of the device-timed total, sum of the
# units all ranks processed (weak scaling: each rank owns its own system)
# ---------------------------------------------------------------------------
def aggregate(ms_total_local, units_local, steps, dist=None, device="cpu"):
    import torch
    t = torch.tensor([ms_total_local, float(units_local)], dtype=torch.float64, device=device)
    if dist is not None:
        mx = t[:1].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t[1:].clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_total, units = float(mx.item()), float(sm.item())
    else:
        ms_total, units = float(t[0].item()), float(t[1].item())
    ms_step = ms_total / steps
    return ms_step, units, units / (ms_step / 1e3)


# ---------------------------------------------------------------------------
# our GPU path
# ---------------------------------------------------------------------------
OTHER = [(0, 1 << 20, 1024), (2, 1 << 20, 16384), (3, 1 << 24, 32768), (4, 1 << 18, 4096)]


def other_configs(psg, torch, peak, dev, steps=20):
    """The other BASELINE configs through the same production path (one handle,
    refactor + async certified solve per step, device-timed), reported beside
    the headline -- informative, outside its timed region."""
    out = []
    for cfg, size, p in OTHER:
        A, f = psg.generate_config(cfg, size, cfg + 1, device=dev)
        x = torch.empty_like(f)
        H = psg.parallel_factor(A, p, psg.Strategy.Lu)
        for _ in range(2):
            H.refactor(A)
            H.solve_async(f, x)
        H.sync()
        torch.cuda.synchronize()
        st = psg.SolveStats()
        corner = 0 if A.corner is None else A.corner.numel()
        in_bytes = (A.data.numel() + corner + 2 * A.n) * 8
        if in_bytes < 4 * (126 << 20):  # fits in L2: flush it before every step, time each step alone
            flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            for e0, e1 in evs:
                flush.random_(0, 255)
                e0.record()
                H.refactor(A)
                H.solve_async(f, x)
                e1.record()
                H.sync(st)  # certificate checked (and repaired) before the next step's flush
            torch.cuda.synchronize()
            ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / steps
            l2 = ("L2 flushed (512 MB write) before each step; each step's device time (refactor + certified "
                  "solve incl. its certificate kernel) timed alone")
            del flush
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):  # no per-phase events inside the bracket (as the headline)
                H.refactor(A)
                H.solve_async(f, x)
            H.sync(st)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            l2 = "inputs larger than L2; back-to-back steps"
        min_bytes = in_bytes
        out.append({"cfg": cfg, "n": A.n, "p": p, "ms_per_step": ms, "unknowns_per_s": A.n / (ms / 1e3),
                    "hbm_roofline_frac": min_bytes / (ms / 1e3) / 1e9 / peak, "min_bytes": min_bytes,
                    "residual": psg.residual(A, x, f), "certificate": st.certificate, "l2": l2,
                    "path": "speculative" if st.speculative else "exact", "fallbacks": st.fallbacks})
        H.close()
        del A, f, x
    return out


def impl_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_0912_3678_b200 as psg

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n, p = N_CFG1, P_CFG1
    seed = 2 + rank
    A, f = psg.generate_config(1, n, seed, device=dev)
    x = torch.empty_like(f)
    torch.cuda.synchronize()

    # drop-in path: parallel_factor + blocking solve per step (a new handle each step)
    def dropin_step(stats):
        F = psg.parallel_factor(A, p, psg.Strategy.Lu)
        psg.solve(F, f, stats, x=x)
        fl, sl = F.launches()
        F.close()
        return fl + sl

    # production path: one handle, per step refactor (new values, same structure)
    # + asynchronous certified solve; failed certificates are repaired in sync()
    H = psg.parallel_factor(A, p, psg.Strategy.Lu)

    def async_step(timing=False):
        H.refactor(A)
        H.solve_async(f, x, timing=timing)
        fl, sl = H.launches()
        return fl + sl

    for _ in range(args.warmup):
        dropin_step(psg.SolveStats())
        async_step()
    H.sync()
    torch.cuda.synchronize()

    clocks = Clocks(local_rank) if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    launches = 0
    for _ in range(args.steps):
        launches += async_step()
    st0 = psg.SolveStats()
    H.sync(st0)                # certificates of every step checked (and repaired) inside the bracket
    ev1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_total = ev0.elapsed_time(ev1)
    clk = clocks.stop() if clocks else None

    # phase breakdown (roofline of K3): the same loop with per-phase events,
    # timed separately so the events do not sit inside the headline bracket
    torch.cuda.synchronize()
    for _ in range(args.steps):
        async_step(timing=True)
    st = psg.SolveStats()
    H.sync(st)
    torch.cuda.synchronize()

    # the drop-in path, same bracket discipline (reported beside the headline)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev2.record()
    dst = []
    for _ in range(args.steps):
        s1 = psg.SolveStats()
        dropin_step(s1)
        dst.append(s1)
    ev3.record()
    torch.cuda.synchronize()
    dropin_ms = ev2.elapsed_time(ev3) / args.steps

    ms_step, units, _ = aggregate(ms_total, n, args.steps, dist if world > 1 else None, dev)

    # correctness of the timed run (outside the timed region)
    res = psg.residual(A, x, f)
    cert = max(st0.certificate, st.certificate, max(s1.certificate for s1 in dst))
    spec = st0.speculative == 1 and st0.fallbacks == 0 and st.fallbacks == 0

    if rank != 0:
        return 0

    peak, peak_src = peaks()
    min_bytes = (5 * n - 2) * 8  # every entry of A and f read once, x written once
    k3_s = st.phase3_seconds / args.steps
    k3_bytes = min_bytes  # K3 reads a,b,c,f of every row and writes x
    achieved = k3_bytes / k3_s / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "k3_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as fh:
                traffic = json.load(fh).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    phases = {
        "factor_ms": 1e3 * statistics.mean(s1.factor_seconds for s1 in dst),
        "phase1_ms": 1e3 * st.phase1_seconds / args.steps,
        "phase2_ms": 1e3 * st.phase2_seconds / args.steps,
        "phase3_ms": 1e3 * k3_s,
    }

    # ---- end-to-end through the C ABI with host (pinned) buffers ----------
    e2e = None
    if not args.no_e2e:
        hd = torch.empty(A.data.numel(), dtype=torch.float64, pin_memory=True)
        hf = torch.empty(n, dtype=torch.float64, pin_memory=True)
        hx = torch.empty(n, dtype=torch.float64, pin_memory=True)
        hd.copy_(A.data)
        hf.copy_(f)
        HA = psg.StructuredMatrix(A.kind, A.n, A.m, A.s, A.r, hd)  # host descriptor (copied by psg_factor)

        def e2e_step():
            F = psg.parallel_factor(HA, p, psg.Strategy.Lu)
            psg.solve(F, hf, None, x=hx)  # H2D of f, D2H of x inside
            F.close()

        e2e_step()
        torch.cuda.synchronize()
        ne = max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        for _ in range(ne):
            e2e_step()
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / ne
        e2e = {"value": n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(hd.numel() * 8 + n * 8),
               "d2h_bytes_per_step": int(n * 8), "ms_per_step": 1e3 * e2e_s, "steps": ne,
               "path": "psg_factor(host A) + psg_solve(host f -> host x), pinned buffers"}
        assert torch.allclose(hx, x.cpu(), rtol=0, atol=1e-12)

    other = None if args.no_other_configs else other_configs(psg, torch, peak, dev)

    cpu = None
    if not args.no_cpu_baseline:
        def cpu_fig(cfg, sequential=False):
            try:
                d, _ = run_cpu_reference(cfg, sequential=sequential)
                d.pop("seconds_per_sample", None)
                return d
            except Exception as e:  # baseline is informative only
                return {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable", "sample": str(e)}

        cpu = cpu_fig(1)
        cpu["single_core_solve_sequential"] = cpu_fig(1, sequential=True)
        for oc in other or []:
            oc["cpu_baseline"] = cpu_fig(oc["cfg"])

    value = units / (ms_step / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64 on device, BASELINE cfg1 distribution; seed 2+rank)",
        "config": {"workload": "cfg1: tridiagonal fp64 n=2^26, p=65536, factor+solve per step "
                               "(psg_refactor + psg_solve_async, certificates checked in psg_sync inside the "
                               "timed region)",
                   "n": n, "p": p, "strategy": "Lu", "per_gpu_n": n,
                   "parallelism": f"independent system per GPU x{world}",
                   "l2": "inputs larger than L2 (2.15 GB in, 0.54 GB out vs 126 MB L2); no flush"},
        "hbm_roofline_frac": (min_bytes / (ms_step / 1e3) / 1e9) / peak,
        "roofline": {"bound": "hbm", "kernel": "tri_segment_solve_kernel<33> (K3, incl. certificate kernel)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": k3_bytes},
        "phases": phases,
        "dropin": {"ms_per_step": dropin_ms, "value": world * n / (dropin_ms / 1e3),
                   "path": "parallel_factor (new handle) + blocking solve per step"},
        "certificate_max": cert, "speculative": spec, "residual": res,
        "gpu_launches": launches,
        "build": psg.lib().psg_version().decode(),
        "other_configs": other,
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return impl_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return impl_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
