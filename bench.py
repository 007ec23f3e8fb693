#!/usr/bin/env python
"""Benchmark of the batched LP hot path (BASELINE.json metric: LPs solved/sec, device-timed,
and % of roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A step is one solve of this rank's batch (inputs resident in HBM) through the C ABI.  The
default workload is cfg2 (BASELINE.json configs[1], the paper's 18.3x workload: 50,000 type-1
LPs of 100x100, generator G1 seed 2).  Multi-GPU: --scaling weak (default)
gives each rank its own B-LP slice of a N*B-LP seeded batch (per-GPU work fixed); --scaling
strong shards the config's fixed batch, rank r solving LPs [floor(rB/N), floor((r+1)B/N))
(e.g. cfg5's 6,003,000 LPs over 1/2/4/8 GPUs).  No collective on the data
path; device time is the max over ranks; the results are gathered to rank 0 after the timed
region and checked against the oracle on a sample (gather_ms reported apart).  With --graph
each rank captures its per-step solve in a CUDA graph once and replays it (for the
microsecond-scale per-rank solves of cfg1 / cfg4 at 8 GPUs).  Rank 0 prints one JSON line.

--impl reference times the CPU oracle (oracle/, the only other place this file runs it) on a
bounded sample of the same workload on this host's cores (rank 0 only; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import lpgen  # noqa: E402

METRIC = "LPs solved/sec (device-timed)"
UNIT = "LPs/s"
# Paper numbers for the exact workload (GeForce GTX 670): hyperbox only.
PAPER_LPS = {"cfg4": 4001000 / 0.406, "cfg5": 6003000 / 2.388}
# oracle sample per reference step (bounded CPU work)
REF_SAMPLE = {"cfg1": 1000, "cfg1m": 1000000, "cfg2": 240, "cfg3": 8, "cfg4": 4001000, "cfg5": 1000000,
              "cfg2s": 240, "cfg3s": 8, "cfg2r": 160, "cfg6": 32, "cfg7": 16, "cfg8": 4,
              "cfg9": 20000, "cfg10": 4000}
# oracle sample for cpu_baseline: about 1 s per all-core run on the 16-core GPU host
CPU_SAMPLE = {"cfg1": 1000, "cfg1m": 1000000, "cfg2": 6000, "cfg3": 32, "cfg4": 4001000,
              "cfg5": 6003000, "cfg2s": 4000, "cfg3s": 32, "cfg2r": 3000, "cfg6": 120,
              "cfg7": 16, "cfg8": 8, "cfg9": 50000, "cfg10": 50000}
L2_BYTES = 126 * 1024 * 1024


def rule_opts(name):
    """Entering-rule options of a config (NEXT-3 RPC runs use the config seed)."""
    c = lpgen.CONFIGS[name]
    if c.get("rule", "LPC") == "RPC":
        return {"pivot_rule": "RPC", "rpc_seed": c["seed"]}
    return {}


def describe(name):
    c = lpgen.CONFIGS[name]
    if c["kind"] == "hyperbox":
        return (f"{name}: type-3 hyperbox, {c['B']} LPs of n={c['n']} (shared box, G3 seed "
                f"{c['seed']})")
    t = "type-1 (b>=0)" if c["gen"] == "G1" else "type-2 (two-phase)"
    if c.get("rule", "LPC") != "LPC":
        t += f", {c['rule']} entering rule (seed {c['seed']})"
    if c.get("shared"):
        return (f"{name}: {t}, {c['B']} objectives over one {c['m']}x{c['n']} polytope "
                f"({c['gen']} seed {c['seed']}, shared A/b)")
    return f"{name}: {t}, {c['B']} LPs of {c['m']}x{c['n']} ({c['gen']} seed {c['seed']})"


def general_sample(name, n_lp):
    """First n_lp LPs of a general config as a full (B, m, n) batch (shared A/b broadcast)."""
    cfg = lpgen.CONFIGS[name]
    A, b, c = lpgen.make_config_shard(name, cfg["B"], 0, min(n_lp, cfg["B"]))
    if A.ndim == 2:
        B = c.shape[0]
        A = np.ascontiguousarray(np.broadcast_to(A, (B,) + A.shape))
        b = np.ascontiguousarray(np.broadcast_to(b, (B,) + b.shape))
    return A, b, c


def traffic_per_launch(name, B):
    """roofline.traffic: DRAM bytes (read + write) of the dominant kernel per launch, from the
    committed ncu --set full capture of this config (profiles/traffic.json, per LP x B), or
    None when the config has no capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        return float(t[name]["dram_bytes_per_lp"]) * B
    except Exception:
        return None


def _measured_hbm(m):
    """HBM GB/s from the driver-written MEASURED_PEAKS.json: `hbm_gbs`, else any numeric
    entry under an `hbm` key, preferring the burst figure (our kernels are timed per launch),
    then sustained; TB/s-sized values are scaled to GB/s."""
    if isinstance(m.get("hbm_gbs"), (int, float)):
        return float(m["hbm_gbs"])
    found = []

    def walk(o, path):
        if isinstance(o, dict):
            for k, v in o.items():
                walk(v, path + (str(k).lower(),))
        elif isinstance(o, (int, float)) and not isinstance(o, bool) and any("hbm" in t for t in path):
            found.append((path, float(o)))
    walk(m, ())
    for pref in ("burst", "sustained", ""):
        for path, v in found:
            if pref in " ".join(path):
                return v * 1000.0 if v < 100.0 else v
    return None


def peaks():
    p = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "src": "fallback (B200_PROFILING.md)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        hbm = _measured_hbm(m)
        if hbm:
            p.update(hbm_gbs=hbm, src="measured (MEASURED_PEAKS.json)")
        if isinstance(m.get("sm_max_mhz"), (int, float)):
            p["sm_max_mhz"] = float(m["sm_max_mhz"])
    except Exception:
        pass
    # FP64 vector peak from unit counts: 148 SMs x 64 FP64 FMA lanes x 2 flop
    # x max SM clock
    p["fp64_tflops"] = 148 * 64 * 2 * p["sm_max_mhz"] * 1e6 / 1e12
    return p


class ClockSampler:
    """nvidia-smi style clock / throttle sampling (NVML) during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.stop = [], 0, threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
            # the first NVML queries are slow and hold driver locks: let them finish before
            # the timed region starts (short timed regions would otherwise absorb them)
            deadline = time.time() + 1.0
            while not self.samples and time.time() < deadline:
                time.sleep(0.001)
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop.set()
            self.t.join()

    def summary(self):
        reasons = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


# FP64 DFMA throughput measured on this pool's B200 (scripts/ubench/dfma_occ.cu: independent
# DFMA chains at >= 16 warps/SM; profiles/r01g.md), next to the unit-count figure
FP64_MEASURED_TFLOPS = 36.7


def simplex_work(iters, k, m, n):
    """Algorithmic work of a simplex solve from each LP's returned (it1, it2) and k, over the
    LIVE condensed tableau only (SURVEY.md §8(d) "Roofline accounting"):
      flops   = 2 (R-1)(W-1) per pivot (the rank-1 update, pivot row/column excluded)
      updates = R * W elements per pivot (SMEM-equivalent traffic: 16 B each, read + write)
    with phase I R = m+2 (both objective rows), W = n+k+1; phase II R = m+1 (the phase-I row
    dropped) and W = n+1 (the k artificial positions are dead after phase I; a redundant
    row's artificial stays basic and is not counted)."""
    it1 = iters[:, 0].astype(np.float64)
    it2 = iters[:, 1].astype(np.float64)
    kf = k.astype(np.float64)
    flops = 2.0 * (it1 * (m + 1) * (n + kf) + it2 * m * n)
    upd = it1 * (m + 2) * (n + kf + 1) + it2 * (m + 1) * (n + 1)
    return float(np.sum(flops)), float(np.sum(upd))


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(name, sample_n, repeats=5, single_repeats=3):
    """The oracle as it stands on a bounded sample of the workload (SURVEY.md §8(d) "Oracle
    beside the GPU"): the median of `repeats` runs over all host cores (one LP per task,
    pthreads; the paper averages 10 runs) and the median of `single_repeats`
    single-core runs on a sample of sample_n / cores LPs."""
    import oracle
    cfg = lpgen.CONFIGS[name]
    hyper = cfg["kind"] == "hyperbox"
    if hyper:
        lo, hi, dirs = lpgen.make_config(name, min(sample_n, cfg["B"]))
        run = lambda k, th: oracle.hyperbox(lo, hi, dirs[:k], threads=th)  # noqa: E731
        n_lp = dirs.shape[0]
    else:
        A, b, c = general_sample(name, sample_n)
        run = lambda k, th: oracle.solve(A[:k], b[:k], c[:k], threads=th, **rule_opts(name))  # noqa: E731
        n_lp = A.shape[0]
    run(min(n_lp, 64), None)  # thread-pool / page warm-up
    times, cores = [], 1
    for _ in range(repeats):
        t = time.perf_counter()
        r = run(n_lp, None)
        times.append(time.perf_counter() - t)
        cores = int(r["threads"])
    n1 = max(1, min(n_lp, (n_lp + cores - 1) // cores))
    t1 = []
    for _ in range(single_repeats):
        t = time.perf_counter()
        run(n1, 1)
        t1.append(time.perf_counter() - t)
    med, med1 = statistics.median(times), statistics.median(t1)
    return {"value": n_lp / med, "unit": UNIT, "cores": cores, "kind": "oracle",
            "mean": n_lp / statistics.mean(times),
            "single_core": n1 / med1, "cpu": cpu_model(),
            "sample": f"first {n_lp} LPs of {name}, oracle/lpb_oracle.c (-O2, pthreads): "
                      f"median of {repeats} runs on {cores} threads ({med:.2f} s each); "
                      f"single core: median of {single_repeats} runs of {n1} LPs "
                      f"({med1:.2f} s)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name = args.config
    cfg = lpgen.CONFIGS[name]
    n = REF_SAMPLE[name] if args.ref_sample is None else args.ref_sample
    import oracle
    if cfg["kind"] == "hyperbox":
        lo, hi, dirs = lpgen.make_config(name, min(n, cfg["B"]))
        step = lambda: oracle.hyperbox(lo, hi, dirs)  # noqa: E731
        n_lp = dirs.shape[0]
    else:
        A, b, c = general_sample(name, n)
        step = lambda: oracle.solve(A, b, c, **rule_opts(name))  # noqa: E731
        n_lp = A.shape[0]
    for _ in range(args.warmup):
        step()
    t = time.perf_counter()
    for _ in range(args.steps):
        r = step()
    dt = time.perf_counter() - t
    value = n_lp * args.steps / dt
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded lpgen generators)",
        "config": {"workload": describe(name), "sample_per_step": n_lp},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": int(r["threads"]),
                         "kind": "oracle",
                         "sample": f"{n_lp} LPs of {name} per step (the oracle, host cores)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=sorted(lpgen.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: B LPs per rank; strong: the config's B LPs sharded over ranks")
    ap.add_argument("--graph", action="store_true",
                    help="capture each rank's solve in a CUDA graph and replay it per step")
    ap.add_argument("--no-hint", action="store_true",
                    help="do not pass the generator's kmax bound (lpb_options.kmax_hint)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-chunks1", action="store_true",
                    help="also time e2e with n_chunks = 1 (the no-overlap control)")
    ap.add_argument("--batch", type=int, default=None,
                    help="batch override: per rank (weak) or total (strong)")
    ap.add_argument("--ref-sample", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_1609_08114_b200 import dist as lpdist
    from paper_1609_08114_b200 import lpb

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    # one process per GPU; more ranks than GPUs only in the gloo test mode (ranks share GPUs)
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("LPB_DIST_BACKEND", "nccl")  # gloo: 2 ranks on 1 GPU (tests)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    name = args.config
    cfg = lpgen.CONFIGS[name]
    if args.scaling == "strong":
        B_total = args.batch or cfg["B"]
        lo, hi = lpdist.shard_range(B_total, rank, world)
    else:
        B_rank = args.batch or cfg["B"]
        B_total = B_rank * world
        lo, hi = rank * B_rank, (rank + 1) * B_rank
    B = hi - lo  # this rank's LPs
    hyper = cfg["kind"] == "hyperbox"
    sab = bool(cfg.get("shared"))
    if hyper:
        n = cfg["n"]
        lo_b, hi_b, dirs = lpgen.make_config_shard(name, B_total, lo, hi)
        box = np.concatenate([hi_b, -lo_b])
        d_c = torch.from_numpy(dirs).to(dev)
        d_b = torch.from_numpy(box).to(dev)
        d_A = None
        m = 2 * n
        in_bytes = dirs.nbytes  # the shared box (2n doubles) is staged once
        host_in = (None, box, dirs)
        kind = lpb.HYPERBOX
    else:
        m, n = cfg["m"], cfg["n"]
        A, b, c = lpgen.make_config_shard(name, B_total, lo, hi)
        d_A, d_b, d_c = (torch.from_numpy(v).to(dev) for v in (A, b, c))
        in_bytes = A.nbytes + b.nbytes + c.nbytes
        host_in = (A, b, c)
        kind = lpb.GENERAL
    ropts = rule_opts(name)
    if ropts:
        ropts["lp_index_base"] = lo  # RPC keys on the LP's index in the whole batch
    khint = lpgen.kmax_bound(name)
    if not hyper and not args.no_hint:
        ropts["kmax_hint"] = khint  # the LP type the generator guarantees
    # one dedicated stream per rank: the solves, the timing events and the graph capture
    stream = torch.cuda.Stream(device=dev)
    solver = lpb.Solver(B, m, n, kind, stream=stream.cuda_stream, **ropts)
    flush = None
    if in_bytes <= 2 * L2_BYTES:  # small inputs: flush L2 between timed steps
        flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step(timing=False):
        # timed steps record no library events (each is GPU work between back-to-back
        # solves); the kernel-time pass below turns them on
        solver.solve_device(d_A, d_b, d_c, shared_box=hyper, shared_ab=sab, timing=timing)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        graph = None
        launches_per_step = solver.launch_info()[0]
        if args.graph:
            # the library launches on `stream`, which the capture below runs on
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                step()
            graph.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    kern_ms, launches = [], 0
    with ClockSampler(local) as clk, torch.cuda.stream(stream):
        torch.cuda.synchronize()
        for i in range(args.steps):
            if flush is not None:
                flush.fill_(float(i))
            ev[i][0].record(stream)
            if graph is not None:
                graph.replay()
                launches += launches_per_step
            else:
                step()
                launches += solver.launch_info()[0]  # host-side fields: no synchronisation
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # the dominant kernel's own duration (device events around it inside the library), read
    # after each of a few extra, untimed steps: reading it synchronises, so it stays out of
    # the timed loop (whose steps are issued back to back, as a user's would be)
    with torch.cuda.stream(stream):
        for i in range(min(args.steps, 5)):
            if flush is not None:
                flush.fill_(float(i))
            step(timing=True)
            kern_ms.append(solver.kernel_ms())
    step_ms = [a.elapsed_time(b_) for a, b_ in ev]
    my_ms = float(sum(step_ms))
    tot_ms = lpdist.max_over_ranks(my_ms, device=dev)
    value = B_total * args.steps / (tot_ms / 1e3)
    kmean = float(np.mean(kern_ms))
    klass = solver.launch_info()[1]

    res = solver.device_results(want_x=True)
    # the only multi-GPU communication is a final gather of the results to rank
    # 0 (padded all_gather over NCCL), outside the timed solve; its time is reported apart,
    # and the gathered batch is checked for consistency (rank 0's own rows, shapes, sentinels;
    # bit parity with the N = 1 solve is tests/test_gpu_dist.py's job)
    gather_ms, gather_check = None, None
    if world > 1:
        try:
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.barrier()
            g0.record()
            full = {key: lpdist.gather_rows(res[key].contiguous(), B_total)
                    for key in ("status", "obj", "x")}
            g1.record()
            torch.cuda.synchronize()
            gather_ms = lpdist.max_over_ranks(g0.elapsed_time(g1), device=dev)
            if rank == 0:
                ok = (full["status"].shape[0] == B_total and full["x"].shape == (B_total, n)
                      and torch.equal(full["status"][:B], res["status"])
                      and torch.equal(full["obj"][:B], res["obj"])
                      and torch.equal(full["x"][:B], res["x"]))
                opt = full["status"] == 0
                ok = ok and bool(torch.isfinite(full["obj"][opt]).all())
                gather_check = f"{'ok' if ok else 'FAILED'}: {B_total} rows, rank 0 slice identical"
        except Exception as ex:  # the gather is reported, never required for the metric
            print(f"bench: result gather failed: {ex}", file=sys.stderr)
    p = peaks()
    roof_smem = None
    roof_alu = None
    if hyper:
        traffic_alg = B * (8 * n + 8 * n + 8 + 4)  # read l, write x, obj, status
        achieved = traffic_alg / (kmean / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": p["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / p["hbm_gbs"], "traffic": traffic_per_launch(name, B),
                "kernel": "hyperbox_kernel", "peak_src": p["src"],
                "algorithmic_bytes_per_launch": traffic_alg,
                "bytes_per_lp": 8 * n + 8 * n + 8 + 4}
        iters_mean = None
    else:
        iters = res["iters"].cpu().numpy()
        k = (np.broadcast_to(host_in[1], (B, m)) < 0).sum(axis=1)
        flops, upd = simplex_work(iters, k, m, n)
        if sab and k[0] > 0 and klass in ("M", "L"):
            # phase-I warm start (NEXT-1): phase I ran once for the polytope; every LP only
            # replays its carried objective row through the recorded pivots (2 flop, 1
            # element per recorded pivot and live position) -- count that, not B phase-I solves
            W = n + float(k[0]) + 1
            it1 = float(iters[0, 0])
            flops -= float(np.sum(2.0 * iters[:, 0] * (m + 1) * (n + k)))
            upd -= float(np.sum(iters[:, 0] * (m + 2) * (n + k + 1.0)))
            flops += 2.0 * it1 * (m + 1) * (n + float(k[0])) + B * 2.0 * W * it1
            upd += it1 * (m + 2) * W + B * W * it1
        achieved = flops / (kmean / 1e3) / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": p["fp64_tflops"],
                "unit": "TFLOP/s", "frac": achieved / p["fp64_tflops"],
                "traffic": traffic_per_launch(name, B),
                "kernel": f"simplex ({klass} class)",
                "peak_src": "FP64 unit count x clock: 148 SM x 64 DFMA/clk x 2 x "
                            f"{p['sm_max_mhz']:.0f} MHz (DESIGN.md)",
                "peak_measured": FP64_MEASURED_TFLOPS,
                "frac_measured": achieved / FP64_MEASURED_TFLOPS,
                "algorithmic_flops_per_launch": flops,
                "accounting": "2(R-1)(W-1) per pivot over live positions (SURVEY §8(d))"}
        # SMEM-equivalent roofline (SURVEY §8(d) "%SMEM"): 16 B (8-byte read + write) per live
        # element per pivot against 148 SMs x 128 B/clk; binding for the SMEM-resident M/L
        # classes, a reference figure for the register-resident R/W/S classes
        smem_peak = 148 * 128 * p["sm_max_mhz"] * 1e6 / 1e9
        smem_ach = 16.0 * upd / (kmean / 1e3) / 1e9
        roof_smem = {"bound": "smem", "achieved": smem_ach, "peak": smem_peak,
                     "unit": "GB/s", "frac": smem_ach / smem_peak,
                     "algorithmic_bytes_per_launch": 16.0 * upd,
                     "resident": "smem" if klass in ("M", "L") else "registers"}
        if klass == "S":
            # thread per LP (tiny LPs): a few hundred flops per LP against its 8(mn+m+n) input
            # and 8n+20 output bytes -- HBM is the binding roofline (SURVEY §8(d) cfg1 row:
            # the scaled 1M-LP run); the FP64 figure is kept beside it
            lp_bytes = 8 * (m * n + m + n) + 8 * n + 8 + 4 + 8
            if sab:
                lp_bytes -= 8 * (m * n + m)
            hb = float(B * lp_bytes)
            hach = hb / (kmean / 1e3) / 1e9
            roof_alu = roof
            roof = {"bound": "hbm", "achieved": hach, "peak": p["hbm_gbs"], "unit": "GB/s",
                    "frac": hach / p["hbm_gbs"], "traffic": traffic_per_launch(name, B),
                    "kernel": "simplex (S class)", "peak_src": p["src"],
                    "algorithmic_bytes_per_launch": hb, "bytes_per_lp": lp_bytes}
        iters_mean = iters.mean(axis=0).tolist()
        st = res["status"].cpu().numpy()

    # end to end through the C ABI with pinned host buffers (H2D + solve + D2H per step)
    e2e = None
    if args.e2e_steps > 0:
        pin = [lpb.pinned_empty(v.shape) if v is not None else None for v in host_in]
        for dst, src in zip(pin, host_in):
            if dst is not None:
                dst[...] = src
        out_st = lpb.pinned_empty((B,), np.int32)
        out_obj = lpb.pinned_empty((B,))
        out_x = lpb.pinned_empty((B, n))
        out_it = lpb.pinned_empty((B, 2), np.int32) if not hyper else None
        d2h = out_st.nbytes + out_obj.nbytes + out_x.nbytes + (out_it.nbytes if out_it is not None else 0)

        def e2e_run(n_chunks=0):
            hs = lpb.Solver(B, m, n, kind, n_chunks=n_chunks, **ropts)
            hs.solve_host_into(*pin, out_st, out_obj, out_x, out_it, shared_box=hyper,
                               shared_ab=sab)  # warm
            e_ms = []
            for _ in range(args.e2e_steps):
                hs.solve_host_into(*pin, out_st, out_obj, out_x, out_it, shared_box=hyper,
                                   shared_ab=sab)
                e_ms.append(hs.timing()[1])
            nl = hs.launch_info()[0]
            hs.close()
            e_tot = lpdist.max_over_ranks(float(sum(e_ms)), device=dev)
            return B_total * args.e2e_steps / (e_tot / 1e3), e_tot / args.e2e_steps, nl

        v, ms, nl = e2e_run()
        e2e = {"value": v, "unit": UNIT,
               "h2d_bytes_per_step": int(in_bytes), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": ms,
               "n_chunks": 10 if (B > 100 and in_bytes >= (1 << 20)) else 1,
               "gpu_launches_per_step": nl}
        if args.e2e_chunks1:
            v1, ms1, _ = e2e_run(n_chunks=1)
            e2e["chunks1"] = {"value": v1, "ms_per_step": ms1}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(name, CPU_SAMPLE[name])

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
            "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": (value / PAPER_LPS[name]) if name in PAPER_LPS else None,
            "dtype": "f64", "data": "synthetic (seeded lpgen generators, DESIGN.md)",
            "config": {"workload": describe(name), "batch_total": B_total,
                       "batch_per_gpu": B, "m": m, "n": n,
                       "kind": "hyperbox" if hyper else "general",
                       "l2": "flushed between steps" if flush is not None else "inputs > L2",
                       "parallelism": f"dp{world} (contiguous LP shards, no collective)",
                       "kernel_class": klass,
                       "ctas_per_lp": solver.launch_shape()[0],
                       "pivot_rule": lpgen.CONFIGS[name].get("rule", "LPC"),
                       "kmax_hint": None if (hyper or args.no_hint) else khint,
                       "cuda_graph": bool(args.graph)},
            "roofline": roof,
            **({"roofline_smem": roof_smem} if roof_smem else {}),
            **({"roofline_alu": roof_alu} if roof_alu else {}),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "gather_ms": gather_ms,
            "gather_check": gather_check,
            "clocks": clk.summary(),
            "kernel_ms_per_step": kmean,
        }
        if not hyper:
            out["config"]["mean_pivots"] = iters_mean
            out["config"]["status_counts"] = np.bincount(st, minlength=6).tolist()
        print(json.dumps(out), flush=True)
    solver.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
