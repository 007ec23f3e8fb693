#!/usr/bin/env python
"""Benchmark of the batched LP hot path (BASELINE.json metric: LPs solved/sec, device-timed,
and % of roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A step is one solve of this rank's batch (inputs resident in HBM) through the C ABI.  The
default workload is cfg2 (BASELINE.json configs[1], the paper's 18.3x workload: 50,000 type-1
LPs of 100x100, generator G1 seed 2).  Multi-GPU: each rank solves its own 50,000-LP slice of
a N*50,000-LP seeded batch (per-GPU work fixed: weak scaling); no collective on the data path,
device time is the max over ranks.  Rank 0 prints one JSON line.

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
CPU_SAMPLE = {"cfg1": 1000, "cfg1m": 1000000, "cfg2": 1200, "cfg3": 24, "cfg4": 4001000, "cfg5": 6003000,
              "cfg2s": 1200, "cfg3s": 24, "cfg2r": 800, "cfg6": 160, "cfg7": 32, "cfg8": 16,
              "cfg9": 50000, "cfg10": 20000}
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


def algorithmic_flops(iters, k, m, n):
    """2 flops per condensed-tableau element touched per pivot:
    phase I (R = m+2 rows, W = n+k+1 columns), phase II (R = m+1, W = n+k+1)."""
    it1 = iters[:, 0].astype(np.float64)
    it2 = iters[:, 1].astype(np.float64)
    W = n + k.astype(np.float64) + 1
    return float(np.sum(2.0 * W * (it1 * (m + 2) + it2 * (m + 1))))


def cpu_baseline(name, sample_n):
    """The oracle as it stands, multi-threaded over this host's cores, on a bounded sample."""
    import oracle
    cfg = lpgen.CONFIGS[name]
    if cfg["kind"] == "hyperbox":
        lo, hi, dirs = lpgen.make_config(name, min(sample_n, cfg["B"]))
        t = time.perf_counter()
        r = oracle.hyperbox(lo, hi, dirs)
        dt = time.perf_counter() - t
        n_lp = dirs.shape[0]
    else:
        A, b, c = general_sample(name, sample_n)
        t = time.perf_counter()
        r = oracle.solve(A, b, c, **rule_opts(name))
        dt = time.perf_counter() - t
        n_lp = A.shape[0]
    return {"value": n_lp / dt, "unit": UNIT, "cores": int(r["threads"]), "kind": "oracle",
            "sample": f"first {n_lp} LPs of {name}, oracle/lpb_oracle.c (-O2, pthreads), "
                      f"{dt:.2f} s wall"}


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
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--batch", type=int, default=None, help="per-rank batch override")
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
    if world > 1:
        backend = os.environ.get("LPB_DIST_BACKEND", "nccl")  # gloo: 2 ranks on 1 GPU (tests)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    name = args.config
    cfg = lpgen.CONFIGS[name]
    B = args.batch or cfg["B"]
    lo, hi = rank * B, (rank + 1) * B
    hyper = cfg["kind"] == "hyperbox"
    sab = bool(cfg.get("shared"))
    if hyper:
        n = cfg["n"]
        lo_b, hi_b, dirs = lpgen.make_config_shard(name, B * world, lo, hi)
        box = np.concatenate([hi_b, -lo_b])
        d_c = torch.from_numpy(dirs).cuda()
        d_b = torch.from_numpy(box).cuda()
        d_A = None
        m = 2 * n
        in_bytes = dirs.nbytes
        host_in = (None, box, dirs)
        kind = lpb.HYPERBOX
    else:
        m, n = cfg["m"], cfg["n"]
        A, b, c = lpgen.make_config_shard(name, B * world, lo, hi)
        d_A, d_b, d_c = (torch.from_numpy(v).cuda() for v in (A, b, c))
        in_bytes = A.nbytes + b.nbytes + c.nbytes
        host_in = (A, b, c)
        kind = lpb.GENERAL
    ropts = rule_opts(name)
    if ropts:
        ropts["lp_index_base"] = lo  # RPC keys on the LP's index in the whole N*B batch
    solver = lpb.Solver(B, m, n, kind, **ropts)
    flush = None
    if in_bytes <= 2 * L2_BYTES:  # small inputs: flush L2 between timed steps
        flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def step(timing=False):
        # timed steps record no library events (each is GPU work between back-to-back
        # solves); the kernel-time pass below turns them on
        solver.solve_device(d_A, d_b, d_c, shared_box=hyper, shared_ab=sab, timing=timing)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    kern_ms, launches = [], 0
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            if flush is not None:
                flush.fill_(float(i))
            ev[i][0].record()
            step()
            ev[i][1].record()
            nl, klass = solver.launch_info()  # host-side fields: no synchronisation
            launches += nl
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # the dominant kernel's own duration (device events around it inside the library), read
    # after each of a few extra, untimed steps: reading it synchronises, so it stays out of
    # the timed loop (whose steps are issued back to back, as a user's would be)
    for i in range(min(args.steps, 5)):
        if flush is not None:
            flush.fill_(float(i))
        step(timing=True)
        kern_ms.append(solver.kernel_ms())
    step_ms = [a.elapsed_time(b_) for a, b_ in ev]
    my_ms = float(sum(step_ms))
    tot_ms = lpdist.max_over_ranks(my_ms, device=torch.device("cuda", local))
    value = B * world * args.steps / (tot_ms / 1e3)
    kmean = float(np.mean(kern_ms))

    # roofline of the dominant kernel (per launch, averaged over the timed launches)
    res = solver.device_results(want_x=True)
    # the only multi-GPU communication is a final gather of the results to rank
    # 0 (padded all_gather over NCCL), outside the timed solve; its time is reported apart
    gather_ms = None
    if world > 1:
        try:
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.barrier()
            g0.record()
            for key in ("status", "obj", "x"):
                lpdist.gather_rows(res[key], B * world)
            g1.record()
            torch.cuda.synchronize()
            gather_ms = lpdist.max_over_ranks(g0.elapsed_time(g1),
                                              device=torch.device("cuda", local))
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
                "algorithmic_bytes_per_launch": traffic_alg}
        iters_mean = None
    else:
        iters = res["iters"].cpu().numpy()
        k = (np.broadcast_to(host_in[1], (B, m)) < 0).sum(axis=1)
        flops = algorithmic_flops(iters, k, m, n)
        if sab and k[0] > 0 and klass in ("M", "L"):
            # phase-I warm start (NEXT-1): phase I ran once for the polytope; every LP only
            # replays its carried objective row through the recorded pivots (2 flop per
            # element per pivot) -- count that, not B phase-I solves
            W = n + float(k[0]) + 1
            it1 = float(iters[0, 0])
            flops -= float(np.sum(2.0 * W * iters[:, 0] * (m + 2)))
            flops += 2.0 * W * it1 * (m + 2) + B * 2.0 * W * it1
        achieved = flops / (kmean / 1e3) / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": p["fp64_tflops"],
                "unit": "TFLOP/s", "frac": achieved / p["fp64_tflops"],
                "traffic": traffic_per_launch(name, B),
                "kernel": f"simplex ({klass} class)",
                "peak_src": "FP64 unit count x clock: 148 SM x 64 DFMA/clk x 2 x "
                            f"{p['sm_max_mhz']:.0f} MHz (DESIGN.md)",
                "algorithmic_flops_per_launch": flops}
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
                    "algorithmic_bytes_per_launch": hb}
        if klass in ("M", "L"):
            # SMEM-resident tableau (SURVEY §8(d) "%SMEM"): every updated element is one 8-byte
            # SMEM read + one write; peak = 148 SMs x 128 B/clk (one shared wavefront per
            # clock, ncu's l1tex__data_pipe_lsu_wavefronts_mem_shared model) x max SM clock
            smem_peak = 148 * 128 * p["sm_max_mhz"] * 1e6 / 1e9
            smem_ach = 16.0 * (flops / 2.0) / (kmean / 1e3) / 1e9
            roof_smem = {"bound": "smem", "achieved": smem_ach, "peak": smem_peak,
                         "unit": "GB/s", "frac": smem_ach / smem_peak,
                         "algorithmic_bytes_per_launch": 16.0 * flops / 2.0}
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
        hs = lpb.Solver(B, m, n, kind, **ropts)
        hs.solve_host_into(*pin, out_st, out_obj, out_x, out_it, shared_box=hyper,
                           shared_ab=sab)  # warm
        e_ms = []
        for _ in range(args.e2e_steps):
            hs.solve_host_into(*pin, out_st, out_obj, out_x, out_it, shared_box=hyper,
                               shared_ab=sab)
            e_ms.append(hs.timing()[1])
            launches_e2e = hs.launch_info()[0]
        e_tot = lpdist.max_over_ranks(float(sum(e_ms)), device=torch.device("cuda", local))
        d2h = out_st.nbytes + out_obj.nbytes + out_x.nbytes + (out_it.nbytes if out_it is not None else 0)
        e2e = {"value": B * world * args.e2e_steps / (e_tot / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(in_bytes), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e_tot / args.e2e_steps,
               "n_chunks": 10 if (B > 100 and in_bytes >= (1 << 20)) else 1,
               "gpu_launches_per_step": launches_e2e}
        hs.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(name, CPU_SAMPLE[name])

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": (value / PAPER_LPS[name]) if name in PAPER_LPS else None,
            "dtype": "f64", "data": "synthetic (seeded lpgen generators, DESIGN.md)",
            "config": {"workload": describe(name), "batch_per_gpu": B, "m": m, "n": n,
                       "kind": "hyperbox" if hyper else "general",
                       "l2": "flushed between steps" if flush is not None else "inputs > L2",
                       "parallelism": f"dp{world} (contiguous LP shards, no collective)",
                       "kernel_class": klass,
                       "ctas_per_lp": solver.launch_shape()[0],
                       "pivot_rule": lpgen.CONFIGS[name].get("rule", "LPC")},
            "roofline": roof,
            **({"roofline_smem": roof_smem} if roof_smem else {}),
            **({"roofline_alu": roof_alu} if roof_alu else {}),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "gather_ms": gather_ms,
            "clocks": clk.summary(),
            "kernel_ms_per_step": kmean,
        }
        if not hyper:
            out["config"]["mean_pivots"] = iters_mean
            out["config"]["status_counts"] = np.bincount(st, minlength=5).tolist()
        print(json.dumps(out), flush=True)
    solver.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
