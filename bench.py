#!/usr/bin/env python3
"""Benchmark: simulated events/s on the 65,536-replica DSD sweep (BASELINE.json
configs[4]) on N B200s.

One "step" = one pass of the sweep's simulate path over all replicas of this
rank's shard: the device workload-staging kernel (generate_synthetic for every
replica) + the discrete-event simulation kernel, and for N > 1 the NCCL
all-gather of per-replica summaries.  `value` is timed with CUDA events on the
library's stream with inputs resident in HBM (L2 flushed between steps by a
512 MiB memset that is outside the timed events); `e2e` is the same metric
through the public C ABI with host buffers (YAML parse, sweep planning,
host->device upload, kernels, device->host summaries, per-point means).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
SPEC = os.path.join(REPO, "configs", "c5_sweep_65536.yaml")
SPEC_DIR = os.path.dirname(SPEC)


def sweep_text(world):
    """The C5 sweep with 16*world repetitions: every rank simulates its own
    65,536-replica shard (repetitions r, r+world, ...) of one sweep (weak scaling)."""
    text = open(SPEC).read()
    assert "repetitions: 16" in text
    return text.replace("repetitions: 16", f"repetitions: {16 * world}")
B_EV = 64  # algorithmic replica-state bytes per simulated event
METRIC = "simulated_events_per_sec"
WORKLOAD = ("c5_sweep_65536: 4096 points (gamma 1..16 x rtt 2..32 ms x alpha 0.50..0.95) x 16 reps per GPU "
            "(16*N repetitions sharded by repetition over N GPUs), C1 single edge-cloud pair")


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_summary():
    """The committed ncu --set full summary of the simulate kernel (profiles/), if any."""
    p = os.path.join(REPO, "profiles", "ncu_sim_kernel.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


def ncu_traffic():
    """dram read+write bytes per simulate-kernel launch from the committed ncu capture, if any."""
    return ncu_summary().get("dram_bytes_per_launch")


class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, devices):
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", ",".join(str(d) for d in devices)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = max(smax, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference arm: the reference simulator (oracle/_ref) on host cores
# ---------------------------------------------------------------------------
def cpu_reference(seconds_target=8.0, threads=None):
    """Times the reference's own run_sweep worker (resolve_config + run_simulation
    + aggregate_run per replica, sweep.cpp:112-150) on a strided sample of the
    sweep's points with all host threads.  Falls back to the C restatement
    (kind "port") when oracle/_ref was not built."""
    sys.path.insert(0, os.path.join(REPO, "tests"))
    threads = threads or os.cpu_count() or 1
    spec = open(SPEC).read()
    base = os.path.dirname(SPEC)
    import reforacle
    if reforacle.available():
        def run(npts):
            pts = [int(i * 4096 / npts) for i in range(npts)]
            r = reforacle.sweep_bench(spec, base, threads, pts)
            return r["events"], r["replicas"], r["seconds"]
        kind = "reference"
    else:
        import ctypes
        import restate
        from paper_2511_21669_b200 import _lib
        L = _lib.lib()
        p = ctypes.c_void_p()
        err = ctypes.create_string_buffer(1024)
        assert L.dsd_plan_sweep(spec.encode(), base.encode(), 0, 1, ctypes.byref(p), err, 1024) == 0
        sc, rp = ctypes.c_void_p(), ctypes.c_void_p()
        L.dsd_sweep_plan_scenarios(p, ctypes.byref(sc))
        nrep = L.dsd_sweep_plan_replicas(p, ctypes.byref(rp))
        reps = ctypes.cast(rp, ctypes.POINTER(restate.Replica))

        def run(npts):
            idx = [int(i * nrep / (npts * 16)) for i in range(npts * 16)]
            arr = (restate.Replica * len(idx))(*[reps[i] for i in idx])
            out = (_lib.ReplicaSummary * len(idx))()
            t = time.perf_counter()
            restate.olib().oracle_run_batch(sc, arr, len(idx), threads, out, err, 1024)
            dt = time.perf_counter() - t
            return float(sum(o.events_processed for o in out)), float(len(idx)), dt
        kind = "port"
    ev, rep, sec = run(max(8, threads))  # calibration probe
    rate = rep / max(sec, 1e-6)
    npts = int(min(4096, max(16, rate * seconds_target / 16)))
    ev, rep, sec = run(npts)
    return {"events": ev, "replicas": rep, "seconds": sec, "kind": kind, "cores": threads,
            "sample": f"{npts} of 4096 sweep points (strided) x 16 reps = {int(rep)} replicas, {int(ev)} events"}


def main_reference(args, rank, world):
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_reference(seconds_target=2.0)
    ev = rep = sec = 0.0
    last = None
    for _ in range(args.steps):
        r = cpu_reference(seconds_target=6.0)
        ev += r["events"]
        rep += r["replicas"]
        sec += r["seconds"]
        last = r
    value = ev / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * sec / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64+f64",
        "data": "synthetic (reference generate_synthetic streams)",
        "config": {"workload": WORKLOAD, "replicas_sampled_per_step": last["replicas"] if last else 0},
        "replicas_per_sec": rep / sec,
        "cpu_baseline": {"value": value, "unit": "events/s", "cores": last["cores"], "kind": last["kind"],
                         "sample": last["sample"]},
        "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    from paper_2511_21669_b200 import Simulator

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    sim = Simulator(local_rank)
    spec = sweep_text(world)
    n_rep, n_pts = sim.prepare_sweep(spec, base_dir=SPEC_DIR, shard=rank, n_shards=world)
    stream = torch.cuda.ExternalStream(sim.stream(), device=torch.device("cuda", local_rank))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    sum_ptr, sum_bytes = sim.device_summaries()
    gather = None
    if world > 1:
        # per-replica summaries, gathered once per step over NVLink
        max_rep = n_rep
        rows = torch.zeros(max_rep * 96, dtype=torch.uint8, device="cuda")
        gather = torch.zeros(world * max_rep * 96, dtype=torch.uint8, device="cuda")

    def one_step():
        sim.launch()
        if gather is not None:
            with torch.cuda.stream(stream):
                dev = torch.as_tensor(_DevView(sum_ptr, sum_bytes), device="cuda")
                rows[:sum_bytes].copy_(dev)
                dist.all_gather_into_tensor(gather, rows)

    for _ in range(args.warmup):
        one_step()
        sim.sync()
        torch.cuda.synchronize()
    sm = sim.summaries()
    if (sm["status"] != 0).any():
        raise SystemExit("engine reported failed replicas")
    ev_local = float(sm["events_processed"].sum())

    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks([local_rank]) if rank == 0 else None
    t0 = time.perf_counter()
    step_ms, sim_ms = [], []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()  # evict L2 between steps (outside the timed events)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        one_step()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        sim_ms.append(sim.last_kernel_ms()["sim_ms"])
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    wall = time.perf_counter() - t0
    clk = clocks.stop() if clocks else None

    tot_ms = sum(step_ms)
    if dist:
        t = torch.tensor([tot_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
        e = torch.tensor([ev_local, float(n_rep)], dtype=torch.float64, device="cuda")
        dist.all_reduce(e, op=dist.ReduceOp.SUM)
        ev_all, rep_all = float(e[0].item()), float(e[1].item())
    else:
        ev_all, rep_all = ev_local, float(n_rep)
    ms_per_step = tot_ms / args.steps
    value = ev_all / (ms_per_step / 1e3)

    # ---- e2e through the public C ABI with host buffers ----
    e2e_times = []
    h2d = d2h = 0
    for k in range(args.steps + 1):
        if dist:
            dist.barrier()
        t = time.perf_counter()
        if world == 1:
            out = sim.run_sweep(spec, base_dir=SPEC_DIR)
            assert out.failed_points == 0
        else:
            sim.prepare_sweep(spec, base_dir=SPEC_DIR, shard=rank, n_shards=world)
            sim.launch()
            s2 = sim.summaries()
            _ = s2["throughput_rps"].sum()
        dt = time.perf_counter() - t
        if k > 0:  # first call warms the host caches
            e2e_times.append(dt)
        h2d, d2h = sim.last_transfer_bytes()
    e2e_s = sum(e2e_times) / len(e2e_times)
    if dist:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    # restore the prepared device batch
    if world == 1:
        sim.prepare_sweep(spec, base_dir=SPEC_DIR, shard=rank, n_shards=world)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_kind = peaks()
    sim_avg = sum(sim_ms) / len(sim_ms)
    achieved = B_EV * ev_local / (sim_avg / 1e3) / 1e9
    traffic = ncu_traffic()
    line = {
        "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64+f64",
        "data": "synthetic (reference generate_synthetic streams, regenerated on device every step)",
        "config": {"workload": WORKLOAD, "replicas": int(rep_all), "points": n_pts,
                   "events_per_step": int(ev_all), "l2": "flushed between steps (512 MiB memset)",
                   "parallelism": f"replica shards x{world} + NCCL all-gather of summaries" if world > 1
                   else "single GPU"},
        "replicas_per_sec": rep_all / (ms_per_step / 1e3),
        "e2e": {"value": ev_all / e2e_s, "unit": "events/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * e2e_s,
                "path": "dsd_run_sweep" if world == 1 else "dsd_prepare_sweep+dsd_batch_launch+dsd_batch_summaries"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_kind, "bytes_per_event": B_EV,
                     "kernel": "k_simulate", "kernel_ms": sim_avg,
                     # the DES is latency-bound, not HBM-bound: the
                     # committed capture's SM issue activity and top warp stalls
                     "ncu_issue_active_pct": ncu_summary().get("issue_active_pct"),
                     "ncu_stall_pct": dict(list(ncu_summary().get("stall_pct", {}).items())[:4])},
        "gpu_launches": sim.last_launch_count() * args.steps,
        "wall_s": wall,
    }
    if clk:
        line["clocks"] = clk
    if world == 1 and not args.no_cpu_baseline:
        cb = cpu_reference()
        line["cpu_baseline"] = {"value": cb["events"] / cb["seconds"], "unit": "events/s", "cores": cb["cores"],
                                "kind": cb["kind"], "sample": cb["sample"],
                                "replicas_per_sec": cb["replicas"] / cb["seconds"]}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


class _DevView:
    """__cuda_array_interface__ over the library's device summary buffer."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        main_reference(args, rank, world)
    else:
        main_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
