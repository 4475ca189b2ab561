#!/usr/bin/env python3
"""Benchmark: simulated events/s of the DSD-Sim simulate-a-sweep path on N B200s.

Default workload: BASELINE.json configs[4], the 65,536-replica C5 sweep
(SURVEY.md §8(d)): 4,096 points (gamma 1..16 x rtt 2..32 ms x alpha 0.50..0.95)
x 16 repetitions of the C1 single edge-cloud pair.

One "step" = one pass of the sweep's simulate path over this rank's replicas:
the device workload-staging kernel (generate_synthetic for every replica) +
the discrete-event simulation kernel, and for N > 1 the NCCL all-gather of the
96-byte per-replica summaries.  Scaling is STRONG by default: the same 65,536
replicas are dealt across the N GPUs in cost order (the split the library's
multi-device handle makes); --weak gives every GPU its own 65,536 replicas.

  value  CUDA events on the library's stream, inputs resident in HBM, L2
         flushed between steps (512 MiB memset outside the timed events),
         max over ranks.
  e2e    the same metric through the public C ABI with host buffers:
         dsd_run_sweep (YAML parse, sweep planning, pack + H2D, kernels, D2H
         of the summaries, per-point means, summary JSON/CSV).  For N > 1 rank
         0 makes the drop-in call on a handle over all N GPUs
         (dsd_create_devices) while the other ranks wait.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--weak] [--workload c5|c2_seeds|c2_seeds_16k|c3_seeds|c3_seeds_4k|c4s_seeds|c4a_seeds|
                   c1_single|c2_single|c3_single|c4s_single|c4a_single]
"""
import argparse
import json
import os
import statistics
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
CONFIGS = os.path.join(REPO, "configs")
GOLDEN = os.path.join(REPO, "tests", "golden", "configs")
GEN = os.path.join(REPO, "tests", "golden", "_gen")  # mixed.jsonl / model.json (reference-built fixtures)
B_EV = 64  # algorithmic replica-state bytes per simulated event
METRIC = "simulated_events_per_sec"
C5 = os.path.join(CONFIGS, "c5_sweep_65536.yaml")


def _seed_sweep(base, reps, n_points):
    """n_points x reps replicas of one config: the points differ only in the
    default link RTT (network.rtt_ms 2..n_points+1; every C3/C4 pair has an
    override, so there it only changes the point id and hence the seeds) -
    the reference's run_sweep parallelises over points, not repetitions."""
    vals = ", ".join(str(v) for v in range(2, n_points + 2))
    return f"base: {base}\nseed: 42\nrepetitions: {reps}\naxes:\n  network.rtt_ms: [{vals}]\n"


# name -> (kind, text or path, base_dir, description)
WORKLOADS = {
    "c5": ("sweep", C5, CONFIGS,
           "c5_sweep_65536: 4096 points (gamma 1..16 x rtt 2..32 ms x alpha 0.50..0.95) x 16 reps, "
           "C1 single edge-cloud pair (BASELINE configs[4])"),
    "c2_seeds": ("sweep", _seed_sweep(os.path.join(GOLDEN, "c2_8x1_batching.yaml"), 32, 32),
                 GOLDEN, "C2 (8 drafts x 1 target, 2 ms batching window, jsq): rtt 2..33 ms x 32 seeds = 1024 replicas"),
    "c2_seeds_16k": ("sweep", _seed_sweep(os.path.join(GOLDEN, "c2_8x1_batching.yaml"), 32, 512), GOLDEN,
                     "C2 (8 drafts x 1 target, 2 ms batching window, jsq): rtt 2..513 ms x 32 seeds = 16384 replicas"),
    "c3_seeds_4k": ("sweep", _seed_sweep(os.path.join(GOLDEN, "c3_64x4_awc.yaml"), 16, 256), GEN,
                    "C3 (64 drafts x 4 targets, heterogeneous RTT, AWC) x 4096 seeds"),
    "c3_seeds": ("sweep", _seed_sweep(os.path.join(GOLDEN, "c3_64x4_awc.yaml"), 16, 16), GEN,
                 "C3 (64 drafts x 4 targets, heterogeneous RTT, AWC) x 256 seeds"),
    "c4s_seeds": ("sweep", _seed_sweep(os.path.join(GOLDEN, "c4_1024x16_static.yaml"), 4, 16), GEN,
                  "C4 static (1024 drafts x 16 targets, mixed trace) x 64 seeds"),
    "c4a_seeds": ("sweep", _seed_sweep(os.path.join(GOLDEN, "c4_1024x16_awc.yaml"), 4, 16), GEN,
                  "C4 AWC (1024 drafts x 16 targets, mixed trace) x 64 seeds"),
    "c1_single": ("single", os.path.join(GOLDEN, "c1_single_pair.yaml"), GOLDEN, "C1 single run"),
    "c2_single": ("single", os.path.join(GOLDEN, "c2_8x1_batching.yaml"), GOLDEN, "C2 single run"),
    "c3_single": ("single", os.path.join(GOLDEN, "c3_64x4_awc.yaml"), GEN, "C3 single run (AWC)"),
    "c4s_single": ("single", os.path.join(GOLDEN, "c4_1024x16_static.yaml"), GEN, "C4 static single run"),
    "c4a_single": ("single", os.path.join(GOLDEN, "c4_1024x16_awc.yaml"), GEN, "C4 AWC single run"),
}


def workload_text(name, weak_world=1):
    kind, src, base, desc = WORKLOADS[name]
    text = open(src).read() if os.path.exists(src) else src
    if kind == "sweep" and weak_world > 1:
        import re
        m = re.search(r"repetitions: (\d+)", text)
        text = text.replace(m.group(0), f"repetitions: {int(m.group(1)) * weak_world}")
    return kind, text, base, desc


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
    """The committed ncu --set full summary of the simulate kernel on the
    default workload at N=1 (profiles/ncu_sim_kernel.json), if any."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_sim_kernel.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


_SAMPLER = r"""
import sys, time
import pynvml as nv
nv.nvmlInit()
hs = [nv.nvmlDeviceGetHandleByIndex(int(i)) for i in sys.argv[1].split(",")]
masks = [(n, getattr(nv, a)) for n, a in (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
         ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
         ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
         ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))]
smax = max(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM) for h in hs)
print("ready", smax, flush=True)
while True:
    for h in hs:
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        print(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), *[n for n, m in masks if r & m], flush=True)
    time.sleep(0.002)
"""


class Clocks:
    """SM clocks and throttle reasons sampled DURING the timed region by an NVML
    poller every 2 ms in a separate process (the timed region of a default run
    is ~0.1 s, too short for nvidia-smi -lms; a thread would contend for the
    GIL with the launching thread).  CUDA ordinals map to NVML indices through
    CUDA_VISIBLE_DEVICES when it is set."""

    def __init__(self, devices):
        import subprocess
        import tempfile
        self.proc = None
        try:
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = [vis.split(",")[d] if vis else str(d) for d in devices]
            fd, self.path = tempfile.mkstemp(suffix=".clocks")
            os.close(fd)
            with open(self.path, "ab") as sink:  # O_APPEND: the reader's offset is its own
                self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER, ",".join(idx)], stdout=sink,
                                             stderr=subprocess.DEVNULL)
            self.smax, self.start = 0.0, None
            t = time.time()
            while time.time() - t < 20 and self.proc.poll() is None:  # until it samples
                with open(self.path) as f:
                    first = f.readline()
                    if first.startswith("ready") and first.endswith("\n"):
                        self.smax = float(first.split()[1])
                        f.seek(0, 2)
                        self.start = f.tell()  # the timed region starts after this
                        break
                time.sleep(0.01)
            if self.start is None:
                self.proc.kill()
                self.proc = None
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        self.proc.wait(timeout=5)
        sm, reasons = [], set()
        with open(self.path) as f:
            f.seek(self.start)
            for line in f.read().splitlines():
                parts = line.split()
                if not parts or parts[0] == "ready":
                    continue
                sm.append(float(parts[0]))
                reasons.update(parts[1:])
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.smax, "reasons": sorted(reasons),
                "samples": len(sm), "sampler": "nvml, 2 ms, own process"}


# ---------------------------------------------------------------------------
# CPU reference: the reference simulator (oracle/_ref) on the host cores
# ---------------------------------------------------------------------------
def cpu_reference(name, threads=None, sample_points=None):
    """Times the reference's own run_sweep worker (resolve_config +
    run_simulation + aggregate_run per replica, sweep.cpp:112-150) over the
    WHOLE sweep (every point x every repetition) with all host threads, or the
    reference's run_simulation of a single config on one core.  Falls back to
    the C restatement (kind "port") when oracle/_ref was not built."""
    sys.path.insert(0, os.path.join(REPO, "tests"))
    threads = threads or os.cpu_count() or 1
    kind, text, base, desc = workload_text(name)
    import reforacle
    if kind == "single":
        if not reforacle.available():
            raise SystemExit("reference oracle not built")
        t = time.perf_counter()
        _, ev, _, _ = reforacle.run_config(text, base)
        dt = time.perf_counter() - t
        return {"events": float(ev), "replicas": 1.0, "seconds": dt, "kind": "reference", "cores": 1,
                "sample": f"{desc}: the whole run ({ev} events) on one core (a run is single-threaded)"}
    if reforacle.available():
        r = reforacle.sweep_bench(text, base, threads, sample_points)
        ev, rep, sec = r["events"], r["replicas"], r["seconds"]
        k = "reference"
        # the sim-only split: run_simulation alone vs resolve_config
        # (+ generate_synthetic), thread-summed
        split = {"run_simulation_share": r["sim_thread_s"] / max(r["sim_thread_s"] + r["resolve_thread_s"], 1e-12),
                 "sim_only_events_per_sec": ev / max(r["sim_thread_s"] / threads, 1e-12)}
    else:
        import ctypes
        import restate
        from paper_2511_21669_b200 import _lib
        L = _lib.lib()
        p = ctypes.c_void_p()
        err = ctypes.create_string_buffer(1024)
        assert L.dsd_plan_sweep(text.encode(), base.encode(), 0, 1, ctypes.byref(p), err, 1024) == 0
        sc, rp = ctypes.c_void_p(), ctypes.c_void_p()
        L.dsd_sweep_plan_scenarios(p, ctypes.byref(sc))
        nrep = L.dsd_sweep_plan_replicas(p, ctypes.byref(rp))
        out = (_lib.ReplicaSummary * nrep)()
        t = time.perf_counter()
        restate.olib().oracle_run_batch(sc, rp, nrep, threads, out, err, 1024)
        sec = time.perf_counter() - t
        ev, rep, k = float(sum(o.events_processed for o in out)), float(nrep), "port"
    what = "the whole sweep" if not sample_points else f"{len(sample_points)} points of the sweep"
    res = {"events": ev, "replicas": rep, "seconds": sec, "kind": k, "cores": threads,
           "sample": f"{desc}: {what} ({int(rep)} replicas, {int(ev)} events) on {threads} threads "
                     f"({cpu_model()})"}
    if k == "reference":
        res["split"] = split
    return res


def main_reference(args, rank, world):
    if rank != 0:
        return
    kind = WORKLOADS[args.workload][0]
    # warm-up: a few points (threads, allocator, page cache) - not the full sweep
    for _ in range(args.warmup):
        cpu_reference(args.workload, sample_points=list(range(0, 4096, 256)) if kind == "sweep" else None)
    ev = rep = sec = 0.0
    last = None
    for _ in range(args.steps):
        r = cpu_reference(args.workload)
        ev += r["events"]
        rep += r["replicas"]
        sec += r["seconds"]
        last = r
    value = ev / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * sec / args.steps,
        "higher_is_better": True, "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
        "dtype": "int64+f64", "data": "synthetic (reference generate_synthetic streams)",
        "config": {"workload": WORKLOADS[args.workload][3], "replicas_per_step": int(last["replicas"]),
                   "events_per_step": int(last["events"])},
        "replicas_per_sec": rep / sec,
        "cpu_baseline": {"value": value, "unit": "events/s", "cores": last["cores"], "kind": last["kind"],
                         "sample": last["sample"]},
        "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if "split" in last:
        line["cpu_baseline"]["split"] = last["split"]
    emit(line)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def roofline(ev_local, sim_ms, clk, same_launch=True):
    """same_launch: the committed capture is of this launch (the N=1 default
    workload); a strong-scaling shard is a different launch, so its line
    carries no capture-derived fields."""
    peak, peak_kind = peaks()
    achieved = B_EV * ev_local / (sim_ms / 1e3) / 1e9
    nc = ncu_summary() if same_launch else {}
    out = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
           "traffic": nc.get("dram_bytes_per_launch"), "peak_source": peak_kind, "bytes_per_event": B_EV,
           "kernel": "k_simulate", "kernel_ms": sim_ms,
           "from_committed_capture": ["traffic", "issue.warp_instructions", "issue.threads_per_instruction",
                                      "ncu_issue_active_pct", "ncu_stall_pct"] if nc else []}
    # The DES is latency/issue-bound, not HBM-bound: the issue
    # roofline = warp instructions of the launch (deterministic for the
    # workload; from the committed capture) / (SMs x 4 schedulers x clock x
    # the live kernel time), and the SIMT efficiency of those instructions.
    wi = nc.get("warp_instructions")
    if wi and clk and clk.get("sm_mhz"):
        sms = nc.get("sms", 148)
        slots = sms * 4 * clk["sm_mhz"] * 1e6 * (sim_ms / 1e3)
        out["issue"] = {"warp_instructions": wi, "issue_slots": slots, "frac": wi / slots,
                        "threads_per_instruction": nc.get("threads_per_instruction"),
                        "clock_mhz": clk["sm_mhz"], "sms": sms}
    out["ncu_issue_active_pct"] = nc.get("issue_active_pct")
    out["ncu_stall_pct"] = dict(list(nc.get("stall_pct", {}).items())[:4])
    return out


def main_single(args, rank, world, local_rank):
    """A single config through dsd_run_simulation (one replica; no sharding)."""
    import torch
    from paper_2511_21669_b200 import Simulator
    if rank != 0:
        return
    _, text, base, desc = workload_text(args.workload)
    torch.cuda.set_device(local_rank)
    sim = Simulator(local_rank)
    for _ in range(args.warmup):
        out = sim.run_simulation(text, base_dir=base, report=False)
    clocks = Clocks([local_rank])
    dev_ms, wall = [], []
    for _ in range(args.steps):
        t = time.perf_counter()
        out = sim.run_simulation(text, base_dir=base, report=False)
        wall.append(time.perf_counter() - t)
        dev_ms.append(sim.last_kernel_ms()["total_ms"])
    clk = clocks.stop()
    ev = out.events_processed
    ms = sum(dev_ms) / len(dev_ms)
    e2e_s = sum(wall) / len(wall)
    h2d, d2h = sim.last_transfer_bytes()
    line = {"metric": METRIC, "value": ev / (ms / 1e3), "unit": "events/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "none",
            "vs_baseline": None, "dtype": "int64+f64", "data": "synthetic / reference-built trace fixtures",
            "config": {"workload": desc, "events_per_step": ev, "replicas": 1},
            "e2e": {"value": ev / e2e_s, "unit": "events/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * e2e_s, "path": "dsd_run_simulation"},
            "gpu_launches": sim.last_launch_count() * args.steps}
    if clk:
        line["clocks"] = clk
    if not args.no_cpu_baseline:
        cb = cpu_reference(args.workload)
        line["cpu_baseline"] = {"value": cb["events"] / cb["seconds"], "unit": "events/s", "cores": cb["cores"],
                                "kind": cb["kind"], "sample": cb["sample"]}
    emit(line)


def main_ours(args, rank, world, local_rank):
    import torch
    from paper_2511_21669_b200 import Simulator

    if WORKLOADS[args.workload][0] == "single":
        return main_single(args, rank, world, local_rank)
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    sim = Simulator(local_rank)
    _, spec, base, desc = workload_text(args.workload, world if args.weak else 1)
    # this rank's shard: strong = 1/N of the same replicas, weak = 1/N of an N-times larger sweep
    n_rep, n_pts = sim.prepare_sweep(spec, base_dir=base, shard=rank, n_shards=world)
    stream = torch.cuda.ExternalStream(sim.stream(), device=torch.device("cuda", local_rank))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    sum_ptr, sum_bytes = sim.device_summaries()
    gather = None
    if world > 1:
        # per-replica summaries, gathered once per step over NVLink;
        # shards differ by at most one replica: pad to the largest
        nmax = torch.tensor([n_rep], dtype=torch.int64, device="cuda")
        dist.all_reduce(nmax, op=dist.ReduceOp.MAX)
        max_rep = int(nmax.item())
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

    # (the sampler starts before the barrier: the other ranks would otherwise
    # wait for rank 0 inside their first timed step)
    clocks = Clocks([local_rank]) if rank == 0 else None
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
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
    per_rank = None
    if dist:
        # every rank's step and simulate-kernel times (the max is the value)
        mine = torch.tensor([tot_ms / args.steps, sum(sim_ms) / len(sim_ms)], dtype=torch.float64, device="cuda")
        allr = torch.zeros(world * 2, dtype=torch.float64, device="cuda")
        dist.all_gather_into_tensor(allr, mine)
        per_rank = [{"ms_per_step": round(float(allr[2 * r]), 3), "sim_kernel_ms": round(float(allr[2 * r + 1]), 3)}
                    for r in range(world)]
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
    sim_avg = sum(sim_ms) / len(sim_ms)
    launches = sim.last_launch_count() * args.steps

    # ---- e2e through the public C ABI with host buffers: the drop-in call ----
    e2e_s, h2d, d2h, e2e_path = None, 0, 0, "dsd_run_sweep"
    # the other ranks wait on a host (gloo) barrier: an NCCL barrier would
    # spin a kernel on the GPUs rank 0 is now using
    cpu_group = dist.new_group(backend="gloo") if dist else None
    if dist:
        dist.barrier(group=cpu_group)
    if rank == 0:
        devices = list(range(world))
        esim = sim if world == 1 else Simulator(devices)
        if world > 1:
            e2e_path = f"dsd_run_sweep on dsd_create_devices({devices}) from rank 0"
        times = []
        for k in range(args.steps + 1):
            t = time.perf_counter()
            out = esim.run_sweep(spec, base_dir=base)
            dt = time.perf_counter() - t
            assert out.failed_points == 0
            if k > 0:  # the first call warms the host caches and the other devices
                times.append(dt)
            h2d, d2h = esim.last_transfer_bytes()
        e2e_s = sum(times) / len(times)
        e2e_events = out.events_processed
        if esim is not sim:
            esim.close()
    if dist:
        dist.barrier(group=cpu_group)
    if rank != 0:
        dist.destroy_process_group()
        return

    line = {
        "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "int64+f64",
        "data": "synthetic (reference generate_synthetic streams, regenerated on device every step)",
        "config": {"workload": desc, "replicas": int(rep_all), "points": n_pts, "events_per_step": int(ev_all),
                   "l2": "flushed between steps (512 MiB memset)",
                   "parallelism": (f"{'weak' if args.weak else 'strong'}: replicas dealt over {world} GPUs in "
                                   f"cost order + NCCL all-gather of summaries") if world > 1 else "single GPU"},
        "replicas_per_sec": rep_all / (ms_per_step / 1e3),
        "e2e": {"value": e2e_events / e2e_s, "unit": "events/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * e2e_s, "path": e2e_path},
        "roofline": roofline(ev_local, sim_avg, clk, same_launch=world == 1 and args.workload == "c5"),
        "gpu_launches": launches,
        "wall_s": wall,
    }
    if world > 1:
        line["rank0"] = {"replicas": n_rep, "events": int(ev_local), "sim_kernel_ms": sim_avg}
        line["ranks"] = per_rank
    if clk:
        line["clocks"] = clk
    if world == 1 and not args.no_cpu_baseline:
        cb = cpu_reference(args.workload)
        line["cpu_baseline"] = {"value": cb["events"] / cb["seconds"], "unit": "events/s", "cores": cb["cores"],
                                "kind": cb["kind"], "sample": cb["sample"],
                                "replicas_per_sec": cb["replicas"] / cb["seconds"]}
        if "split" in cb:
            line["cpu_baseline"]["split"] = cb["split"]
    emit(line)
    if dist:
        dist.destroy_process_group()


class _DevView:
    """__cuda_array_interface__ over the library's device summary buffer."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


_STDOUT = None


def emit(line):
    """The one JSON line, on the process's real stdout (libraries' banners -
    NCCL prints its version at communicator creation - go to stderr)."""
    os.write(_STDOUT if _STDOUT is not None else 1, (json.dumps(line) + "\n").encode())


def main():
    global _STDOUT
    # everything else written to fd 1 (C libraries included) goes to stderr
    sys.stdout.flush()
    _STDOUT = os.dup(1)
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--weak", action="store_true", help="every GPU simulates its own copy of the workload")
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
