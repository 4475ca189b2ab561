"""N>1 host logic on CPU: world_size-2 gloo processes each plan their shard of
a sweep (dsd_plan_sweep with shard/n_shards, the set dsd_prepare_sweep runs
on a GPU), simulate it (the C oracle stands in for the device engine here),
all-gather the 96-byte summaries, and rank 0 rebuilds the per-point means the
way run_sweep does (sweep.cpp:131-144).  The result must equal the reference
run_sweep summary byte for byte, and the shards must partition the sweep."""
import ctypes
import json
import os
import socket

import numpy as np
import pytest

import reforacle as ref

pytestmark = pytest.mark.skipif(not ref.available(), reason="reference oracle not built")

SPEC = ("base: c1_single_pair.yaml\nseed: 5\nrepetitions: 4\naxes:\n"
        "  network.rtt_ms: [4, 20]\n  policies.window.gamma: [2, 6]\n  workload.n_requests: [12, 20]\n")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def plan_shard(spec, base_dir, shard, n_shards):
    from paper_2511_21669_b200 import _lib
    L = _lib.lib()
    p = ctypes.c_void_p()
    err = ctypes.create_string_buffer(1024)
    assert L.dsd_plan_sweep(spec.encode(), base_dir.encode(), shard, n_shards, ctypes.byref(p), err, 1024) == 0, \
        err.value
    sc, rp = ctypes.c_void_p(), ctypes.c_void_p()
    L.dsd_sweep_plan_scenarios(p, ctypes.byref(sc))
    n = L.dsd_sweep_plan_replicas(p, ctypes.byref(rp))
    pts = (ctypes.c_int64 * max(n, 1))()
    reps = (ctypes.c_int32 * max(n, 1))()
    L.dsd_sweep_plan_origin(p, pts, reps, n)
    return L, p, sc, rp, n, list(pts)[:n], list(reps)[:n]


def _worker(rank, world, port, out_path):
    import torch.distributed as dist
    import torch
    import restate
    from paper_2511_21669_b200 import _lib
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, p, sc, rp, n, pts, reps = plan_shard(SPEC, ref.CONFIGS, rank, world)
    out = (_lib.ReplicaSummary * max(n, 1))()
    err = ctypes.create_string_buffer(256)
    restate.olib().oracle_run_batch(sc, rp, n, 1, out, err, 256)
    rows = np.zeros((n, 5), dtype=np.float64)
    for k in range(n):
        rows[k] = (pts[k], reps[k], out[k].throughput_rps, out[k].mean_ttft_ms, out[k].mean_tpot_ms)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([n]))
    mx = int(max(s.item() for s in sizes))
    buf = torch.zeros(mx, 5, dtype=torch.float64)
    buf[:n] = torch.from_numpy(rows)
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf)
    if rank == 0:
        allrows = np.concatenate([b[: int(s.item())].numpy() for b, s in zip(bufs, sizes)])
        with open(out_path, "w") as f:
            json.dump(allrows.tolist(), f)
    L.dsd_sweep_plan_free(p)
    dist.destroy_process_group()


def test_shards_partition_the_sweep():
    _, p0, _, _, n_all, pts_all, reps_all = plan_shard(SPEC, ref.CONFIGS, 0, 1)
    seen = set()
    for r in range(3):
        _, p, _, _, n, pts, reps = plan_shard(SPEC, ref.CONFIGS, r, 3)
        s = set(zip(pts, reps))
        assert not (s & seen)
        seen |= s
    assert seen == set(zip(pts_all, reps_all))
    assert n_all == 8 * 4


def test_gloo_two_ranks_rebuild_reference_summary(tmp_path):
    import torch.multiprocessing as mp
    out_path = str(tmp_path / "rows.json")
    mp.spawn(_worker, args=(2, _free_port(), out_path), nprocs=2, join=True)
    rows = json.load(open(out_path))
    js, _ = ref.run_sweep(SPEC, ref.CONFIGS, 2)
    want = json.loads(js)["points"]
    R = 4
    sums = {}
    for pt, rep, thr, ttft, tpot in sorted(rows, key=lambda r: (r[0], r[1])):  # rep order, as run_sweep
        a = sums.setdefault(int(pt), [0.0, 0.0, 0.0])
        a[0] += thr
        a[1] += ttft
        a[2] += tpot
    assert len(sums) == len(want)
    for i, w in enumerate(want):
        thr, ttft, tpot = (x / R for x in sums[i])
        assert w["throughput_rps"] == "%.6f" % thr or float(w["throughput_rps"]) == float("%.6f" % thr)
        assert float(w["mean_ttft_ms"]) == float("%.3f" % ttft)
        assert float(w["mean_tpot_ms"]) == float("%.3f" % tpot)


def test_cost_ordered_shards_partition_the_sweep():
    """dsd_plan_sweep's shards (the deal dsd_create_devices makes) partition
    the sweep, each in point-major order, sizes within one of each other."""
    spec = ("base: c1_single_pair.yaml\nseed: 5\nrepetitions: 3\naxes:\n"
            "  policies.window.gamma: [1, 4, 16]\n  workload.acceptance_rate: [0.5, 0.9]\n  network.rtt_ms: [2, 30]\n")
    _, _, _, _, n_all, pts_all, reps_all = plan_shard(spec, ref.CONFIGS, 0, 1)
    for world in (2, 3, 4, 8):
        seen = []
        sizes = []
        for shard in range(world):
            _, _, _, _, n, pts, reps = plan_shard(spec, ref.CONFIGS, shard, world)
            origin = list(zip(pts, reps))
            assert origin == sorted(origin)
            seen += origin
            sizes.append(n)
        assert sorted(seen) == sorted(zip(pts_all, reps_all))
        assert max(sizes) - min(sizes) <= 1
