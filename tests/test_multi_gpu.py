"""One handle over several GPUs (dsd_create_devices): the replicas of every
batch and sweep are dealt across the devices in cost order and the results
come back in replica order - byte-identical to a one-device handle and to
the reference run_sweep (proj/src/runner/sweep.cpp:87-162).  Needs a lease
with >= 2 GPUs (gpurun --gpus 2); skipped otherwise."""
import os

import pytest

import reforacle as ref

pytestmark = pytest.mark.gpu
CFG = ref.CONFIGS


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


need2 = pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")


def _all():
    return list(range(_gpus()))


@need2
def test_c5_sweep_on_every_gpu_matches_reference():
    """BASELINE's workload through the drop-in call on all of the lease's GPUs."""
    from paper_2511_21669_b200 import Simulator
    spec = open(os.path.join(CFG, "c5_sweep_65536.yaml")).read()
    js, cs = ref.run_sweep(spec, CFG, os.cpu_count() or 8)
    with Simulator(_all()) as s:
        out = s.run_sweep(spec, base_dir=CFG)
        sizes = s.shard_sizes()
    assert (out.points, out.replicas, out.failed_points) == (4096, 65536, 0)
    assert out.events_processed == 880021538
    assert out.summary_json == js and out.summary_csv == cs
    assert sum(sizes) == 65536 and max(sizes) - min(sizes) <= 1


@need2
def test_multi_device_batch_equals_single_device():
    """Per-replica summaries (a generic-kernel sweep with jitter, dynamic
    windows and batching windows) are identical on one and on all GPUs."""
    from paper_2511_21669_b200 import Simulator
    spec = ("base: c2_8x1_batching.yaml\nseed: 3\nrepetitions: 5\naxes:\n"
            "  network.rtt_ms: [2, 20, 60]\n  policies.window.kind: [static, dynamic, fused]\n"
            "  workload.rate_rps: [6, 12]\n")
    sums = []
    for devs in ([0], _all()):
        with Simulator(devs) as s:
            s.prepare_sweep(spec, base_dir=CFG)
            s.launch()
            s.sync()
            sums.append(s.summaries())
    assert len(sums[0]) == 90 and (sums[0]["status"] == 0).all()
    assert sums[0].tobytes() == sums[1].tobytes()


@need2
def test_multi_device_report_files_match_reference(tmp_path):
    """Per-replica reports (records fetched from whichever GPU ran the replica)."""
    from paper_2511_21669_b200 import Simulator
    spec = "base: c1_single_pair.yaml\nseed: 3\nrepetitions: 3\naxes:\n  network.rtt_ms: [4, 30]\n"
    ref_dir, my_dir = tmp_path / "ref", tmp_path / "mine"
    ref.run_sweep(spec, CFG, 2, str(ref_dir))
    with Simulator(_all()) as s:
        s.run_sweep(spec, base_dir=CFG, out_dir=str(my_dir))
    files = sorted(os.listdir(ref_dir))
    assert files == sorted(os.listdir(my_dir))
    for f in files:
        assert (ref_dir / f).read_bytes() == (my_dir / f).read_bytes(), f


@need2
def test_multi_device_dataset_matches_single_device(gen_dir):
    """generate_dataset (2,400 probed replicas) on all GPUs == on one."""
    from paper_2511_21669_b200 import Simulator
    outs = []
    for devs in ([0], _all()):
        with Simulator(devs) as s:
            outs.append(s.generate_dataset(""))
    assert outs[0] == outs[1]


@need2
def test_device_listed_twice_is_rejected():
    from paper_2511_21669_b200 import EngineError, Simulator
    with pytest.raises(EngineError, match="twice"):
        Simulator([0, 0])
