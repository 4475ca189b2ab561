"""Host configuration layer vs the reference (CPU only): config digests,
resolved scenarios, error codes and error texts, sweep planning and seeds."""
import ctypes
import json
import os

import pytest

import reforacle as ref
import restate
from paper_2511_21669_b200 import ConfigError, DsdError, _lib

pytestmark = pytest.mark.skipif(not ref.available(), reason="reference oracle not built")
CFG = ref.CONFIGS


def _cfg(name):
    with open(os.path.join(CFG, name)) as f:
        return f.read()


@pytest.mark.parametrize("name", ["c1_single_pair.yaml", "c2_8x1_batching.yaml", "c3_64x4_awc.yaml",
                                  "c4_1024x16_static.yaml"])
def test_digest_and_seed_match_reference(gen_dir, name):
    text = _cfg(name)
    rep = json.loads(ref.run_config(text, gen_dir)[0])
    r = restate.Resolved(text, gen_dir)
    assert r.digest == rep["config_digest"]
    assert r.replica.seed == rep["seed"]


C1 = open(os.path.join(CFG, "c1_single_pair.yaml")).read()
BAD = [
    C1.replace("routing: random", "routing: nearest"),
    C1.replace("kind: fifo", "kind: greedy"),
    C1.replace("gamma: 4", "gamma: 40"),
    C1.replace("jitter_ms: 0", "jitter_ms: 20"),
    C1.replace("targets: 1", "targets: 0"),
    C1.replace("drafts: 1", "drafts: 0"),
    C1.replace("seed: 42", "seed: 42\nbogus: 1"),
    C1.replace("acceptance_rate: 0.8", "acceptance_rate: 1.5"),
    C1.replace("rate_rps: 2", "rate_rps: 0"),
    C1.replace("mode: poisson", "mode: replay"),
    C1.replace("n_requests: 100", "n_requests: -3"),
    C1.replace("cost_ratio: 0.1", "cost_ratio: 0"),
    C1.replace("cost_ratio: 0.1", "cost_ratio: 0.1\n    warp: 9"),
    C1.replace("kind: static", "kind: awc"),
    C1.replace("kind: static", "kind: awc\n    model: nowhere.json"),
    C1.replace("prompt_median: 32", "preset: wiki-like"),
    C1.replace("max_batch_size: 8", "max_batch_size: 0"),
    C1.replace("gamma_max: 16", "gamma_max: 16\n    gamma_min: 20"),
    C1.replace("targets: 1", "targets: oops"),
    C1.replace("targets: 1", "targets:\n  count: 2\n  groups:\n    - count: 1"),
    C1.replace("network:", "network:\n  overrides:\n    - draft_group: 3\n      target_group: 0\n"),
    C1.replace("latency_profile:", "latency_profile: missing_profile.json\nold_profile:"),
    C1.replace("  rtt_ms: 10", "\trtt_ms: 10"),
    C1.replace("seed: 42", "seed: [1, 2"),
    C1.replace("seed: 42", "seed: 4.5"),
    "targets: 1\ntargets: 2\n",
    "- a\n- b\n",
]


@pytest.mark.parametrize("k", range(len(BAD)))
def test_errors_match_reference(k):
    text = BAD[k]
    with pytest.raises(ref.RefError) as r:
        ref.run_config(text)
    with pytest.raises(DsdError) as m:
        restate.Resolved(text)
    assert m.value.code == r.value.code
    # the harness prefixes the exception class ("config error: ...")
    assert r.value.msg.split(": ", 1)[1] == m.value.message


def test_sweep_plan_seeds_match_reference():
    spec = open(os.path.join(CFG, "c5_sweep_65536.yaml")).read()
    L = _lib.lib()
    p = ctypes.c_void_p()
    err = ctypes.create_string_buffer(1024)
    assert L.dsd_plan_sweep(spec.encode(), CFG.encode(), 0, 1, ctypes.byref(p), err, 1024) == 0
    reps = ctypes.c_void_p()
    n = L.dsd_sweep_plan_replicas(p, ctypes.byref(reps))
    assert n == 65536
    arr = ctypes.cast(reps, ctypes.POINTER(restate.Replica))
    assert arr[0].seed == 156043105876269134
    pid = "network.rtt_ms=2;policies.window.gamma=1;workload.acceptance_rate=0.53000000000000003"
    assert arr[16].seed == ref.lib().ref_sweep_point_seed(42, pid.encode(), 0)
    L.dsd_sweep_plan_free(p)


def test_sweep_point_ids_and_seeds_match_reference():
    """Axes declared out of sorted order: every replica's seed must be the
    reference's sweep_point_seed of the point id it builds (sorted "key=value"
    parts joined by ';', sweep.cpp:51-73)."""
    import itertools
    axes = [("workload.rate_rps", [1, 2]), ("network.jitter_ms", [0, 1]), ("network.rtt_ms", [10, 20]),
            ("policies.window.gamma", [2, 3])]
    spec = "base: c1_single_pair.yaml\nseed: 7\nrepetitions: 3\naxes:\n" + "".join(
        f"  {k}: [{', '.join(str(v) for v in vals)}]\n" for k, vals in axes)
    L = _lib.lib()
    p = ctypes.c_void_p()
    err = ctypes.create_string_buffer(1024)
    assert L.dsd_plan_sweep(spec.encode(), CFG.encode(), 0, 1, ctypes.byref(p), err, 1024) == 0, err.value
    reps = ctypes.c_void_p()
    n = L.dsd_sweep_plan_replicas(p, ctypes.byref(reps))
    assert n == 16 * 3
    arr = ctypes.cast(reps, ctypes.POINTER(restate.Replica))
    # points in declaration order, last axis fastest
    for k, combo in enumerate(itertools.product(*[vals for _, vals in axes])):
        pid = ";".join(sorted(f"{key}={v}" for (key, _), v in zip(axes, combo)))
        for r in range(3):
            assert arr[k * 3 + r].seed == ref.lib().ref_sweep_point_seed(7, pid.encode(), r), (k, r, pid)
    L.dsd_sweep_plan_free(p)
