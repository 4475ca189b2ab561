"""GPU parity: the sm_100a engine vs the reference simulator (oracle/_ref) on
the same configs.  Bit-exact: every report byte (all integer outputs and the
3/6-decimal float renderings), events_processed and end_time must match."""
import os
import re

import pytest

import reforacle as ref

pytestmark = pytest.mark.gpu
CFG = ref.CONFIGS


def _cfg(name):
    with open(os.path.join(CFG, name)) as f:
        return f.read()


def _compare(sim, text, base_dir=".", seed=None):
    rep, ev, end, agg = ref.run_config(text, base_dir, seed)
    out = sim.run_simulation(text, base_dir=base_dir, seed=seed)
    assert out.events_processed == ev
    assert out.end_time_us == end
    if out.report_json != rep:
        a, b = rep.splitlines(), out.report_json.splitlines()
        for i, (x, y) in enumerate(zip(a, b)):
            assert x == y, f"first report difference at line {i}"
        assert len(a) == len(b)
    assert out.completed == int(agg[0])
    assert out.throughput_rps == agg[1]
    assert out.mean_ttft_ms == agg[2]
    assert out.mean_tpot_ms == agg[3]
    return out


@pytest.mark.parametrize("name,golden", [
    ("c1_single_pair.yaml", "12253632ad5d73e55984bf1b64a17e8b4cb966f1c137e65367a1d78f228ed7ce"),
    ("c2_8x1_batching.yaml", "cb0d409d66afb46dab47f25590fb30a3f8f6f88531bfd088b640837eb4bf90a1"),
    ("c3_64x4_awc.yaml", "eb1dbe06b534b6e52dde1a7da752cf91abac9712e5005936bff30af8a197bdb3"),
    ("c4_1024x16_static.yaml", "3b4a3e55b3f2f45bb5d613e107b06605735cd1ed21f102516c28a816b3bb156f"),
    ("c4_1024x16_awc.yaml", None),
])
def test_baseline_configs_bit_exact(sim, gen_dir, name, golden):
    out = _compare(sim, _cfg(name), gen_dir)
    if golden:
        assert ref.sha256(out.report_json) == golden


VARIANTS = {
    "rr_lab": [("routing: random", "routing: rr"), ("kind: fifo", "kind: lab")],
    "jsq_dynamic": [("routing: random", "routing: jsq"), ("kind: static", "kind: dynamic")],
    "fused": [("kind: static", "kind: fused")],
    "jitter": [("jitter_ms: 0", "jitter_ms: 4")],
    "window_us": [("max_batch_size: 8", "max_batch_size: 3\n    batching_window_us: 1500")],
    "gen_seed": [("acceptance_rate: 0.8", "acceptance_rate: 0.3\n  gen_seed: 99")],
    "preset": [("prompt_median: 32\n  output_median: 72", "preset: cnndm-like")],
    "multi": [("targets: 1", "targets: 3"), ("drafts: 1", "drafts: 5"), ("routing: random", "routing: random"),
              ("jitter_ms: 0", "jitter_ms: 3"), ("rate_rps: 2", "rate_rps: 9")],
    "draft_batch": [("drafts: 1", "drafts: 4"), ("routing: random", "routing: jsq\n  draft_max_batch: 3")],
}


@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_policy_variants_bit_exact(sim, variant):
    text = _cfg("c1_single_pair.yaml")
    for a, b in VARIANTS[variant]:
        assert a in text
        text = text.replace(a, b, 1)
    _compare(sim, text)


@pytest.mark.parametrize("seed", [1, 7, 123456789, 2**63 + 5])
def test_seed_override(sim, seed):
    _compare(sim, _cfg("c2_8x1_batching.yaml"), seed=seed)


def test_trace_poisson_resampling(sim, gen_dir):
    text = _cfg("c4_1024x16_static.yaml").replace("mode: trace", "mode: poisson\n  rate_rps: 80")
    _compare(sim, text, gen_dir)


def test_sweep_summary_matches_reference(sim):
    spec = ("base: c2_8x1_batching.yaml\nseed: 7\nrepetitions: 3\naxes:\n"
            "  network.rtt_ms: [0, 10, 50]\n  policies.window.kind: [static, fused, dynamic]\n"
            "  policies.window.gamma: [2, 13]\n")
    js, cs = ref.run_sweep(spec, CFG, 4)
    out = sim.run_sweep(spec, base_dir=CFG)
    assert out.summary_json == js
    assert out.summary_csv == cs


def test_sweep_report_files_match_reference(sim, tmp_path):
    spec = "base: c1_single_pair.yaml\nseed: 3\nrepetitions: 2\naxes:\n  network.rtt_ms: [4, 30]\n"
    ref_dir, my_dir = tmp_path / "ref", tmp_path / "mine"
    ref.run_sweep(spec, CFG, 2, str(ref_dir))
    sim.run_sweep(spec, base_dir=CFG, out_dir=str(my_dir))
    ref_files = sorted(os.listdir(ref_dir))
    assert ref_files == sorted(os.listdir(my_dir))
    for f in ref_files:
        assert (ref_dir / f).read_bytes() == (my_dir / f).read_bytes(), f


def test_full_c5_sweep_matches_reference():
    """The benchmark workload itself at full size: the 65,536-replica C5 sweep
    (4,096 points x 16 repetitions, 8.8e8 events) through dsd_run_sweep must
    give the reference run_sweep's summary JSON/CSV byte for byte (the
    reference runs on all host cores, ~10 s)."""
    from paper_2511_21669_b200 import Simulator
    spec = open(os.path.join(CFG, "c5_sweep_65536.yaml")).read()
    js, cs = ref.run_sweep(spec, CFG, os.cpu_count() or 8)
    with Simulator(0) as s:
        out = s.run_sweep(spec, base_dir=CFG)
    assert (out.points, out.replicas, out.failed_points) == (4096, 65536, 0)
    assert out.events_processed == 880021538
    assert out.summary_json == js
    assert out.summary_csv == cs


def test_full_c5_per_replica_matches_reference():
    """Every one of the 65,536 C5 replicas, as the benchmark runs them (the
    specialised kernel with the session fast path, no record collection):
    events_processed, end_time and the RunAggregates (completed, throughput,
    mean TTFT / TPOT) must equal the reference run_sweep worker's bit for bit."""
    import numpy as np
    from paper_2511_21669_b200 import Simulator
    spec = open(os.path.join(CFG, "c5_sweep_65536.yaml")).read()
    rows = ref.sweep_replicas(spec, CFG, os.cpu_count() or 8, 65536)
    with Simulator(0) as s:
        n, _ = s.prepare_sweep(spec, base_dir=CFG)
        s.launch()
        s.sync()
        sm = s.summaries()
    assert n == 65536 and (sm["status"] == 0).all()
    np.testing.assert_array_equal(sm["events_processed"].astype(np.float64), rows[:, 0])
    np.testing.assert_array_equal(sm["end_time_us"].astype(np.float64), rows[:, 1])
    np.testing.assert_array_equal(sm["completed"].astype(np.float64), rows[:, 2])
    for k, f in ((3, "throughput_rps"), (4, "mean_ttft_ms"), (5, "mean_tpot_ms")):
        assert sm[f].tobytes() == rows[:, k].tobytes(), f


def test_large_sweep_parallel_aggregation_matches_reference():
    """A sweep above the host's parallel thresholds (4,096 replicas for the
    per-point sums, 1,024 points for the summary text): sums split across host
    threads at point boundaries (7 repetitions, so the raw split falls inside a
    point), failed points (max_batch_size 0) among them; the summaries must
    equal the reference's with any host thread count."""
    from paper_2511_21669_b200 import Simulator
    spec = ("base: c1_single_pair.yaml\nseed: 5\nrepetitions: 7\naxes:\n"
            "  policies.window.gamma: [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16]\n"
            "  network.rtt_ms: [2, 6, 10, 14, 20, 30, 45, 60]\n"
            "  policies.batching.max_batch_size: [0, 4, 8, 16]\n"
            "  workload.acceptance_rate: [0.6, 0.9]\n  workload.n_requests: [30]\n")
    js, cs = ref.run_sweep(spec, CFG, 8)
    for threads in ("16", "1"):
        os.environ["DSD_HOST_THREADS"] = threads
        try:
            with Simulator(0) as s:
                out = s.run_sweep(spec, base_dir=CFG)
        finally:
            del os.environ["DSD_HOST_THREADS"]
        assert (out.points, out.replicas, out.failed_points) == (1024, 768 * 7, 256)
        assert out.summary_json == js
        assert out.summary_csv == cs


def test_specialized_stack_overflow_reruns_on_hbm_variant(capfd):
    """The specialised kernel keeps a shorter action stack; a replica that
    overflows it fails with kFailStack and runs again - in the specialised
    kernel with the full stack and a larger heap, then (if it still fails) on
    the HBM variant.  DSD_SPEC_STACK_LIMIT=1 forces that for nearly every
    replica: the summaries must not change."""
    from paper_2511_21669_b200 import Simulator
    spec = ("base: c1_single_pair.yaml\nseed: 5\nrepetitions: 3\naxes:\n"
            "  policies.window.gamma: [1, 4, 9, 16]\n  network.rtt_ms: [2, 30]\n"
            "  workload.acceptance_rate: [0.5, 0.9]\n  workload.rate_rps: [2, 40]\n")
    js, cs = ref.run_sweep(spec, CFG, 4)
    os.environ.update({"DSD_SPEC_STACK_LIMIT": "1", "DSD_HOST_TIMING": "1"})
    try:
        with Simulator(0) as s:
            out = s.run_sweep(spec, base_dir=CFG)
    finally:
        del os.environ["DSD_SPEC_STACK_LIMIT"], os.environ["DSD_HOST_TIMING"]
    err = capfd.readouterr().err
    m = re.search(r"re-run in the shared-memory kernel \(\d+-slot heap\): (\d+) of (\d+) replicas", err)
    assert m and int(m.group(1)) > int(m.group(2)) // 2, err[-2000:]
    assert out.summary_json == js
    assert out.summary_csv == cs


@pytest.mark.parametrize("smem_heap", ["0", "2", "8"])
def test_kernel_variants_and_overflow_rerun(smem_heap):
    """HBM variant (0), shared-memory variant with forced heap overflow and
    HBM re-run (2), default shared-memory variant (8): identical results."""
    from paper_2511_21669_b200 import Simulator
    spec = ("base: c1_single_pair.yaml\nseed: 11\nrepetitions: 4\naxes:\n"
            "  network.jitter_ms: [0, 3]\n  policies.window.gamma: [1, 4, 9]\n"
            "  workload.rate_rps: [2, 30]\n")
    js, _ = ref.run_sweep(spec, CFG, 4)
    os.environ["DSD_SMEM_HEAP"] = smem_heap
    try:
        with Simulator(0) as s:
            out = s.run_sweep(spec, base_dir=CFG)
    finally:
        del os.environ["DSD_SMEM_HEAP"]
    assert out.summary_json == js


@pytest.mark.parametrize("smem_heap", ["7", "2"])
def test_specialized_kernel_matches_generic_and_reference(smem_heap):
    """A sweep whose every point is a single (target, draft) pair with a static
    window runs the specialised kernel (Engine::spec): its per-replica
    summaries must equal the generic kernel's bit for bit (DSD_SPECIALIZE=0),
    and its sweep summary the reference's; heap 2 forces overflow re-runs."""
    from paper_2511_21669_b200 import Simulator
    spec = ("base: c1_single_pair.yaml\nseed: 5\nrepetitions: 3\naxes:\n"
            "  policies.window.gamma: [1, 4, 9, 16]\n  network.rtt_ms: [2, 30]\n"
            "  workload.acceptance_rate: [0.5, 0.9]\n  workload.rate_rps: [2, 40]\n")
    js, _ = ref.run_sweep(spec, CFG, 4)
    sums = {}
    # (specialised kernel, cost-aware lane placement) on / off: the placement
    # only chooses which thread runs which replica
    for specialize, placement in (("1", "1"), ("0", "1"), ("1", "0")):
        os.environ["DSD_SPECIALIZE"] = specialize
        os.environ["DSD_PLACEMENT"] = placement
        os.environ["DSD_SMEM_HEAP"] = smem_heap
        try:
            with Simulator(0) as s:
                s.prepare_sweep(spec, base_dir=CFG)
                s.launch()
                s.sync()
                sums[specialize + placement] = s.summaries()
                assert s.run_sweep(spec, base_dir=CFG).summary_json == js
        finally:
            for k in ("DSD_SPECIALIZE", "DSD_PLACEMENT", "DSD_SMEM_HEAP"):
                del os.environ[k]
    assert len(sums["11"]) == 32 * 3
    assert (sums["11"]["status"] == 0).all()
    assert sums["11"].tobytes() == sums["01"].tobytes() == sums["10"].tobytes()


@pytest.mark.parametrize("env", [
    {"DSD_SOLO": "0"},  # the per-lane HBM / shared-memory variants
    {"DSD_SOLO": "2"},  # solo mode for the small topologies too
    {"DSD_SOLO_REC": "0"},  # solo mode with the records left in HBM
    {"DSD_SOLO_HEAP": "6", "DSD_HOST_TIMING": "1"},  # solo heap overflow -> HBM re-run
])
def test_solo_mode_matches_reference(env, gen_dir, tmp_path, capfd):
    """Batches of at most one wave of large-topology replicas run one replica
    per block (solo mode: servers, heap and records in shared memory); the
    single runs, a sweep summary and the per-point report files (records
    copied back for the export) must match the reference whichever variant
    runs them."""
    from paper_2511_21669_b200 import Simulator
    spec = ("base: c2_8x1_batching.yaml\nseed: 4\nrepetitions: 2\naxes:\n"
            "  network.rtt_ms: [1, 20]\n  policies.window.kind: [static, dynamic]\n")
    js, cs = ref.run_sweep(spec, CFG, 4, str(tmp_path / "ref"))
    os.environ.update(env)
    try:
        with Simulator(0) as s:
            for name in ("c2_8x1_batching.yaml", "c3_64x4_awc.yaml"):
                _compare(s, _cfg(name), gen_dir)
            _compare(s, _cfg("c1_single_pair.yaml"))
            out = s.run_sweep(spec, base_dir=CFG, out_dir=str(tmp_path / "mine"))
    finally:
        for k in env:
            del os.environ[k]
    assert (out.summary_json, out.summary_csv) == (js, cs)
    files = sorted(os.listdir(tmp_path / "ref"))
    assert files == sorted(os.listdir(tmp_path / "mine"))
    for f in files:
        assert (tmp_path / "ref" / f).read_bytes() == (tmp_path / "mine" / f).read_bytes(), f
    if "DSD_SOLO_HEAP" in env:
        m = re.findall(r"re-run on the HBM variant: (\d+) of (\d+) replicas", capfd.readouterr().err)
        assert m and max(int(a) for a, _ in m) > 0


def test_rewritten_input_files_are_read_again(sim, tmp_path):
    """A trace and a WC-DNN model rewritten at the same path between two calls
    on one handle: the second call must use the new contents (the reference
    re-reads every input in resolve_config, runner.cpp:96-134)."""
    trace = tmp_path / "t.jsonl"
    model = tmp_path / "m.json"
    text = _cfg("c1_single_pair.yaml").replace("kind: static", "kind: awc\n    model: m.json")
    text = text.replace("mode: poisson", "mode: trace\n  trace: t.jsonl")
    text = "\n".join(l for l in text.splitlines() if not l.strip().startswith(("rate_rps", "n_requests")))
    outs = []
    for k in range(2):
        trace.write_text(ref.gen_trace(3.0 + k, 40 + 10 * k, 0.6 + 0.2 * k, seed=11 + k))
        ref.random_model(str(model), seed=5 + k)
        outs.append(_compare(sim, text, str(tmp_path)))
    assert outs[0].report_json != outs[1].report_json


def test_long_batching_window_matches_reference(sim):
    """A batching window far longer than the service time with batches of 2:
    full-batch dispatches leave stale BatchReady timers pending
    (engine.cpp:508-519) - the case that can outgrow the HBM heap."""
    text = _cfg("c2_8x1_batching.yaml")
    for a, b in (("batching_window_us: 2000", "batching_window_us: 10000000"), ("max_batch_size: 8", "max_batch_size: 2"),
                 ("n_requests: 400", "n_requests: 20"), ("output_median: 72", "output_median: 400")):
        assert a in text
        text = text.replace(a, b)
    _compare(sim, text)


@pytest.mark.parametrize("cap", ["3", "6"])
def test_heap_overflow_retries_with_a_larger_heap(capfd, cap):
    """Replicas whose HBM event heap overflows run again with the heap
    doubled until they fit: forced here with a tiny heap
    (DSD_HEAP_CAP) on a generic-kernel sweep; the summaries must not change."""
    from paper_2511_21669_b200 import Simulator
    spec = ("base: c2_8x1_batching.yaml\nseed: 9\nrepetitions: 2\naxes:\n"
            "  network.rtt_ms: [2, 40]\n  policies.batching.max_batch_size: [2, 8]\n  workload.n_requests: [60]\n")
    js, cs = ref.run_sweep(spec, CFG, 4)
    os.environ.update({"DSD_HEAP_CAP": cap, "DSD_HOST_TIMING": "1"})
    try:
        with Simulator(0) as s:
            out = s.run_sweep(spec, base_dir=CFG)
    finally:
        del os.environ["DSD_HEAP_CAP"], os.environ["DSD_HOST_TIMING"]
    assert "event heap overflow" in capfd.readouterr().err
    assert out.summary_json == js and out.summary_csv == cs
