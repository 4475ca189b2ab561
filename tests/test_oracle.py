"""CPU tests that pin the oracle before it is trusted (no GPU).

1. the reference oracle (oracle/_ref, the real reference library) reproduces
   the golden values recorded in SURVEY.md §8(c) / Appendix C;
2. the C restatement (oracle/dsd_oracle.c) reproduces the reference byte for
   byte on the golden configs and on policy variants."""
import os

import pytest

import reforacle as ref
import restate

pytestmark = pytest.mark.skipif(not ref.available(), reason="reference oracle not built")
CFG = ref.CONFIGS


def _cfg(name):
    with open(os.path.join(CFG, name)) as f:
        return f.read()


# ---- reference golden vectors ------------------
def test_fnv_labels():
    L = ref.lib()
    assert L.ref_fnv1a64(b"arrivals", 8, 0xcbf29ce484222325) == 0xb10bc22ca203cc53
    assert L.ref_fnv1a64(b"jitter", 6, 0xcbf29ce484222325) == 0x2e701e89a7ab0cd3
    assert L.ref_fnv1a64(b"accept-bits", 11, 0xcbf29ce484222325) == 0x78ad23fe9688e42c


def test_rng_and_net_delay_goldens():
    import ctypes
    L = ref.lib()
    u = (ctypes.c_uint64 * 4)()
    L.ref_rng_u64(42, b"arrivals", u, 4)
    assert set(u) == {4826540322874552481, 461399563008123880, 6246729661996744084, 3334472219076958205}
    d = (ctypes.c_double * 3)()
    L.ref_rng_unit(42, b"jitter", d, 3)
    assert sorted(d) == sorted([0.39306529634601362, 0.83489794432545317, 0.78364176904357485])
    nd = (ctypes.c_int64 * 3)()
    L.ref_net_delay(30.0, 4.0, 7, nd, 3)
    assert sorted(nd) == [15428, 16135, 16236]


def test_sweep_seed_golden():
    from paper_2511_21669_b200 import sweep_point_seed
    pid = "network.rtt_ms=2;policies.window.gamma=1;workload.acceptance_rate=0.5"
    assert ref.lib().ref_sweep_point_seed(42, pid.encode(), 0) == 156043105876269134
    for rep in range(4):
        assert sweep_point_seed(42, pid, rep) == ref.lib().ref_sweep_point_seed(42, pid.encode(), rep)


def test_generated_fixture_hashes(gen_dir):
    h = {k: ref.sha256(open(os.path.join(gen_dir, k), "rb").read()) for k in ("mixed.jsonl", "model.json")}
    assert h["mixed.jsonl"] == "697cc3b44876736b5c0b18cb0e9a8e7971b3a23e3c5e0ef7fb8ddac9f5b3f4dc"
    assert h["model.json"] == "3f00e5cc2c0484e5cea2fa7f7e019dd4fb697be3bbbf933866f2ad001dba104a"


GOLDEN = [
    ("c1_single_pair.yaml", 12192, 84554872, "12253632ad5d73e55984bf1b64a17e8b4cb966f1c137e65367a1d78f228ed7ce"),
    ("c2_8x1_batching.yaml", 45417, 91387860, "cb0d409d66afb46dab47f25590fb30a3f8f6f88531bfd088b640837eb4bf90a1"),
    ("c3_64x4_awc.yaml", 80739, 76807981, "eb1dbe06b534b6e52dde1a7da752cf91abac9712e5005936bff30af8a197bdb3"),
    ("c4_1024x16_static.yaml", 904698, 138015287,
     "3b4a3e55b3f2f45bb5d613e107b06605735cd1ed21f102516c28a816b3bb156f"),
]


@pytest.mark.parametrize("name,events,end,sha", GOLDEN)
def test_reference_reproduces_appendix_c(gen_dir, name, events, end, sha):
    rep, ev, t_end, _ = ref.run_config(_cfg(name), gen_dir)
    assert (ev, t_end, ref.sha256(rep)) == (events, end, sha)


# ---- restatement vs reference ---------------------------------------------
@pytest.mark.parametrize("name", ["c1_single_pair.yaml", "c2_8x1_batching.yaml", "c3_64x4_awc.yaml",
                                  "c4_1024x16_static.yaml", "c4_1024x16_awc.yaml"])
def test_restatement_matches_reference(gen_dir, name):
    text = _cfg(name)
    rep, ev, end, agg = ref.run_config(text, gen_dir)
    mine, s = restate.oracle_report(text, gen_dir)
    assert s.events_processed == ev and s.end_time_us == end
    assert mine == rep
    assert (s.throughput_rps, s.mean_ttft_ms, s.mean_tpot_ms) == (agg[1], agg[2], agg[3])


VARIANTS = [
    [("routing: random", "routing: rr"), ("kind: fifo", "kind: lab"), ("targets: 1", "targets: 2")],
    [("routing: random", "routing: jsq"), ("kind: static", "kind: dynamic"), ("drafts: 1", "drafts: 3")],
    [("kind: static", "kind: fused")],
    [("jitter_ms: 0", "jitter_ms: 6"), ("rate_rps: 2", "rate_rps: 20")],
    [("max_batch_size: 8", "max_batch_size: 2\n    batching_window_us: 700"), ("drafts: 1", "drafts: 6")],
    [("prompt_median: 32\n  output_median: 72", "preset: humaneval-like\n  gen_seed: 5")],
]


@pytest.mark.parametrize("k", range(len(VARIANTS)))
def test_restatement_policy_variants(k):
    text = _cfg("c1_single_pair.yaml")
    for a, b in VARIANTS[k]:
        text = text.replace(a, b, 1)
    rep, ev, end, _ = ref.run_config(text)
    mine, s = restate.oracle_report(text)
    assert s.events_processed == ev
    assert mine == rep
