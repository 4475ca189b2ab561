"""Randomised parity: seeded random configs (topology sizes and groups with
link overrides, routing / batching / window policies incl. AWC, batching
windows, jitter, presets, gen_seed, profiles) run on the GPU engine and on the
reference (oracle/_ref) must give identical report bytes, events_processed,
end_time and aggregates; random sweeps must give identical summaries.  The
configs reach every kernel variant: the single-pair specialisation, the
shared-memory variant (<= 4 servers) and the HBM variant."""
import os
import random

import pytest

import reforacle as ref

pytestmark = pytest.mark.gpu


def _yaml(obj, indent=0):
    pad = "  " * indent
    out = []
    for k, v in obj.items():
        if isinstance(v, dict):
            out.append(f"{pad}{k}:")
            out.append(_yaml(v, indent + 1))
        elif isinstance(v, list):
            out.append(f"{pad}{k}:")
            for item in v:
                lines = _yaml(item, indent + 2).split("\n")
                out.append(f"{pad}  - " + lines[0].strip())
                out.extend(lines[1:])
        else:
            out.append(f"{pad}{k}: {v}")
    return "\n".join(out)


def _pool(rng, lo, hi):
    if rng.random() < 0.35:
        return [{"count": rng.randint(1, max(1, hi // 2))} for _ in range(rng.randint(1, 2))]
    return rng.randint(lo, hi)


def _count(pool):
    return sum(g["count"] for g in pool) if isinstance(pool, list) else pool


# DSD_FUZZ_BIG=1: larger topologies and workloads (a longer campaign);
# DSD_FUZZ_SEED: offset of the case seeds
BIG = os.environ.get("DSD_FUZZ_BIG") == "1"
SEED0 = int(os.environ.get("DSD_FUZZ_SEED", "0"))


def random_config(rng, awc_model=None):
    targets = _pool(rng, 1, 8 if BIG else 3)
    drafts = _pool(rng, 0, 40 if BIG else 6)
    rtt = rng.choice([0, 1, 4, 10, 30])
    net = {"rtt_ms": rtt, "jitter_ms": round(rng.random() * rtt, 2) if rng.random() < 0.5 else 0}
    if isinstance(targets, list) and isinstance(drafts, list) and rng.random() < 0.6:
        ov = []
        for dg in range(len(drafts)):
            for tg in range(len(targets)):
                if rng.random() < 0.5:
                    r = rng.choice([1, 5, 20, 60])
                    ov.append({"draft_group": dg, "target_group": tg, "rtt_ms": r,
                               "jitter_ms": round(rng.random() * r * 0.3, 2)})
        if ov:
            net["overrides"] = ov
    batching = {"kind": rng.choice(["fifo", "lab"]), "max_batch_size": rng.randint(1, 8)}
    if batching["kind"] == "lab":
        batching["similarity_fraction"] = rng.choice([0, 0.2, 0.5, 1.5])
    if rng.random() < 0.3:
        batching["batching_window_us"] = rng.choice([300, 1500, 5000])
    kinds = ["static", "dynamic", "fused"] + (["awc"] if awc_model and _count(drafts) > 0 else [])
    window = {"kind": rng.choice(kinds), "gamma": rng.randint(1, 8)}
    if window["kind"] == "dynamic" or rng.random() < 0.3:
        window["gamma_min"] = rng.randint(1, 2)
        window["gamma_max"] = rng.randint(window["gamma_min"] + 1, 12)
        window["gamma"] = min(max(window["gamma"], window["gamma_min"]), window["gamma_max"])
    if window["kind"] == "awc":
        window["model"] = awc_model
    pol = {"routing": rng.choice(["random", "rr", "jsq"]), "batching": batching, "window": window}
    if rng.random() < 0.3:
        pol["draft_max_batch"] = rng.randint(1, 4)
    if rng.random() < 0.2:
        pol["queue_capacity"] = rng.choice([4, 16, 64])
    wl = {"mode": "poisson", "rate_rps": rng.choice([0.5, 2, 8, 30]), "n_requests": rng.randint(1, 250 if BIG else 40),
          "acceptance_rate": round(rng.random(), 2)}
    if rng.random() < 0.25:
        wl["preset"] = rng.choice(["gsm8k-like", "cnndm-like", "humaneval-like"])
    else:
        wl["prompt_median"] = rng.randint(4, 64)
        wl["output_median"] = rng.randint(1, 96)
    if rng.random() < 0.25:
        wl["gen_seed"] = rng.randint(0, 2**31)
    synth = {"target_decode_ms": rng.choice([5, 15, 25]), "cost_ratio": rng.choice([0.05, 0.1, 0.3])}
    if rng.random() < 0.3:
        synth["batch_coef"] = rng.choice([0, 0.05, 0.2])
        synth["context_coef"] = rng.choice([0, 0.3, 1.0])
    cfg = {"targets": targets, "drafts": drafts, "network": net, "policies": pol, "workload": wl,
           "seed": rng.randint(0, 2**40), "latency_profile": {"synth": synth}}
    return _yaml(cfg) + "\n"


@pytest.mark.parametrize("case", range(int(os.environ.get("DSD_FUZZ_CASES", "48"))))
def test_random_config_bit_exact(sim, gen_dir, case):
    rng = random.Random(1000 + SEED0 + case)
    text = random_config(rng, awc_model=os.path.join(gen_dir, "model.json"))
    try:
        rep, ev, end, agg = ref.run_config(text, gen_dir, None)
    except ref.RefError as e:  # the reference rejects it: so must we, with the same class
        from paper_2511_21669_b200 import ConfigError, EngineError
        with pytest.raises(ConfigError if e.code == 2 else EngineError):
            sim.run_simulation(text, base_dir=gen_dir)
        return
    out = sim.run_simulation(text, base_dir=gen_dir)
    assert (out.events_processed, out.end_time_us) == (ev, end), text
    assert out.report_json == rep, text
    assert (out.completed, out.throughput_rps, out.mean_ttft_ms, out.mean_tpot_ms) == (int(agg[0]), agg[1], agg[2],
                                                                                       agg[3])


@pytest.mark.parametrize("case", range(int(os.environ.get("DSD_FUZZ_SWEEPS", "6"))))
def test_random_sweep_summary_matches_reference(sim, gen_dir, case, tmp_path):
    """Batched: a random base config swept over two axes x repetitions (many
    replicas per warp, lane placement, specialised kernel when eligible)."""
    rng = random.Random(2000 + SEED0 + case)
    base = random_config(rng, awc_model=os.path.join(gen_dir, "model.json"))
    (tmp_path / "base.yaml").write_text(base)
    axes = rng.sample([("network.rtt_ms", [1, 10, 40]), ("workload.acceptance_rate", [0.3, 0.7, 0.95]),
                       ("workload.rate_rps", [1, 6, 20]), ("policies.batching.max_batch_size", [1, 4, 8])], 2)
    spec = f"base: base.yaml\nseed: {rng.randint(0, 999)}\nrepetitions: {rng.randint(2, 9)}\naxes:\n" + "".join(
        f"  {k}: [{', '.join(str(v) for v in vals)}]\n" for k, vals in axes)
    try:
        js, cs = ref.run_sweep(spec, str(tmp_path), 4)
    except ref.RefError:
        pytest.skip("the reference rejects this random sweep")
    out = sim.run_sweep(spec, base_dir=str(tmp_path))
    assert out.summary_json == js, base
    assert out.summary_csv == cs
