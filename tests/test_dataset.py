"""AWC dataset generation and window-policy evaluation on the GPU engine
(proj/src/awc/dataset.cpp) against the compiled reference.

Host-only parts (build_scenarios, the seeded split, the JSONL format) run on
CPU; generate_dataset / eval_policy_on_scenarios run the sm_100a engine with
the feature probe and must reproduce the reference's text byte for byte.
"""
import json

import pytest

import reforacle as ref
from paper_2511_21669_b200 import ConfigError, build_scenarios

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")

# DatasetGrid variants: the reference's defaults (== proj/configs/dataset_grid.yaml),
# and the small grids of test_awc.cpp:280-330
GRID_DEFAULT = ""
GRID_FOUR = ("rtt_ms: [5, 40]\nalpha: [0.4, 0.9]\nload_factor: [0.5]\ndrafts: [2]\ncost_ratio: [0.1]\n"
             "n_requests: 12\n")
GRID_ONE = "rtt_ms: [4]\nalpha: [0.95]\nload_factor: [0.5]\ndrafts: [2]\ncost_ratio: [0.1]\nn_requests: 20\n"
GRID_MIXED = ("rtt_ms: [2, 30, 100]\nalpha: [0.3, 0.85]\nload_factor: [0.35, 0.8]\ndrafts: [1, 6]\n"
              "cost_ratio: [0.15]\nn_requests: 24\nseed: 7\n")


@needs_ref
@pytest.mark.parametrize("grid", [GRID_DEFAULT, GRID_FOUR, GRID_ONE, GRID_MIXED])
def test_build_scenarios_matches_reference(grid):
    assert build_scenarios(grid) == ref.build_scenarios(grid)


def test_build_scenarios_split_and_seeds():
    lines = [json.loads(x) for x in build_scenarios("").splitlines()]
    assert len(lines) == 200
    splits = [x["split"] for x in lines]
    assert (splits.count("train"), splits.count("val"), splits.count("test")) == (160, 20, 20)
    assert [x["scenario_id"] for x in lines] == list(range(200))
    assert len({x["seed"] for x in lines}) == 200
    # jitter is 10% of rtt from 4 ms up (dataset.cpp:60)
    assert all(x["jitter_ms"] == (x["rtt_ms"] * 0.1 if x["rtt_ms"] >= 4 else 0.0) for x in lines)


def test_build_scenarios_rejects_bad_grid():
    with pytest.raises(ConfigError):
        build_scenarios("drafts: [two]\n")


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("grid", [GRID_FOUR, GRID_ONE, GRID_MIXED])
def test_generate_dataset_matches_reference(sim, grid):
    ds, sc = sim.generate_dataset(grid)
    rds, rsc = ref.generate_dataset(grid)
    assert sc == rsc
    assert ds == rds


@pytest.mark.gpu
@needs_ref
def test_generate_dataset_default_grid_matches_reference(sim):
    """The full 200-scenario x 12-candidate dataset (`specsim gen-dataset`)."""
    ds, sc = sim.generate_dataset("")
    rds, rsc = ref.generate_dataset("")
    assert len(ds.splitlines()) == 2400
    assert sc == rsc
    assert ds == rds


@pytest.mark.gpu
def test_dataset_label_dominates_candidates(sim):
    """test_awc.cpp:309-330: the label's objective is the scenario minimum."""
    ds, _ = sim.generate_dataset(GRID_FOUR)
    rows = [json.loads(x) for x in ds.splitlines()]
    assert len(rows) == 4 * 12
    by = {}
    for r in rows:
        by.setdefault(r["scenario_id"], []).append(r)
    for cands in by.values():
        assert [c["candidate_gamma"] for c in cands] == list(range(2, 13)) + [1]
        assert cands[-1]["candidate_mode"] == "fused"
        label = cands[0]["label_gamma"]
        best = min(c["objective"] for c in cands if c["candidate_gamma"] == label)
        assert all(best <= c["objective"] + 1e-12 for c in cands)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("kind,gamma", [("static", 4), ("static", 9), ("dynamic", 4), ("fused", 4)])
def test_eval_policy_matches_reference(sim, kind, gamma):
    sc = build_scenarios(GRID_MIXED)
    assert sim.eval_policy(sc, kind, gamma, split="all") == {
        "policy": kind, **dict(zip(["throughput_rps", "mean_ttft_ms", "mean_tpot_ms", "mean_gamma"],
                                   ref.eval_policy(sc, kind, gamma, split="all")))}


@pytest.mark.gpu
@needs_ref
def test_eval_policy_awc_matches_reference(sim, gen_dir):
    """The `specsim eval-policy` comparison on the default grid's test split with
    the reference-trained model (AWC decisions run the FP64 MLP on device)."""
    import os
    model = os.path.join(gen_dir, "model.json")
    sc = build_scenarios("")
    ours = sim.eval_policy(sc, "awc", 4, model, split="test")
    theirs = ref.eval_policy(sc, "awc", 4, model, split="test")
    assert [ours["throughput_rps"], ours["mean_ttft_ms"], ours["mean_tpot_ms"], ours["mean_gamma"]] == theirs


@pytest.mark.gpu
def test_eval_policy_empty_split_is_config_error(sim):
    sc = build_scenarios(GRID_ONE)
    with pytest.raises(ConfigError, match="no scenarios with split 'val'"):
        sim.eval_policy(sc, "static", 4, split="val")
