"""Latency-profile files with real (model, hardware) keys through the GPU
engine (VERDICT r1 missing #5).  LatencyProfile::parse
(proj/src/latency/profile.cpp:190-211) reads `entries` of (model, hardware,
op, calibration, batch_axis, context_axis, values_ms); every device group
picks its grids by its own `model` / `hardware` keys (topology.hpp:14-21,
topology.cpp:33-41), and predict() interpolates them (profile.cpp:129-151).
The reports must equal the reference's byte for byte."""
import json
import math
import os

import pytest

import reforacle as ref

pytestmark = pytest.mark.gpu

KEYS = {  # (model, hardware): (decode ms scale, prefill ms per token)
    ("llama-70b", "h100-sxm"): (14.0, 0.11),
    ("llama-70b", "a100-40g"): (23.5, 0.19),
    ("llama-1b", "jetson-orin"): (3.1, 0.05),
    ("llama-1b", "rtx-4090"): (1.7, 0.02),
}


def profile_json(context_top=8192.0, odd_axes=False):
    """A profile file: irregular axes, calibration != 1, values with full mantissas."""
    batch = [1.0, 2.0, 3.0, 4.0, 8.0, 16.0, 32.0, 64.0] if not odd_axes else [1.0, 1.5, 2.75, 6.0, 12.5, 40.0]
    ctx = [1.0, 64.0, 128.0, 384.0, 1024.0, 2048.0, 4096.0, context_top]
    entries = []
    for (model, hw), (dec, pre) in sorted(KEYS.items()):
        for op in ("decode", "prefill"):
            vals = []
            for b in batch:
                for c in ctx:
                    if op == "decode":
                        v = dec * (1.0 + 0.047 * math.log2(b)) * (1.0 + 0.31 * c / 4096.0) + 0.013 * math.sqrt(c)
                    else:
                        v = pre * c * (1.0 + 0.09 * (b - 1.0)) + 0.7 + 1.0 / (3.0 + b)
                    vals.append(v)
            entries.append({"model": model, "hardware": hw, "op": op,
                            "calibration": 1.0 + (len(entries) % 3) * 0.0625 + 1.0 / 3.0 * 1e-3,
                            "batch_axis": batch, "context_axis": ctx, "values_ms": vals})
    return json.dumps({"meta": {"units": "ms", "axes": "batch_size x context_length", "note": "test"},
                       "entries": entries}, indent=1)


CONFIG = """targets:
  - count: 2
    model: llama-70b
    hardware: h100-sxm
  - count: 1
    model: llama-70b
    hardware: a100-40g
drafts:
  - count: 3
    model: llama-1b
    hardware: jetson-orin
  - count: 2
    model: llama-1b
    hardware: rtx-4090
network:
  rtt_ms: 12
  jitter_ms: 1.5
policies:
  routing: jsq
  batching:
    kind: fifo
    max_batch_size: 4
  window:
    kind: dynamic
    gamma: 4
workload:
  mode: poisson
  rate_rps: 6
  n_requests: 150
  acceptance_rate: 0.75
  prompt_median: 200
  output_median: 90
seed: 7
latency_profile: prof.json
"""

PAIR = """targets:
  - count: 1
    model: llama-70b
    hardware: a100-40g
drafts:
  - count: 1
    model: llama-1b
    hardware: rtx-4090
network:
  rtt_ms: 20
  jitter_ms: 0
policies:
  routing: random
  batching:
    kind: fifo
    max_batch_size: 8
  window:
    kind: static
    gamma: 5
workload:
  mode: poisson
  rate_rps: 3
  n_requests: 80
  acceptance_rate: 0.7
  prompt_median: 300
  output_median: 120
seed: 3
latency_profile: prof.json
"""


@pytest.mark.parametrize("context_top,odd", [(8192.0, False), (131072.0, False), (8192.0, True)])
def test_heterogeneous_profile_file_matches_reference(sim, tmp_path, context_top, odd):
    """Two target and two draft hardware types; a context axis past the
    device's segment tables (131072: binary search) and non-integer batch
    axes."""
    (tmp_path / "prof.json").write_text(profile_json(context_top, odd))
    rep, ev, end, _ = ref.run_config(CONFIG, str(tmp_path))
    out = sim.run_simulation(CONFIG, base_dir=str(tmp_path))
    assert (out.events_processed, out.end_time_us) == (ev, end)
    assert out.report_json == rep


def test_profile_file_sweep_through_the_specialised_kernel(sim, tmp_path):
    """A single-pair sweep over a profile file (the specialised kernel and
    its session latency tables) against the reference run_sweep."""
    (tmp_path / "prof.json").write_text(profile_json())
    (tmp_path / "pair.yaml").write_text(PAIR)
    spec = ("base: pair.yaml\nseed: 11\nrepetitions: 4\naxes:\n  policies.window.gamma: [1, 3, 8]\n"
            "  network.rtt_ms: [4, 40]\n")
    js, cs = ref.run_sweep(spec, str(tmp_path), 4)
    out = sim.run_sweep(spec, base_dir=str(tmp_path))
    assert out.failed_points == 0
    assert out.summary_json == js and out.summary_csv == cs
