"""Python mirror of the reference's simulate-a-sweep API over libdsdsim.so.

Names and semantics follow the reference C++ API
(proj/include/specsim/runner/runner.hpp:36-60, runner/sweep.hpp:17-50):

    run_simulation(config)  -> SimulationOutput   (resolve_config + run_simulation + aggregate_run)
    run_sweep(spec, out_dir) -> SweepOutput       (SweepSpec::from_node + run_sweep + summaries)
    sweep_point_seed(base, point_id, rep)         (sweep.cpp:51-57)

Errors raise ConfigError (reference ParseError / ConfigError / ValidationError /
UnknownProfileKey / CorruptModelFile, CLI exit code 2) or EngineError (every
other failure, exit code 3), carrying the reference's message text.
All simulation work runs in the sm_100a kernels; there is no CPU fallback.
"""
import ctypes
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import RequestRecord, ReplicaSummary

SUMMARY_DTYPE = np.dtype([
    ("events_processed", "<u8"), ("end_time_us", "<i8"), ("completed", "<i8"), ("first_arrival_us", "<i8"),
    ("last_completion_us", "<i8"), ("net_queue_wait_total_us", "<i8"), ("net_queue_wait_count", "<i8"),
    ("n_requests", "<i8"), ("throughput_rps", "<f8"), ("mean_ttft_ms", "<f8"), ("mean_tpot_ms", "<f8"),
    ("has_duration", "<i4"), ("status", "<i4"),
])
assert SUMMARY_DTYPE.itemsize == ctypes.sizeof(ReplicaSummary)


class DsdError(Exception):
    code = _lib.DSD_ERR_RUNTIME

    def __init__(self, message, code=None):
        super().__init__(message)
        self.message = message
        if code is not None:
            self.code = code


class ConfigError(DsdError):
    code = _lib.DSD_ERR_CONFIG


class EngineError(DsdError):
    code = _lib.DSD_ERR_RUNTIME


def _check(rc, err):
    if rc == _lib.DSD_OK:
        return
    msg = err.value.decode(errors="replace")
    if rc == _lib.DSD_ERR_CONFIG:
        raise ConfigError(msg, rc)
    raise EngineError(msg, rc)


def _take(ptr):
    if not ptr:
        return None
    s = ctypes.cast(ptr, ctypes.c_char_p).value.decode()
    _lib.lib().dsd_free(ptr)
    return s


def _text(config):
    """Accept YAML text or a path to a YAML file."""
    if os.path.exists(config) and "\n" not in config:
        with open(config) as f:
            return f.read(), os.path.dirname(os.path.abspath(config)) or "."
    return config, None


@dataclass
class SimulationOutput:
    """SimulationOutput (runner.hpp:46-51) + RunAggregates (runner.hpp:53-60)."""
    report_json: str
    report_csv: Optional[str]
    events_processed: int
    end_time_us: int
    completed: int
    throughput_rps: float
    mean_ttft_ms: float
    mean_tpot_ms: float


@dataclass
class SweepOutput:
    summary_json: str
    summary_csv: str
    points: int
    replicas: int
    failed_points: int
    events_processed: int


class Simulator:
    """One libdsdsim handle: one CUDA device (dsd_create) or a list of them
    (dsd_create_devices; every batch / sweep is spread over all of them and
    its results come back in replica order, as on one device)."""

    def __init__(self, device=0):
        L = _lib.lib()
        self._L = L
        self._h = ctypes.c_void_p()
        err = ctypes.create_string_buffer(1024)
        devices = [int(d) for d in device] if isinstance(device, (list, tuple)) else [int(device)]
        arr = (ctypes.c_int * len(devices))(*devices)
        _check(L.dsd_create_devices(arr, len(devices), ctypes.byref(self._h), err, 1024), err)
        self.devices = devices
        self.device = devices[0]

    # ---- lifecycle ----
    def close(self):
        if self._h:
            self._L.dsd_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- reference-facing API ----
    def run_simulation(self, config: str, base_dir: Optional[str] = None, seed: Optional[int] = None,
                       strict: bool = True, csv: bool = False, report: bool = True) -> SimulationOutput:
        text, d = _text(config)
        base_dir = base_dir or d or "."
        c = ctypes
        rep, rcsv = c.c_void_p(), c.c_void_p()
        ev, end = c.c_uint64(), c.c_int64()
        agg = (c.c_double * 4)()
        err = c.create_string_buffer(4096)
        rc = self._L.dsd_run_simulation(self._h, text.encode(), base_dir.encode(), int(strict), int(seed is not None),
                                        seed or 0, c.byref(rep) if report else None,
                                        c.byref(rcsv) if csv else None, c.byref(ev), c.byref(end), agg, err, 4096)
        _check(rc, err)
        return SimulationOutput(_take(rep) if report else None, _take(rcsv) if csv else None, ev.value, end.value,
                                int(agg[0]), agg[1], agg[2], agg[3])

    def run_simulation_traced(self, config: str, base_dir: Optional[str] = None, seed: Optional[int] = None,
                              strict: bool = True):
        """`specsim run --event-log`: (report_json, event_log text, busy intervals
        [(role 't'|'d', server id, start_us, end_us)], events_processed) with
        EngineOptions::collect_event_log (engine.hpp:32-35)."""
        text, d = _text(config)
        base_dir = base_dir or d or "."
        c = ctypes
        rep, log = c.c_void_p(), c.c_void_p()
        n_iv, ev = c.c_int64(), c.c_uint64()
        err = c.create_string_buffer(4096)
        _check(self._L.dsd_run_simulation_traced(self._h, text.encode(), base_dir.encode(), int(strict),
                                                 int(seed is not None), seed or 0, c.byref(rep), c.byref(log), None,
                                                 0, c.byref(n_iv), c.byref(ev), err, 4096), err)
        report, log_text = _take(rep), _take(log)
        # the intervals from the same run (kept by the handle until the next batch)
        buf = (_lib.BusyInterval * max(1, n_iv.value))()
        _check(self._L.dsd_fetch_event_log(self._h, 0, None, buf, n_iv.value, c.byref(n_iv), err, 4096), err)
        iv = [("d" if b.role else "t", b.server_id, b.start_us, b.end_us) for b in buf[:n_iv.value]]
        return report, log_text, iv, ev.value

    def run_sweep(self, spec: str, base_dir: Optional[str] = None, out_dir: str = "") -> SweepOutput:
        text, d = _text(spec)
        base_dir = base_dir or d or "."
        c = ctypes
        js, cs = c.c_void_p(), c.c_void_p()
        tot = (c.c_double * 4)()
        err = c.create_string_buffer(4096)
        rc = self._L.dsd_run_sweep(self._h, text.encode(), base_dir.encode(), out_dir.encode(), c.byref(js),
                                   c.byref(cs), tot, err, 4096)
        _check(rc, err)
        return SweepOutput(_take(js), _take(cs), int(tot[0]), int(tot[1]), int(tot[2]), int(tot[3]))

    # ---- device-resident batch (benchmarking, multi-GPU shards) ----
    def prepare_sweep(self, spec: str, base_dir: Optional[str] = None, shard: int = 0, n_shards: int = 1):
        text, d = _text(spec)
        base_dir = base_dir or d or "."
        c = ctypes
        nrep, npts = c.c_int64(), c.c_int64()
        err = c.create_string_buffer(4096)
        _check(self._L.dsd_prepare_sweep(self._h, text.encode(), base_dir.encode(), shard, n_shards,
                                         c.byref(nrep), c.byref(npts), err, 4096), err)
        self.n_replicas = nrep.value
        return nrep.value, npts.value

    def launch(self):
        err = ctypes.create_string_buffer(1024)
        _check(self._L.dsd_batch_launch(self._h, err, 1024), err)

    def sync(self):
        err = ctypes.create_string_buffer(1024)
        _check(self._L.dsd_batch_sync(self._h, err, 1024), err)

    def summaries(self, n: Optional[int] = None) -> np.ndarray:
        n = self.n_replicas if n is None else n
        out = np.zeros(n, dtype=SUMMARY_DTYPE)
        err = ctypes.create_string_buffer(1024)
        _check(self._L.dsd_batch_summaries(self._h, out.ctypes.data_as(ctypes.POINTER(ReplicaSummary)), n,
                                           err, 1024), err)
        return out

    def device_summaries(self):
        """(device pointer, bytes) of the prepared batch's summary array."""
        p, b = ctypes.c_void_p(), ctypes.c_size_t()
        if self._L.dsd_batch_device_summaries(self._h, ctypes.byref(p), ctypes.byref(b)) != 0:
            raise EngineError("no prepared batch")
        return p.value, b.value

    def shard_sizes(self):
        """Replicas of the prepared batch on each of the handle's devices."""
        buf = (ctypes.c_int64 * 64)()
        n = self._L.dsd_batch_shard_sizes(self._h, buf, 64)
        return [int(buf[k]) for k in range(n)]

    def stream(self) -> int:
        return self._L.dsd_stream(self._h) or 0

    def last_launch_count(self) -> int:
        return int(self._L.dsd_last_launch_count(self._h))

    def last_transfer_bytes(self):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        self._L.dsd_last_transfer_bytes(self._h, ctypes.byref(a), ctypes.byref(b))
        return a.value, b.value

    def last_kernel_ms(self):
        a, b, t = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        self._L.dsd_last_kernel_ms(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(t))
        return {"sim_ms": a.value, "stage_ms": b.value, "total_ms": t.value}

    # ---- AWC dataset generation / policy evaluation (dataset.cpp) ----
    def generate_dataset(self, grid: str = "", weights=None):
        """`specsim gen-dataset`: (dataset.jsonl text, scenarios.jsonl text) for a
        DatasetGrid YAML document or file ("" = DatasetGrid defaults); weights =
        (w_tpot, w_ttft, w_throughput) or None for ObjectiveWeights{}."""
        text, _ = _text(grid) if grid else ("", None)
        c = ctypes
        ds, sc = c.c_void_p(), c.c_void_p()
        w = (c.c_double * 3)(*weights) if weights is not None else None
        err = c.create_string_buffer(4096)
        _check(self._L.dsd_generate_dataset(self._h, text.encode(), w, c.byref(ds), c.byref(sc), err, 4096), err)
        return _take(ds), _take(sc)

    def eval_policy(self, scenarios_jsonl: str, window_kind: str, gamma: int = 4, model_path: str = "",
                    split: str = "all") -> dict:
        """eval_policy_on_scenarios over the scenarios of `split`."""
        c = ctypes
        out = (c.c_double * 4)()
        err = c.create_string_buffer(4096)
        _check(self._L.dsd_eval_policy(self._h, scenarios_jsonl.encode(), split.encode(), window_kind.encode(), gamma,
                                       model_path.encode(), out, err, 4096), err)
        return {"policy": window_kind, "throughput_rps": out[0], "mean_ttft_ms": out[1], "mean_tpot_ms": out[2],
                "mean_gamma": out[3]}

    def probe(self, n: Optional[int] = None) -> np.ndarray:
        """[n, DSD_PROBE_FIELDS] feature-probe sums of the last probed batch."""
        n = self.n_replicas if n is None else n
        out = np.zeros((n, _lib.DSD_PROBE_FIELDS), dtype=np.float64)
        err = ctypes.create_string_buffer(1024)
        _check(self._L.dsd_batch_probe(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n, err, 1024),
               err)
        return out


_default: Optional[Simulator] = None


def default_simulator() -> Simulator:
    global _default
    if _default is None:
        _default = Simulator(0)
    return _default


def run_simulation(config: str, base_dir: Optional[str] = None, seed: Optional[int] = None, strict: bool = True,
                   csv: bool = False) -> SimulationOutput:
    return default_simulator().run_simulation(config, base_dir, seed, strict, csv)


def run_sweep(spec: str, base_dir: Optional[str] = None, out_dir: str = "") -> SweepOutput:
    return default_simulator().run_sweep(spec, base_dir, out_dir)


def sweep_point_seed(base_seed: int, point_id: str, repetition: int) -> int:
    return int(_lib.lib().dsd_sweep_point_seed(base_seed, point_id.encode(), repetition))


def build_scenarios(grid: str = "") -> str:
    """build_scenarios + serialize_scenarios (host only): scenarios.jsonl text
    for a DatasetGrid YAML document or file ("" = the defaults)."""
    text, _ = _text(grid) if grid else ("", None)
    p = ctypes.c_void_p()
    err = ctypes.create_string_buffer(4096)
    _check(_lib.lib().dsd_build_scenarios(text.encode(), ctypes.byref(p), err, 4096), err)
    return _take(p)
