"""ctypes binding of libdsdsim.so (include/dsdsim.h).

The shared library is built in-tree (``paper_2511_21669_b200/libdsdsim.so``)
by ``__graft_entry__.build()``.  There is no Python or CPU fallback: if the
library or a GPU is missing, every entry point raises.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# DSD_LIB: load another build of the same library (A/B timing of kernel variants).
LIB_PATH = os.environ.get("DSD_LIB") or os.path.join(HERE, "libdsdsim.so")

DSD_OK = 0
DSD_ERR_CONFIG = 2
DSD_ERR_RUNTIME = 3


class ReplicaSummary(ctypes.Structure):
    """dsd_replica_summary"""
    _fields_ = [
        ("events_processed", ctypes.c_uint64),
        ("end_time_us", ctypes.c_int64),
        ("completed", ctypes.c_int64),
        ("first_arrival_us", ctypes.c_int64),
        ("last_completion_us", ctypes.c_int64),
        ("net_queue_wait_total_us", ctypes.c_int64),
        ("net_queue_wait_count", ctypes.c_int64),
        ("n_requests", ctypes.c_int64),
        ("throughput_rps", ctypes.c_double),
        ("mean_ttft_ms", ctypes.c_double),
        ("mean_tpot_ms", ctypes.c_double),
        ("has_duration", ctypes.c_int32),
        ("status", ctypes.c_int32),
    ]


class RequestRecord(ctypes.Structure):
    """dsd_request_record"""
    _fields_ = [
        ("drafter_id", ctypes.c_int64),
        ("prompt_length", ctypes.c_int64),
        ("output_length", ctypes.c_int64),
        ("arrival_us", ctypes.c_int64),
        ("first_token_us", ctypes.c_int64),
        ("completion_us", ctypes.c_int64),
        ("proposed", ctypes.c_int64),
        ("accepted", ctypes.c_int64),
        ("target_id", ctypes.c_int32),
        ("n_iterations", ctypes.c_int32),
    ]


class BusyInterval(ctypes.Structure):
    """dsd_busy_interval"""
    _fields_ = [("role", ctypes.c_int32), ("server_id", ctypes.c_int32), ("start_us", ctypes.c_int64),
                ("end_us", ctypes.c_int64)]


class RunOpts(ctypes.Structure):
    """dsd_run_opts"""
    _fields_ = [("collect_records", ctypes.c_int32), ("feature_probe", ctypes.c_int32),
                ("collect_event_log", ctypes.c_int32), ("reserved", ctypes.c_int32)]


# Every symbol include/dsdsim.h declares (checked by tests/test_capi.py).
EXPORTS = [
    "dsd_abi_version", "dsd_create", "dsd_create_devices", "dsd_device_count", "dsd_batch_shard_sizes",
    "dsd_destroy", "dsd_run_batch", "dsd_fetch_records",
    "dsd_batch_prepare", "dsd_batch_launch", "dsd_batch_sync", "dsd_batch_summaries",
    "dsd_batch_device_summaries", "dsd_stream", "dsd_last_launch_count", "dsd_last_kernel_ms",
    "dsd_last_transfer_bytes",
    "dsd_run_simulation", "dsd_run_sweep", "dsd_prepare_sweep", "dsd_resolve_config", "dsd_resolved_scenario",
    "dsd_resolved_replica", "dsd_resolved_digest", "dsd_resolved_free", "dsd_plan_sweep",
    "dsd_sweep_plan_scenarios", "dsd_sweep_plan_replicas", "dsd_sweep_plan_origin", "dsd_sweep_plan_free", "dsd_emit_report",
    "dsd_sweep_point_seed", "dsd_free", "dsd_batch_probe", "dsd_build_scenarios", "dsd_generate_dataset",
    "dsd_eval_policy", "dsd_fetch_event_log", "dsd_run_simulation_traced",
]
DSD_PROBE_FIELDS = 8

_lib = None


def lib():
    """Load libdsdsim.so once; raise loudly when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build the CUDA extension with __graft_entry__.build() "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    c = ctypes
    vp, sz, cp = c.c_void_p, c.c_size_t, c.c_char_p
    L.dsd_abi_version.restype = c.c_int
    L.dsd_create.argtypes = [c.c_int, c.POINTER(vp), cp, sz]
    L.dsd_create_devices.argtypes = [c.POINTER(c.c_int), c.c_int, c.POINTER(vp), cp, sz]
    L.dsd_device_count.argtypes = [vp]
    L.dsd_batch_shard_sizes.argtypes = [vp, c.POINTER(c.c_int64), c.c_int]
    L.dsd_destroy.argtypes = [vp]
    L.dsd_destroy.restype = None
    L.dsd_free.argtypes = [vp]
    L.dsd_free.restype = None
    L.dsd_run_batch.argtypes = [vp, vp, sz, vp, sz, vp, c.POINTER(ReplicaSummary), cp, sz]
    L.dsd_fetch_records.argtypes = [vp, sz, c.POINTER(RequestRecord), sz, c.POINTER(c.c_int64),
                                    c.POINTER(c.c_int32), c.POINTER(c.c_int32), sz, c.POINTER(c.c_int64),
                                    c.POINTER(c.c_int64), sz, cp, sz]
    L.dsd_batch_prepare.argtypes = [vp, vp, sz, vp, sz, vp, cp, sz]
    L.dsd_batch_launch.argtypes = [vp, cp, sz]
    L.dsd_batch_sync.argtypes = [vp, cp, sz]
    L.dsd_batch_summaries.argtypes = [vp, c.POINTER(ReplicaSummary), sz, cp, sz]
    L.dsd_batch_device_summaries.argtypes = [vp, c.POINTER(vp), c.POINTER(sz)]
    L.dsd_stream.argtypes = [vp]
    L.dsd_stream.restype = vp
    L.dsd_last_launch_count.argtypes = [vp]
    L.dsd_last_launch_count.restype = c.c_int64
    L.dsd_last_kernel_ms.argtypes = [vp, c.POINTER(c.c_double), c.POINTER(c.c_double), c.POINTER(c.c_double)]
    L.dsd_last_transfer_bytes.argtypes = [vp, c.POINTER(c.c_int64), c.POINTER(c.c_int64)]
    L.dsd_run_simulation.argtypes = [vp, cp, cp, c.c_int, c.c_int, c.c_uint64, c.POINTER(vp), c.POINTER(vp),
                                     c.POINTER(c.c_uint64), c.POINTER(c.c_int64), c.POINTER(c.c_double), cp, sz]
    L.dsd_fetch_event_log.argtypes = [vp, sz, c.POINTER(vp), c.POINTER(BusyInterval), sz, c.POINTER(c.c_int64), cp, sz]
    L.dsd_run_simulation_traced.argtypes = [vp, cp, cp, c.c_int, c.c_int, c.c_uint64, c.POINTER(vp), c.POINTER(vp),
                                            c.POINTER(BusyInterval), sz, c.POINTER(c.c_int64), c.POINTER(c.c_uint64),
                                            cp, sz]
    L.dsd_run_sweep.argtypes = [vp, cp, cp, cp, c.POINTER(vp), c.POINTER(vp), c.POINTER(c.c_double), cp, sz]
    L.dsd_prepare_sweep.argtypes = [vp, cp, cp, c.c_int, c.c_int, c.POINTER(c.c_int64), c.POINTER(c.c_int64),
                                    cp, sz]
    L.dsd_resolve_config.argtypes = [cp, cp, c.c_int, c.c_int, c.c_uint64, c.POINTER(vp), cp, sz]
    L.dsd_resolved_scenario.argtypes = [vp]
    L.dsd_resolved_scenario.restype = vp
    L.dsd_resolved_replica.argtypes = [vp, vp]
    L.dsd_resolved_replica.restype = None
    L.dsd_resolved_digest.argtypes = [vp]
    L.dsd_resolved_digest.restype = cp
    L.dsd_resolved_free.argtypes = [vp]
    L.dsd_resolved_free.restype = None
    L.dsd_plan_sweep.argtypes = [cp, cp, c.c_int, c.c_int, c.POINTER(vp), cp, sz]
    L.dsd_sweep_plan_origin.argtypes = [vp, c.POINTER(c.c_int64), c.POINTER(c.c_int32), sz]
    L.dsd_sweep_plan_origin.restype = sz
    L.dsd_sweep_plan_scenarios.argtypes = [vp, c.POINTER(vp)]
    L.dsd_sweep_plan_scenarios.restype = sz
    L.dsd_sweep_plan_replicas.argtypes = [vp, c.POINTER(vp)]
    L.dsd_sweep_plan_replicas.restype = sz
    L.dsd_sweep_plan_free.argtypes = [vp]
    L.dsd_sweep_plan_free.restype = None
    L.dsd_emit_report.argtypes = [vp, c.POINTER(RequestRecord), sz, c.POINTER(c.c_int32), c.POINTER(c.c_int32), sz,
                                  c.POINTER(c.c_int64), c.c_int, cp, c.c_uint64, c.POINTER(vp), c.POINTER(vp)]
    L.dsd_sweep_point_seed.argtypes = [c.c_uint64, cp, c.c_int]
    L.dsd_sweep_point_seed.restype = c.c_uint64
    L.dsd_batch_probe.argtypes = [vp, c.POINTER(c.c_double), sz, cp, sz]
    L.dsd_build_scenarios.argtypes = [cp, c.POINTER(vp), cp, sz]
    L.dsd_generate_dataset.argtypes = [vp, cp, c.POINTER(c.c_double), c.POINTER(vp), c.POINTER(vp), cp, sz]
    L.dsd_eval_policy.argtypes = [vp, cp, cp, cp, c.c_int, cp, c.POINTER(c.c_double), cp, sz]
    _lib = L
    return L
