"""ctypes access to the C restatement oracle (oracle/_build/libdsd_oracle.so).

TEST INFRASTRUCTURE ONLY.  Scenarios come from the product library's host-only
resolver (dsd_resolve_config / dsd_plan_sweep, no GPU involved) so the oracle
and the GPU engine consume the identical dsd_scenario; reports are rendered by
the product's dsd_emit_report so they can be compared with the reference's
bytes.
"""
import ctypes
import os

from paper_2511_21669_b200 import _lib
from paper_2511_21669_b200._lib import ReplicaSummary, RequestRecord

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(REPO, "oracle", "_build", "libdsd_oracle.so")


class Replica(ctypes.Structure):
    _fields_ = [("scenario", ctypes.c_uint32), ("reserved", ctypes.c_uint32), ("seed", ctypes.c_uint64),
                ("gen_seed", ctypes.c_uint64)]


_o = None


def olib():
    global _o
    if _o is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError("oracle not built: make -C oracle restate")
        L = ctypes.CDLL(ORACLE_SO)
        c = ctypes
        L.oracle_request_count.argtypes = [c.c_void_p]
        L.oracle_request_count.restype = c.c_int64
        L.oracle_sequence_bound.argtypes = [c.c_void_p, c.c_void_p]
        L.oracle_sequence_bound.restype = c.c_int64
        L.oracle_run.argtypes = [c.c_void_p, c.c_void_p, c.POINTER(ReplicaSummary), c.POINTER(RequestRecord),
                                 c.POINTER(c.c_int32), c.POINTER(c.c_int32), c.c_int64, c.POINTER(c.c_int64),
                                 c.c_char_p, c.c_size_t]
        L.oracle_run_batch.argtypes = [c.c_void_p, c.c_void_p, c.c_size_t, c.c_int, c.POINTER(ReplicaSummary),
                                       c.c_char_p, c.c_size_t]
        _o = L
    return _o


class Resolved:
    """dsd_resolve_config result (owns the scenario arrays)."""

    def __init__(self, yaml_text, base_dir=".", seed=None, strict=True):
        L = _lib.lib()
        self._L = L
        self._p = ctypes.c_void_p()
        err = ctypes.create_string_buffer(4096)
        rc = L.dsd_resolve_config(yaml_text.encode(), base_dir.encode(), int(strict), int(seed is not None),
                                  seed or 0, ctypes.byref(self._p), err, 4096)
        if rc != 0:
            from paper_2511_21669_b200.api import _check
            _check(rc, err)
        self.scenario = L.dsd_resolved_scenario(self._p)
        self.replica = Replica()
        L.dsd_resolved_replica(self._p, ctypes.byref(self.replica))
        self.digest = L.dsd_resolved_digest(self._p).decode()

    def n_targets(self):
        return ctypes.cast(self.scenario, ctypes.POINTER(ctypes.c_int32))[0]

    def __del__(self):
        if getattr(self, "_p", None):
            self._L.dsd_resolved_free(self._p)


def oracle_run(scenario_ptr, replica, n_targets):
    """Returns (summary, records, gamma_seq, committed_seq, busy_us)."""
    L = olib()
    n = L.oracle_request_count(scenario_ptr)
    cap = L.oracle_sequence_bound(scenario_ptr, ctypes.byref(replica))
    s = ReplicaSummary()
    recs = (RequestRecord * max(n, 1))()
    g = (ctypes.c_int32 * max(cap, 1))()
    c = (ctypes.c_int32 * max(cap, 1))()
    busy = (ctypes.c_int64 * max(n_targets, 1))()
    err = ctypes.create_string_buffer(1024)
    rc = L.oracle_run(scenario_ptr, ctypes.byref(replica), ctypes.byref(s), recs, g, c, cap, busy, err, 1024)
    assert rc == 0, err.value
    nseq = sum(recs[i].n_iterations for i in range(n))
    return s, recs, n, g, c, nseq, busy


def render(summary, recs, n, g, c, nseq, busy, n_targets, digest, seed):
    L = _lib.lib()
    out = ctypes.c_void_p()
    rc = L.dsd_emit_report(ctypes.byref(summary), recs, n, g, c, nseq, busy, n_targets, digest.encode(), seed,
                           ctypes.byref(out), None)
    assert rc == 0
    s = ctypes.cast(out, ctypes.c_char_p).value.decode()
    L.dsd_free(out)
    return s


def oracle_report(yaml_text, base_dir=".", seed=None):
    r = Resolved(yaml_text, base_dir, seed)
    s, recs, n, g, c, nseq, busy = oracle_run(r.scenario, r.replica, r.n_targets())
    return render(s, recs, n, g, c, nseq, busy, r.n_targets(), r.digest, r.replica.seed), s
