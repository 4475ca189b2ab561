"""ctypes access to the reference oracle (TEST INFRASTRUCTURE ONLY).

oracle/_ref/libspecsim_ref.so is the UNMODIFIED reference library
(/root/reference/proj/src) compiled by oracle/Makefile plus the thin C shim
oracle/ref_harness.cpp.  Only tests/, bench.py's cpu_baseline leg and
__graft_entry__.smoke() load it; the product path never does.
"""
import ctypes
import hashlib
import os

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(REPO, "oracle", "_ref", "libspecsim_ref.so")
GOLDEN = os.path.join(REPO, "tests", "golden")
CONFIGS = os.path.join(GOLDEN, "configs")
GEN_DIR = os.path.join(GOLDEN, "_gen")  # generated fixtures (git-ignored)

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError("reference oracle not built: run `make -C oracle ref` (needs /root/reference)")
        L = ctypes.CDLL(REF_SO)
        c = ctypes
        L.ref_free.argtypes = [c.c_void_p]
        L.ref_fnv1a64.restype = c.c_uint64
        L.ref_fnv1a64.argtypes = [c.c_char_p, c.c_size_t, c.c_uint64]
        L.ref_rng_u64.argtypes = [c.c_uint64, c.c_char_p, c.POINTER(c.c_uint64), c.c_size_t]
        L.ref_rng_unit.argtypes = [c.c_uint64, c.c_char_p, c.POINTER(c.c_double), c.c_size_t]
        L.ref_net_delay.argtypes = [c.c_double, c.c_double, c.c_uint64, c.POINTER(c.c_int64), c.c_size_t]
        L.ref_gen_trace.argtypes = [c.c_double, c.c_int64, c.c_double, c.c_char_p, c.c_double, c.c_double,
                                    c.c_double, c.c_double, c.c_int64, c.c_uint64, c.POINTER(c.c_void_p),
                                    c.c_char_p, c.c_size_t]
        L.ref_run_config.argtypes = [c.c_char_p, c.c_char_p, c.c_int, c.c_uint64, c.c_int,
                                     c.POINTER(c.c_void_p), c.POINTER(c.c_uint64), c.POINTER(c.c_int64),
                                     c.POINTER(c.c_double), c.c_char_p, c.c_size_t]
        L.ref_run_config_full.argtypes = [c.c_char_p, c.c_char_p, c.c_int, c.c_uint64, c.POINTER(c.c_void_p),
                                          c.POINTER(c.c_void_p), c.POINTER(c.c_void_p), c.POINTER(c.c_uint64),
                                          c.c_char_p, c.c_size_t]
        L.ref_run_config_busy.argtypes = [c.c_char_p, c.c_char_p, c.c_int, c.c_uint64, c.POINTER(c.c_void_p),
                                          c.c_char_p, c.c_size_t]
        L.ref_run_sweep.argtypes = [c.c_char_p, c.c_char_p, c.c_int, c.c_char_p, c.POINTER(c.c_void_p),
                                    c.POINTER(c.c_void_p), c.c_char_p, c.c_size_t]
        L.ref_sweep_point_seed.restype = c.c_uint64
        L.ref_sweep_point_seed.argtypes = [c.c_uint64, c.c_char_p, c.c_int]
        L.ref_sweep_replicas.argtypes = [c.c_char_p, c.c_char_p, c.c_int, c.POINTER(c.c_double), c.c_char_p,
                                         c.c_size_t]
        L.ref_sweep_bench.argtypes = [c.c_char_p, c.c_char_p, c.c_int, c.POINTER(c.c_int64), c.c_int64,
                                      c.POINTER(c.c_double), c.c_char_p, c.c_size_t]
        L.ref_random_model.argtypes = [c.c_uint64, c.c_int, c.c_int, c.POINTER(c.c_double),
                                       c.POINTER(c.c_double), c.c_char_p, c.c_char_p, c.c_size_t]
        L.ref_train_model.argtypes = [c.c_char_p, c.c_int, c.c_int, c.c_uint64, c.POINTER(c.c_double),
                                      c.c_char_p, c.c_size_t]
        L.ref_awc_predict.argtypes = [c.c_char_p, c.POINTER(c.c_double), c.c_size_t, c.POINTER(c.c_double),
                                      c.c_char_p, c.c_size_t]
        L.ref_consume_acceptance.argtypes = [c.POINTER(c.c_uint8), c.c_size_t, c.POINTER(c.c_int), c.c_size_t,
                                             c.POINTER(c.c_int)]
        L.ref_predict_synth.restype = c.c_double
        L.ref_predict_synth.argtypes = [c.c_double] * 5 + [c.c_int, c.c_int, c.c_int, c.c_int, c.c_int64]
        L.ref_build_scenarios.argtypes = [c.c_char_p, c.POINTER(c.c_void_p), c.c_char_p, c.c_size_t]
        L.ref_generate_dataset.argtypes = [c.c_char_p, c.c_int, c.POINTER(c.c_void_p), c.POINTER(c.c_void_p),
                                           c.c_char_p, c.c_size_t]
        L.ref_eval_policy.argtypes = [c.c_char_p, c.c_char_p, c.c_char_p, c.c_int, c.c_char_p, c.c_int,
                                      c.POINTER(c.c_double), c.c_char_p, c.c_size_t]
        _lib = L
    return _lib


def available():
    return os.path.exists(REF_SO)


def _take(p):
    s = ctypes.cast(p, ctypes.c_char_p).value.decode()
    lib().ref_free(p)
    return s


class RefError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def run_config(yaml_text, base_dir=".", seed=None, strict=True):
    """resolve_config + run_simulation; returns (report_json, events, end_time_us, agg[4])."""
    c = ctypes
    rep = c.c_void_p()
    ev = c.c_uint64()
    end = c.c_int64()
    agg = (c.c_double * 4)()
    err = c.create_string_buffer(4096)
    rc = lib().ref_run_config(yaml_text.encode(), base_dir.encode(), int(seed is not None), seed or 0, int(strict),
                              c.byref(rep), c.byref(ev), c.byref(end), agg, err, 4096)
    if rc != 0:
        raise RefError(rc, err.value.decode())
    return _take(rep), ev.value, end.value, list(agg)


def run_config_busy(yaml_text, base_dir=".", seed=None):
    """RunResult::busy_intervals of one run: [(role 't'|'d', server id, start_us, end_us)]."""
    c = ctypes
    out = c.c_void_p()
    err = c.create_string_buffer(4096)
    rc = lib().ref_run_config_busy(yaml_text.encode(), base_dir.encode(), int(seed is not None), seed or 0,
                                   c.byref(out), err, 4096)
    if rc != 0:
        raise RefError(rc, err.value.decode())
    rows = []
    for line in _take(out).splitlines():
        r, i, a, b = line.split()
        rows.append((r, int(i), int(a), int(b)))
    return rows


def run_config_full(yaml_text, base_dir=".", seed=None):
    c = ctypes
    rep, csv, log = c.c_void_p(), c.c_void_p(), c.c_void_p()
    ev = c.c_uint64()
    err = c.create_string_buffer(4096)
    rc = lib().ref_run_config_full(yaml_text.encode(), base_dir.encode(), int(seed is not None), seed or 0,
                                   c.byref(rep), c.byref(csv), c.byref(log), c.byref(ev), err, 4096)
    if rc != 0:
        raise RefError(rc, err.value.decode())
    return _take(rep), _take(csv), _take(log), ev.value


def run_sweep(sweep_yaml, base_dir=".", parallel=8, out_dir=""):
    c = ctypes
    js, cs = c.c_void_p(), c.c_void_p()
    err = c.create_string_buffer(4096)
    rc = lib().ref_run_sweep(sweep_yaml.encode(), base_dir.encode(), parallel, out_dir.encode(), c.byref(js),
                             c.byref(cs), err, 4096)
    if rc != 0:
        raise RefError(rc, err.value.decode())
    return _take(js), _take(cs)


def sweep_replicas(sweep_yaml, base_dir, threads, n_replicas):
    """Per-replica results of the reference run_sweep worker, point-major:
    float64 [n_replicas, 6] = events_processed, end_time, completed,
    throughput_rps, mean_ttft_ms, mean_tpot_ms (failed points: -1)."""
    import numpy as np
    rows = np.zeros((n_replicas, 6), dtype=np.float64)
    err = ctypes.create_string_buffer(4096)
    rc = lib().ref_sweep_replicas(sweep_yaml.encode(), base_dir.encode(), threads,
                                  rows.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), err, 4096)
    if rc != 0:
        raise RuntimeError(err.value.decode())
    return rows


def sweep_bench(sweep_yaml, base_dir, threads, points=None):
    c = ctypes
    out = (c.c_double * 6)()
    err = c.create_string_buffer(4096)
    if points:
        arr = (c.c_int64 * len(points))(*points)
        rc = lib().ref_sweep_bench(sweep_yaml.encode(), base_dir.encode(), threads, arr, len(points), out, err, 4096)
    else:
        rc = lib().ref_sweep_bench(sweep_yaml.encode(), base_dir.encode(), threads, None, 0, out, err, 4096)
    if rc != 0:
        raise RefError(rc, err.value.decode())
    return {"events": out[0], "replicas": out[1], "seconds": out[2], "failed": out[3], "sim_thread_s": out[4],
            "resolve_thread_s": out[5]}


def gen_trace(rate, n, alpha, preset=None, prompt_median=60.0, prompt_sigma=0.4, output_median=90.0,
              output_sigma=0.35, n_drafts=1, seed=1):
    c = ctypes
    out = c.c_void_p()
    err = c.create_string_buffer(4096)
    rc = lib().ref_gen_trace(rate, n, alpha, (preset or "").encode(), prompt_median, prompt_sigma, output_median,
                             output_sigma, n_drafts, seed, c.byref(out), err, 4096)
    if rc != 0:
        raise RefError(rc, err.value.decode())
    return _take(out)


def random_model(path, seed=7, hidden=64, blocks=2, lo=None, hi=None):
    c = ctypes
    lo = lo or [0.0, 0.0, 0.0, 0.0, 1.0]
    hi = hi or [1.0, 1.0, 5.0, 5.0, 12.0]
    err = c.create_string_buffer(4096)
    rc = lib().ref_random_model(seed, hidden, blocks, (c.c_double * 5)(*lo), (c.c_double * 5)(*hi),
                                path.encode(), err, 4096)
    if rc != 0:
        raise RefError(rc, err.value.decode())


def train_model(path, parallel=8, epochs=0, seed=42):
    c = ctypes
    maes = (c.c_double * 3)()
    err = c.create_string_buffer(4096)
    rc = lib().ref_train_model(path.encode(), parallel, epochs, seed, maes, err, 4096)
    if rc != 0:
        raise RefError(rc, err.value.decode())
    return list(maes)


def build_scenarios(grid_yaml=""):
    """build_scenarios + serialize_scenarios of the reference (dataset.cpp:50-108)."""
    c = ctypes
    p = c.c_void_p()
    err = c.create_string_buffer(4096)
    rc = lib().ref_build_scenarios(grid_yaml.encode(), c.byref(p), err, 4096)
    if rc != 0:
        raise RefError(rc, err.value.decode())
    return _take(p)


def generate_dataset(grid_yaml="", parallel=8):
    """`specsim gen-dataset`: (dataset.jsonl, scenarios.jsonl) text of the reference."""
    c = ctypes
    ds, sc = c.c_void_p(), c.c_void_p()
    err = c.create_string_buffer(4096)
    rc = lib().ref_generate_dataset(grid_yaml.encode(), parallel, c.byref(ds), c.byref(sc), err, 4096)
    if rc != 0:
        raise RefError(rc, err.value.decode())
    return _take(ds), _take(sc)


def eval_policy(scenarios_jsonl, window_kind, gamma=4, model_path="", split="all", parallel=8):
    """eval_policy_on_scenarios of the reference -> [thr, ttft, tpot, mean gamma]."""
    c = ctypes
    out = (c.c_double * 4)()
    err = c.create_string_buffer(4096)
    rc = lib().ref_eval_policy(scenarios_jsonl.encode(), split.encode(), window_kind.encode(), gamma,
                               model_path.encode(), parallel, out, err, 4096)
    if rc != 0:
        raise RefError(rc, err.value.decode())
    return list(out)


def sha256(s):
    return hashlib.sha256(s.encode() if isinstance(s, str) else s).hexdigest()


def mixed_trace_text():
    """SURVEY Appendix C mixed.jsonl: three generate_synthetic parts (acceptance.cpp:184-201 pattern)."""
    parts = [("gsm8k-like", 0.8, 1400, 1), ("humaneval-like", 0.85, 1300, 2), ("cnndm-like", 0.6, 1300, 3)]
    return "".join(gen_trace(50.0, n, a, preset=p, n_drafts=1024, seed=s) for p, a, n, s in parts)


def ensure_generated(which=("mixed.jsonl", "model.json")):
    """Materialise the large fixtures into tests/golden/_gen/ (deterministic; built by the reference)."""
    os.makedirs(GEN_DIR, exist_ok=True)
    paths = {}
    if "mixed.jsonl" in which:
        p = os.path.join(GEN_DIR, "mixed.jsonl")
        if not os.path.exists(p):
            with open(p + ".tmp", "w") as f:
                f.write(mixed_trace_text())
            os.replace(p + ".tmp", p)
        paths["mixed.jsonl"] = p
    if "model.json" in which:
        p = os.path.join(GEN_DIR, "model.json")
        if not os.path.exists(p):
            train_model(p + ".tmp", parallel=max(1, os.cpu_count() or 1))
            os.replace(p + ".tmp", p)
        paths["model.json"] = p
    return paths
