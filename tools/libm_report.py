"""Device-vs-glibc transcendental check (tests/native/libm_check.cu) as one
JSON document: per function the inputs, bitwise mismatches and integer flips."""
import ctypes
import json
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = ctypes.CDLL(os.path.join(HERE, "tests", "native", "_build", "liblibm_check.so"))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10 ** 8
out = []
for fn, name in [(0, "log(1-u)"), (1, "cos(2*pi*u)"), (2, "exp(mu+sigma*z)"), (3, "log1p(feature)")]:
    mm, fl, ex = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
    assert L.libm_check(fn, ctypes.c_uint64(12345), ctypes.c_int64(n), ctypes.byref(mm), ctypes.byref(fl),
                        ctypes.byref(ex)) == 0
    out.append({"function": name, "inputs": n, "bitwise_mismatches": mm.value, "integer_flips": fl.value,
                "example_input": ex.value if mm.value else None})
print(json.dumps({"check": "glibc's algorithms restated on the device (glibc_math.cuh, -fmad=false) vs host glibc "
                           "on the generator's and the AWC normaliser's argument domains",
                  "results": out}, indent=1))
