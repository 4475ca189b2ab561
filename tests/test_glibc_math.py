"""glibc's exp / log / cos / log1p restated for the device (VERDICT r1
weak 1b).  CPU checks: the tables in glibc_tables.inc are the host libm's own
data, and the restatement (host build of the same header) equals the host's
exp / log / cos / log1p bit for bit on 2e7 inputs each.  The device side is
tests/test_libm.py."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
LIBM = "/usr/lib/x86_64-linux-gnu/libm.so.6"


@pytest.fixture(scope="module")
def checker():
    subprocess.run(["make", "-C", os.path.join(HERE, "native"), "_build/glibc_check"], check=True,
                   capture_output=True)
    return os.path.join(HERE, "native", "_build", "glibc_check")


@pytest.mark.skipif(not os.path.exists(LIBM), reason="no system libm")
def test_tables_are_the_host_libm_data():
    import sys
    sys.path.insert(0, os.path.join(REPO, "tools"))
    import gen_glibc_tables as g
    committed = open(g.OUT).read()
    assert committed == g.render(*g.extract(LIBM))


def _host_has_fma():
    try:
        return " fma " in " " + open("/proc/cpuinfo").read().replace("\n", " ") + " "
    except OSError:
        return False


# glibc picks its FMA-compiled exp / log (the ones restated) on FMA hosts only
@pytest.mark.skipif(not _host_has_fma(), reason="host libm uses its non-FMA variants")
def test_restated_exp_log_equal_host_glibc(checker):
    out = subprocess.run([checker, "20000000"], check=True, capture_output=True, text=True).stdout
    n, mm_log, mm_exp, mm_cos, mm_log1p = map(int, out.strip().splitlines()[-1].split())
    assert n == 20000000
    assert (mm_log, mm_exp, mm_cos, mm_log1p) == (0, 0, 0, 0), out
