"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/dsdsim.h declares, and refuses to run without a GPU (no CPU
fallback)."""
import ctypes
import os
import re

import pytest

from paper_2511_21669_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(REPO, "include", "dsdsim.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dsd_[a-z_]+)\s*\(", text)))


def test_header_declares_what_python_binds():
    assert header_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    missing = [s for s in header_symbols() if not hasattr(L, s)]
    assert not missing
    assert L.dsd_abi_version() == 2


def test_struct_sizes_match_header():
    assert ctypes.sizeof(_lib.ReplicaSummary) == 96
    assert ctypes.sizeof(_lib.RequestRecord) == 72
    assert ctypes.sizeof(_lib.BusyInterval) == 24
    assert ctypes.sizeof(_lib.RunOpts) == 16


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback():
    from paper_2511_21669_b200 import EngineError, Simulator
    with pytest.raises(EngineError, match="no CPU fallback"):
        Simulator(0)
