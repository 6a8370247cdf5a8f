"""CPU-side checks of the C ABI: the library loads and exports every symbol
include/pdst.h declares (no compute calls without a GPU)."""

import os
import re

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "pdst.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(pdst_\w+)\s*\(", text, re.M)))


def test_header_symbols_exported():
    from paper_2603_28706_b200 import _lib

    lib = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_version_and_error_string():
    from paper_2603_28706_b200 import _lib

    assert b"sm_100a" in _lib.lib().pdst_version()
    assert isinstance(_lib.lib().pdst_last_error(), bytes)


def test_launch_counter_starts_at_zero():
    from paper_2603_28706_b200 import _lib

    assert _lib.lib().pdst_launch_count() == 0


def test_no_unresolved_library_symbols():
    """Every pdst:: symbol the library references is defined in it (a -shared
    link would otherwise defer the failure to the first call on the GPU)."""
    import shutil
    import subprocess

    from paper_2603_28706_b200 import _lib

    if not shutil.which("nm"):
        return
    out = subprocess.run(["nm", "-C", "-u", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "pdst::" not in out, [l for l in out.splitlines() if "pdst::" in l]


def test_vptr_validates_buffers():
    """The C ABI takes bare pointers: the host mirror checks length, dtype and
    contiguity before handing a buffer over (ValueError, like the reference's
    numpy reshapes on a size mismatch)."""
    import numpy as np
    import pytest
    import torch

    from paper_2603_28706_b200 import _lib as L

    assert L.vptr(None, 5) is None
    L.vptr(np.zeros(5), 5)
    L.vptr(torch.zeros(5, dtype=torch.float64), 5)
    for bad in (np.zeros(4), np.zeros(5, dtype=np.float32), np.zeros(10)[::2], torch.zeros(5),
                torch.zeros(10, dtype=torch.float64)[::2]):
        with pytest.raises(ValueError):
            L.vptr(bad, 5, "x")
