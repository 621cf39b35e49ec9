"""The C ABI library loads without a GPU and exports every function that
include/*.h declares, with the ctypes signature table kept in sync."""

import ctypes
import glob
import os
import re

import pytest

from conftest import ROOT
from paper_1003_2022_b200 import _native


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(rubs_b200_\w+)\s*\(", text):
            names.add(m.group(1))
    return names


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_native.LIB_PATH):
        _native.build_native()
    return _native.load()


def test_header_declares_the_boundary():
    names = _declared()
    for required in ("rubs_b200_filter", "rubs_b200_filter_params", "rubs_b200_lookup",
                     "rubs_b200_preintegrate", "rubs_b200_interpolate", "rubs_b200_filter_host"):
        assert required in names


def test_every_declared_symbol_is_exported(lib):
    for name in _declared():
        assert hasattr(lib, name), name
        ctypes.cast(getattr(lib, name), ctypes.c_void_p)


def test_signature_table_matches_header():
    assert set(_native.SIGNATURES) == _declared()


def test_version_and_error_string(lib):
    assert lib.rubs_b200_version().startswith(b"rubs_b200")
    assert isinstance(lib.rubs_b200_last_error(), bytes)


def test_preintegrate_shape_is_reference_geometry(lib):
    # engine.py:169-180 for an 8 x 10 image at the origin: 12 x 24 plane
    # from lattice (-2, -2) (probe P6)
    out = [ctypes.c_int64() for _ in range(4)]
    lib.rubs_b200_preintegrate_shape(8, 10, 0, 0, -2, 11, -2, 9, *(ctypes.byref(o) for o in out))
    rows, cols, c_lo, r_lo = (o.value for o in out)
    assert (rows, cols, c_lo, r_lo) == (12, 24, -2, -2)


def test_library_is_sm100a(lib):
    # the fatbin must carry sm_100a SASS (cuobjdump lists the ELF arch)
    import shutil
    import subprocess
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
