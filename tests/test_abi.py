"""The C-ABI library loads and exports every symbol include/*.h declares (CPU only)."""

import ctypes
import glob
import os
import re

from paper_2109_01173_b200 import _native as nat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        names.update(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(sfb_\w+)\s*\(", text, re.M))
    return names


def test_library_exports_header_symbols():
    lib = nat.load_library()
    declared = declared_symbols()
    assert len(declared) >= 20
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert set(nat.EXPORTS) == declared


def test_version_and_error_channel():
    lib = nat.load_library()
    assert lib.sfb_version() == 1
    assert isinstance(lib.sfb_last_error(), bytes)


def test_library_is_sm100a():
    # the cubin inside the .so targets sm_100a (no PTX fallback for other archs)
    data = open(nat.LIB_PATH, "rb").read()
    assert b"sm_100a" in data
    assert isinstance(ctypes.CDLL(nat.LIB_PATH), ctypes.CDLL)
