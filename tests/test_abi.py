"""The C-ABI library loads and exports every symbol include/*.h declares (CPU:
no compute calls)."""

import glob
import os
import re

from paper_1811_10136_b200 import _lib

from .conftest import ROOT


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names.update(re.findall(r"\b(fr_[a-z0-9_]+)\s*\(", src))
    return names


def test_header_declares_the_binding_table():
    assert declared_symbols() == set(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.fr_abi_version() == 1
    assert lib.fr_rigid_pass_width(0, 0) == 25
    assert lib.fr_rigid_pass_width(1, 1) == 31


def test_invalid_arguments_raise_value_error():
    import ctypes
    import pytest
    lib = _lib.load()
    h = ctypes.c_void_p()
    sig, _keep = _lib.dptr([1.0])
    with pytest.raises(ValueError):
        _lib.check(lib.fr_lattice_create(13, sig, ctypes.byref(h)))
