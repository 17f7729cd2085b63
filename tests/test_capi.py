"""C-ABI library: builds, loads without a GPU, exports every declared symbol."""
import os
import re

from paper_1912_03565_b200 import _native

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared_symbols():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            text = open(os.path.join(ROOT, "include", fn)).read()
            names |= set(re.findall(r"\b(hfb_[a-z0-9_]+)\s*\(", text))
    return names


def test_library_exists():
    assert os.path.exists(_native.LIB_PATH), "run `make` (or __graft_entry__.build())"


def test_every_declared_symbol_is_exported_and_bound():
    declared = declared_symbols()
    assert len(declared) >= 20
    exported = set(_native.exported_symbols())
    assert declared <= exported | set(), declared - exported
    assert declared == set(_native.SIGNATURES), declared ^ set(_native.SIGNATURES)


def test_load_and_strerror_without_gpu():
    lib = _native.load_library()
    assert b"sm_100a" in lib.hfb_version()
    assert lib.hfb_strerror(3).decode().startswith("vanishing pivot")


def test_library_targets_sm100a():
    data = open(_native.LIB_PATH, "rb").read()
    assert b"sm_100a" in data
