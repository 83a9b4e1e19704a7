"""The C-ABI library loads and exports every entry point declared in
include/peakann_b200.h; the ctypes table matches the header (CPU only: no
kernel is launched)."""

import ctypes
import os
import re

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "peakann_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return re.findall(r"^\s*(?:int|void|const char\*)\s+(pk_\w+)\s*\(", src, flags=re.M)


def test_header_declares_entry_points():
    names = declared()
    assert len(names) >= 25
    assert "pk_beam_knn" in names and "pk_build_vamana" in names and "pk_assign_clusters" in names


def test_library_exports_every_declared_symbol():
    from paper_2312_03940_b200 import _lib

    _lib.build_library()
    so = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared() if not hasattr(so, n)]
    assert not missing, missing


def test_ctypes_table_covers_header():
    from paper_2312_03940_b200 import _lib

    names = set(declared()) - {"pk_version", "pk_last_error", "pk_device_info", "pk_prof_enable",
                               "pk_prof_collect", "pk_prof_only"}
    assert names == set(_lib.SIGNATURES), names ^ set(_lib.SIGNATURES)


def test_version_and_error_string_without_gpu():
    from paper_2312_03940_b200 import _lib

    L = _lib.lib()
    assert L.pk_version() == 1
    assert isinstance(L.pk_last_error(), bytes)
