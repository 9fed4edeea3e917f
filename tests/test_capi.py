"""The C-ABI library loads without a GPU and exports every symbol that
include/*.h declares; the face record layout matches the header. CPU only."""

from __future__ import annotations

import ctypes
import glob
import os
import re

from paper_2504_15814_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for header in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(header).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?\w+\s*\*?\s*(th_\w+)\s*\(", text, flags=re.M):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name
    assert names == set(_native.EXPORTED)


def test_abi_version_and_error_plumbing():
    lib = _native.load()
    assert lib.th_abi_version() == 1
    rc = lib.th_scheme_feasible(0, 7, 4, 3)
    assert rc == _native.TH_ERR_CONFIG
    assert b"unknown scheme" in lib.th_last_error()


def test_face_record_size_matches_header():
    text = open(os.path.join(ROOT, "include", "trihalo_b200.h")).read()
    body = re.search(r"typedef struct th_face \{(.*?)\} th_face;", text, flags=re.S).group(1)
    size = 0
    for m in re.finditer(r"(int64_t|int32_t)\s+(\w+)(?:\[(\d+)\])?;", body):
        size += (8 if m.group(1) == "int64_t" else 4) * int(m.group(3) or 1)
    assert size == _native.FACE_DTYPE.itemsize == 144
