"""The C-ABI library builds, loads and exports every symbol include/flash.h declares
(no compute calls: these run on the CPU-only dev box)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flash.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(flash_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1709_01190_b200 import build

    build.build()
    from paper_1709_01190_b200 import flash

    return flash.load_library()


def test_header_declares_the_survey_boundary():
    names = declared_functions()
    for required in ("flash_create", "flash_hash", "flash_insert", "flash_query_topk", "flash_knn_graph"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_1709_01190_b200", "libflash.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (flash_[a-z_]+)$", out, flags=re.M))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    for n in declared_functions():
        assert hasattr(lib, n)


def test_binding_wraps_every_declared_symbol():
    from paper_1709_01190_b200 import flash

    assert sorted(flash.EXPORTS) == declared_functions()
    for n in declared_functions():
        assert callable(getattr(flash, n)), n


def test_library_is_built_for_sm100a_only():
    so = os.path.join(ROOT, "paper_1709_01190_b200", "libflash.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_argument_errors_are_reported_before_any_device_work(lib):
    h = ctypes.c_void_p()
    assert lib.flash_create(0, 16, 32, 1 << 15, 1, ctypes.byref(h)) == 1  # K = 0
    assert b"K" in lib.flash_last_error()
    assert lib.flash_create(4, 16, 0, 1 << 15, 1, ctypes.byref(h)) == 1   # R = 0
    assert lib.flash_create(4, 16, 32, 0, 1, ctypes.byref(h)) == 1        # range = 0
    assert lib.flash_create(4, 3000, 32, 1 << 15, 1, ctypes.byref(h)) == 1  # K*L too large
    assert lib.flash_hash(None, None, None, 1, None, None, None) == 1
    assert lib.flash_launch_count(None) == 0
    lib.flash_destroy(None)  # no-op


def test_oracle_and_cuda_path_share_no_code():
    """The oracle never imports / includes the product and vice versa."""
    pkg = os.path.join(ROOT, "paper_1709_01190_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"(?:import|from|#include)\s+[\"<]?(\w+)", text), f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c", ".h")):
            text = open(os.path.join(ROOT, "oracle", f)).read()
            deps = re.findall(r"^\s*(?:import|from|#include)\s+[\"<]?([\w./]+)", text, flags=re.M)
            assert not [d for d in deps if "paper_1709_01190_b200" in d or "flash" in d], (f, deps)
