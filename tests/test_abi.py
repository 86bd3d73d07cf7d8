"""The C-ABI library loads and exports every symbol include/drotb.h declares,
and the C++ drop-in header compiles against it (CPU only: no CUDA calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "drotb.h")


def declared_symbols():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(drotb_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("drotb_solve_f32", "drotb_solve_f64", "drotb_step_f64", "drotb_engine_pass_f32",
                 "drotb_check_problem_f64", "drotb_session_run_timed", "drotb_gen_gaussian"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2110_11738_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding covers the whole surface
    assert set(declared_symbols()) <= set(_lib.SIGNATURES)


def test_no_cuda_needed_for_host_entry_points():
    import paper_2110_11738_b200 as d
    assert d._lib.load().drotb_abi_version() == 1
    assert d._lib.load().drotb_errc_name(12) == b"fold_state_mismatch"


def test_cpp_dropin_compiles(tmp_path):
    exe = tmp_path / "dropin"
    lib_dir = os.path.join(ROOT, "paper_2110_11738_b200")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "dropin_solve.cpp"), "-o", str(exe),
                        "-L", lib_dir, "-ldrotb200", f"-Wl,-rpath,{lib_dir}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_product_does_not_reference_oracle():
    """The product package never imports or links the CPU oracles."""
    pkg = os.path.join(ROOT, "paper_2110_11738_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".hpp", ".h")):
                src = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "pyoracle" not in src and "libdrotref" not in src and "liborc" not in src, f
