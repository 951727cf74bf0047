"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/empc_b200.h declares.  CPU only (no compute calls)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2001_04931_b200 import _native as nat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "empc_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(empc_[a-z_0-9]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(nat.EXPORTS)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(nat.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(nat.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_library_is_sm100a():
    if not os.path.exists(nat.LIB_PATH):
        pytest.skip("library not built")
    out = subprocess.run(["cuobjdump", "--list-elf", nat.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_rollout_kernels_use_fp32_fma():
    """The rollout hot loop is FFMA work (SURVEY §8d roofline): the default
    C3 variant's SASS is dominated by FFMA and carries no legacy HMMA path."""
    if not os.path.exists(nat.LIB_PATH):
        pytest.skip("library not built")
    listing = _function_names()
    names = re.findall(r"Function : (_ZN4empc14rollout_kernelIfLi48ELi2ELi4ELb1ELb0ELi2E\S*)", listing)
    assert names, "default C3 rollout variant (NP48 RR2 CC4 areg ks2) not compiled"
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", names[0], nat.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert sass.count("FFMA") >= 192  # 24 columns x 2 rows x 4 candidates per step, fully unrolled
    assert "HMMA" not in sass


def test_load_without_gpu_does_not_touch_the_device():
    lib = nat.load()
    assert lib.empc_last_error(None) is not None


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(RuntimeError, match="missing"):
        _load_missing(tmp_path)


def _load_missing(tmp_path):
    saved = nat._lib
    nat._lib = None
    try:
        nat.load(str(tmp_path / "nope.so"))
    finally:
        nat._lib = saved


def test_benched_persistent_kernel_is_ffma_and_uses_no_local_memory():
    """The benched C3 kernel (persist_kernel, warp-synchronous NP48 RR3 CC4
    KS2, half-K, 384-thread bound): FFMA recursion, no HMMA, no register
    spills to local memory (which would put the state recursion on L1)."""
    if not os.path.exists(nat.LIB_PATH):
        pytest.skip("library not built")
    listing = _function_names()
    names = re.findall(r"Function : (_ZN4empc14persist_kernelIfLi48ELi3ELi4ELb1ELb0ELi2ELb1ELi384ELb1E\S*)", listing)
    assert names, "benched persistent variant not compiled"
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", names[0], nat.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert sass.count("FFMA") >= 144  # 12 half-K columns x 3 rows x 4 candidates per step
    assert "HMMA" not in sass
    assert "STL" not in sass and "LDL" not in sass


_NAMES = []


def _function_names() -> str:
    """'Function : <mangled>' lines of the library's SASS (listed once)."""
    if not _NAMES:
        out = subprocess.run(["cuobjdump", "-sass", nat.LIB_PATH], capture_output=True, text=True).stdout
        _NAMES.append("\n".join(line for line in out.splitlines() if "Function :" in line))
    return _NAMES[0]
