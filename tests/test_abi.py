"""The C-ABI library builds, loads and exports every entry point that
include/voltb200.h declares (no compute calls: CPU only)."""
import ctypes
import re
from pathlib import Path

from paper_2403_16438_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "voltb200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(vb_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_expected_surface():
    names = declared_functions()
    for must in ("vb_mean_zncc_scores", "vb_motion_estimate", "vb_summarize", "vb_stage_run_host",
                 "vb_make_reference", "vb_correct_frames", "vb_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    assert set(declared_functions()) == set(_lib.SIGNATURES)


def test_library_is_sm100a_only():
    """The fatbin carries sm_100a SASS (no PTX JIT fallback to other archs)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.lib_path())], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_struct_layouts():
    assert ctypes.sizeof(_lib.VbMotion) == 32 == _lib.MOTION_DTYPE.itemsize
    assert ctypes.sizeof(_lib.VbStageConfig) == 56  # 7 ints, double, int, int64 (C layout)


def test_version_and_error_without_gpu():
    lib = _lib.load()
    assert b"sm_100a" in lib.vb_version()
    assert isinstance(lib.vb_last_error(), bytes)
    n = ctypes.c_int()
    rc = lib.vb_patch_grid(30, 30, 21, 10, None, ctypes.byref(n))  # host-only geometry, reference message
    assert rc == _lib.VB_EINVAL and b"too small for patch 21 with margin 10" in lib.vb_last_error()
    assert lib.vb_patch_grid(256, 512, 21, 8, None, ctypes.byref(n)) == 0 and n.value == 288


def test_host_copy_every_split():
    """The executor's threaded pageable staging copy (stage.cu host_copy_n)
    moves every byte for odd frame sizes and 1-8 threads (a split
    with step = round64(bytes / nt) dropped the last bytes % nt bytes)."""
    import numpy as np

    lib = _lib.load()
    rng = np.random.default_rng(5)
    for n in (299 * 255 * 2 * 250, 341 * 257 * 2 * 250, 213 * 513 * 2 * 250, 100, 64 * 1000003 + 7):
        a = rng.integers(0, 256, n, dtype=np.uint8)
        for nt in range(1, 9):
            b = np.zeros(n, np.uint8)
            assert lib.vb_host_copy(b.ctypes.data, a.ctypes.data, n, nt) == 0
            assert np.array_equal(a, b), (n, nt)
