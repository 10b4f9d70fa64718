"""CPU checks of the C-ABI boundary: the shared library loads on a machine without a GPU and
exports every entry point include/mpmlite.h declares; the binding covers all of them.  No compute
calls are made here (they need a GPU)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "mpmlite.h")).read()
    return sorted(set(re.findall(r"^MPL_API[^;(]*?\b(mpl_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_entry_points():
    syms = header_symbols()
    for s in ("mpl_create", "mpl_resample", "mpl_gradient", "mpl_hvp", "mpl_newton_step",
              "mpl_transfer_to_particles", "mpl_step", "mpl_energy", "mpl_linearize"):
        assert s in syms
    assert len(syms) >= 25


def test_library_loads_and_exports_every_symbol():
    from paper_2602_07853_b200 import build
    path = build.build()
    lib = ctypes.CDLL(path)
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    lib.mpl_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.mpl_version()


def test_binding_covers_header():
    from paper_2602_07853_b200 import mpl
    assert set(header_symbols()) == set(mpl._SIGS)


def test_library_is_sm100a():
    """The fatbin holds sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    from paper_2602_07853_b200 import build
    path = build.build()
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        return
    out = subprocess.run([exe, "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
