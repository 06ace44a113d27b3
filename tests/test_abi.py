"""CPU-side checks of the C-ABI boundary (no GPU needed, no compute calls)."""
import ctypes
import os
import re

import pytest

import __graft_entry__ as entry
import paper_2110_12511_b200 as pbng

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pbng.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pbng_[a-z_]+)\s*\(", src)))


def test_build_and_exports():
    entry.build()
    lib = ctypes.CDLL(pbng.LIB_PATH)
    declared = _declared()
    assert set(declared) == set(pbng.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert pbng.load_library().pbng_version().decode().startswith("pbng-b200")
    assert pbng.load_library().pbng_last_error() == b""


def test_sm100a_cubin():
    """The library carries sm_100a SASS (not PTX-only or another arch)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pbng.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_missing_library_fails_loudly(tmp_path):
    old = pbng._lib
    pbng._lib = None
    try:
        with pytest.raises(ImportError):
            pbng.load_library(str(tmp_path / "nope.so"))
    finally:
        pbng._lib = old


def test_struct_layouts_match_header(tmp_path):
    """sizeof / offsetof of the ABI structs as gcc compiles include/pbng.h = the ctypes binding's."""
    import subprocess
    fields = [f for f, _ in pbng.Stats._fields_]
    src = tmp_path / "lay.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "pbng.h"\nint main(void){'
                   'printf("%zu %zu", sizeof(pbng_csr), sizeof(pbng_stats));'
                   + "".join(f'printf(" %zu", offsetof(pbng_stats, {f}));' for f in fields)
                   + 'printf(" %u\\n", PBNG_MAX_P); return 0;}')
    exe = tmp_path / "lay"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    vals = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    assert vals[0] == ctypes.sizeof(pbng.Csr)
    assert vals[1] == ctypes.sizeof(pbng.Stats)
    assert vals[2:-1] == [getattr(pbng.Stats, f).offset for f in fields]
    assert vals[-1] == pbng.MAX_P == 4096
