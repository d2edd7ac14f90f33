"""CPU checks of the C-ABI library: it loads, exports every symbol include/love.h declares, and
the ctypes structs match the header's layout.  No compute calls (no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "love.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(love_[a-z_]+)\s*\(", src)
    return sorted(set(names))


def _lib():
    from paper_1803_06058_b200 import _abi
    if not os.path.exists(_abi.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return _abi, _abi.load()


def test_header_declares_the_north_star_calls():
    names = _declared_functions()
    for required in ["love_build_cache", "love_predict_var", "love_predict_covar", "love_sample"]:
        assert required in names


def test_library_exports_every_declared_symbol():
    _abi, lib = _lib()
    names = _declared_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n
        assert n in _abi.SIGNATURES, f"binding lacks {n}"


def test_no_gpu_calls_are_safe():
    _abi, lib = _lib()
    assert lib.love_abi_version() == 4
    assert lib.love_launch_count() >= 0
    # argument validation happens before any device work
    out = ctypes.c_void_p()
    st = lib.love_build_cache(None, None, 0.1, None, None, 0, 1, None, None, None, ctypes.byref(out))
    assert st == _abi.LOVE_ERR_ARG
    assert b"NULL" in lib.love_last_error()
    g = _abi.love_grid()
    g.d = 1
    g.m[0], g.lo[0], g.h[0] = 3, 0.0, 0.1          # m < 4
    r = _abi.love_rbf(1.0, (ctypes.c_double * 3)(0.1, 0, 0))
    st = lib.love_build_cache(ctypes.byref(g), ctypes.byref(r), 0.1, None, None, 0, 1, None, None, None,
                              ctypes.byref(out))
    assert st == _abi.LOVE_ERR_ARG
    lib.love_free(None)


def test_struct_layouts_match_header(tmp_path):
    """Compile a C probe against include/love.h and compare sizeof/offsetof with ctypes."""
    import subprocess
    from paper_1803_06058_b200 import _abi
    structs = {"love_grid": _abi.love_grid, "love_rbf": _abi.love_rbf, "love_opts": _abi.love_opts,
               "love_dist": _abi.love_dist, "love_info": _abi.love_info, "love_axis": _abi.love_axis}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} sizeof %zu\\n", sizeof({name}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{name} {fname} %zu\\n", offsetof({name}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    for line in filter(None, got):
        name, field, val = line.split()
        cls = structs[name]
        want = ctypes.sizeof(cls) if field == "sizeof" else getattr(cls, field).offset
        assert int(val) == want, line


def test_product_path_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1803_06058_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
