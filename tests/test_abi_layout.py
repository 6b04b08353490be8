"""The record layouts the Python side reads (numpy dtypes) against the C
headers they mirror: every field's offset and the record size, from offsetof
/ sizeof in a small C program compiled here with gcc (no GPU). Guards the
debug-record ABI (glint.h 2.1, 184 words) and the oracle's twin record."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _c_offsets(header_dir, header, struct, fields):
    src = [f'#include <stdio.h>\n#include <stddef.h>\n#include "{header}"\nint main(void) {{',
           f'  printf("size %zu\\n", sizeof({struct}));']
    src += [f'  printf("{f} %zu\\n", offsetof({struct}, {f}));' for f in fields]
    src += ["  return 0;", "}"]
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "t.c"), os.path.join(d, "t")
        open(c, "w").write("\n".join(src))
        subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", header_dir, c, "-o", exe], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.split("\n")
    return {k: int(v) for k, v in (l.split() for l in out if l)}


def _check(dtype, offs):
    assert offs["size"] == dtype.itemsize
    for f in dtype.names:
        if f in offs:
            assert offs[f] == dtype.fields[f][1], f


def test_debug_record_matches_glint_h():
    from paper_2306_05051_b200 import _lib
    dt = _lib.DEBUG_REC_DTYPE
    offs = _c_offsets(os.path.join(ROOT, "include"), "glint.h", "glint_debug_rec", dt.names)
    _check(dt, offs)
    assert offs["size"] == 184 * 4


def test_oracle_record_matches_its_header():
    import oracle
    dt = oracle.REC_DTYPE
    offs = _c_offsets(os.path.join(ROOT, "oracle"), "glint_oracle.h", "orc_rec", dt.names)
    _check(dt, offs)
    assert offs["size"] == 184 * 4


@pytest.mark.parametrize("name", ["glint_gbuffer", "glint_scene", "glint_light"])
def test_ctypes_structs_match_glint_h(name):
    from paper_2306_05051_b200 import _lib
    import ctypes
    st = getattr(_lib, name)
    fields = [f[0] for f in st._fields_ if not f[0].startswith("pad")]
    offs = _c_offsets(os.path.join(ROOT, "include"), "glint.h", name, fields)
    assert offs["size"] == ctypes.sizeof(st)
    for f in fields:
        assert offs[f] == getattr(st, f).offset, f
