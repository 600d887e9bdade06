"""C-ABI struct layouts: the ctypes mirrors in the binding must match include/fms.h field by
field -- a field appended to one side only would make the library write past or misread the caller's
struct.  A small C program compiled against the header prints sizeof and every field's offsetof."""
import ctypes as C
import os
import subprocess
import tempfile

import pytest

import paper_2007_14283_b200 as fms

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STRUCTS = {"fms_seed_policy": fms.Policy, "fms_frame_stats": fms.FrameStats, "fms_run_stats": fms.RunStats}


def _c_layout():
    lines = ["#include <stddef.h>", "#include <stdio.h>", '#include "fms.h"', "int main(void) {"]
    for cname, cls in STRUCTS.items():
        lines.append(f'  printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for name, _ in cls._fields_:
            lines.append(f'  printf("{cname} {name} %zu\\n", offsetof({cname}, {name}));')
    lines += ["  return 0;", "}"]
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "layout.c"), os.path.join(d, "layout")
        with open(src, "w") as f:
            f.write("\n".join(lines) + "\n")
        subprocess.check_call(["gcc", "-std=c11", "-I" + os.path.join(ROOT, "include"), "-o", exe, src])
        out = subprocess.check_output([exe], text=True)
    got = {}
    for ln in out.splitlines():
        s, field, val = ln.split()
        got[(s, field)] = int(val)
    return got


@pytest.mark.parametrize("cname", sorted(STRUCTS))
def test_struct_layout_matches_header(cname):
    got = _c_layout()
    cls = STRUCTS[cname]
    assert got[(cname, "sizeof")] == C.sizeof(cls), (cname, got[(cname, "sizeof")], C.sizeof(cls))
    for name, _ in cls._fields_:
        assert got[(cname, name)] == getattr(cls, name).offset, (cname, name)
