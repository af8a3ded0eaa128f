"""C-ABI checks that run without a GPU: the library loads, exports every
symbol include/hxf.h declares, and fails loudly (no CPU fallback) when no
device is present."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, has_cuda
from paper_1401_6961_b200 import _native, basis, inputs
from paper_1401_6961_b200.basis import InvalidArgumentError

HEADER = os.path.join(ROOT, "include", "hxf.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(hxf_[a-z0-9_]+)\s*\(", text)))


def test_header_declarations_match_binding_list():
    assert _declared() == sorted(_native.EXPORTED)


def test_library_exports_every_symbol():
    lib = _native.lib()
    for name in _declared():
        assert hasattr(lib, name), name


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of hxf_counters / hxf_exchange_opts == the C compiler's layout."""
    import subprocess
    src = tmp_path / "layout.c"
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "hxf.h"', "int main(void) {"]
    structs = (("hxf_counters", _native.Counters), ("hxf_exchange_opts", _native.ExchangeOpts),
               ("hxf_tie_record", _native.TieRecord))
    for cname, py in structs:
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0; }")
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                 check=True).stdout.splitlines())
    for cname, py in structs:
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, (cname, f)


def test_version():
    assert _native.lib().hxf_version() == 1


@pytest.mark.skipif(has_cuda(), reason="checks the no-device path")
def test_no_device_fails_loudly():
    from paper_1401_6961_b200 import basis, quadtree
    system = inputs.generate_cluster(1, seed=3)
    part = quadtree.build_partition(system)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        quadtree.build_pair_tree(system, part)


def test_partition_matches_reference_rules():
    from paper_1401_6961_b200 import basis, quadtree
    shells = [basis.GaussianShell(center=[i, 0.0, 0.0], primitives=[(1.0, 1.0)]) for i in range(13)]
    system = basis.BasisSystem(shells=basis.assign_offsets(shells), atoms=[])
    part = quadtree.build_partition(system, leaf_size=10)
    assert (part.root.left.n_functions, part.root.right.n_functions) == (6, 7)
    with pytest.raises(InvalidArgumentError):
        quadtree.build_partition(system, leaf_size=0)
