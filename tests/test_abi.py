"""CPU-side checks of the C-ABI boundary: the library builds/loads and exports every symbol that
include/libfem.h declares; host-side marshalling is consistent.  No compute calls (no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "libfem.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s+(fem_[a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_four_hot_path_calls():
    names = declared_functions()
    for n in ["fem_mesh_create", "fem_pattern_build", "fem_assemble_matrix", "fem_assemble_residual"]:
        assert n in names


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2111_03541_b200 import build, fem
    build.build()
    lib = ctypes.CDLL(fem.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared_functions()) == set(fem.EXPORTED)
    assert lib.fem_version() == 1


def test_problem_marshalling_layout():
    from fem_inputs import make_config
    from paper_2111_03541_b200 import fem
    for name, dims in [("c1", (4,)), ("c2", (2, 2, 2)), ("c3", (2, 1, 1)), ("c4", (2, 1, 1)), ("c5", (2, 2, 2))]:
        m, p = make_config(name, "structured", dims)
        P = fem.make_problem(p)
        assert P.n_terms == len(p.terms)
        for i, t in enumerate(p.terms):
            assert P.terms[i].form == fem.FORM[t.form]
            assert P.terms[i].region == t.region
    assert ctypes.sizeof(fem.fem_term) == 8 + 16 * 8
    # fem_problem: 4 ints, time scheme (2 ints + 6 doubles), n_terms, 16 terms
    assert ctypes.sizeof(fem.fem_time_scheme) == 8 + 6 * 8


def test_invalid_arguments_fail_loudly_without_gpu():
    """Host-side validation runs before any device work: bad element ids are rejected."""
    import numpy as np
    from fem_inputs import make_config
    from paper_2111_03541_b200 import fem
    m, p = make_config("c1", "structured", (2,))
    m.conn = m.conn.copy()
    m.conn[0, 0] = 10_000
    with pytest.raises(fem.FemError) as ei:
        fem.fem_mesh_create(p, m, stream=0)
    assert ei.value.code == -1
    m2, p2 = make_config("c1", "structured", (2,))
    p2.etype = "hex"
    with pytest.raises(fem.FemError) as ei:
        fem.fem_mesh_create(p2, m2, stream=0)
    assert ei.value.code == -2
    assert np is not None
