"""The C-ABI library builds, loads and exports every symbol include/saim.h declares (no GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "saim.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(saim_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for f in ["saim_create", "saim_run", "saim_get_info", "saim_destroy", "saim_last_error"]:
        assert f in names


def test_library_exports_every_declared_symbol():
    from paper_2501_04971_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_binding_lists_exports():
    import paper_2501_04971_b200 as P
    assert sorted(P.EXPORTS) == declared_functions()


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2501_04971_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "saim_oracle" not in txt, f


def test_create_rejects_bad_input_without_gpu():
    """Validation happens before any device call, so it is testable on a CPU box."""
    import numpy as np
    import paper_2501_04971_b200 as P
    with pytest.raises(P.SaimError) as ei:
        P.Solver([[0, 1], [2, 0]], [0, 0], [[1, 1]], [1], 1.0, 1.0, 1.0)   # asymmetric Q
    assert ei.value.code == P.SAIM_EINVAL
    with pytest.raises(P.SaimError) as ei:
        P.Solver(None, [0, 0], [[1, 1]], [0], 1.0, 1.0, 1.0)             # b < 1
    assert ei.value.code == P.SAIM_EINVAL
    with pytest.raises(P.SaimError) as ei:
        P.Solver([[1, 0], [0, 0]], [0, 0], [[1, 1]], [3], 1.0, 1.0, 1.0)  # nonzero diagonal
    assert ei.value.code == P.SAIM_EINVAL
    with pytest.raises(P.SaimError) as ei:
        P.Solver(None, [0, 0], [[1, 1]], [3], float("nan"), 1.0, 1.0)      # NaN P
    assert ei.value.code == P.SAIM_EINVAL
    with pytest.raises(P.SaimError) as ei:
        P.Solver(None, [0, 0], [[-1, 1]], [3], 1.0, 1.0, 1.0)              # A < 0
    assert ei.value.code == P.SAIM_EINVAL
    with pytest.raises(P.SaimError) as ei:
        P.Solver(None, [5000000, 0], [[1, 1]], [3], 1.0, 1.0, 1.0)         # |phi| >= 2^22
    assert ei.value.code == P.SAIM_ERANGE
    big = np.zeros((2, 2, 2), np.int32)
    big[:, 0, 1] = big[:, 1, 0] = 1
    with pytest.raises(P.SaimError) as ei:
        P.Solver(big, [[0, 0], [0, 0]], [[[1, 1], [1, 1]], [[1, 1], [1, 1]]], [[1, 1], [1, 1]], 1.0, 1.0, 1.0)
    assert ei.value.code == P.SAIM_EUNSUPPORTED                             # quadratic with M = 2
    for bad in (8192, P.FLAG_MKP_LOCKSTEP | P.FLAG_MKP_L2, P.FLAG_MKP_L2 | P.FLAG_MKP_L4, P.FLAG_MKP_SPLIT2 | P.FLAG_MKP_L4,
                P.FLAG_MKP_SPEC4 | P.FLAG_MKP_SPEC8, P.FLAG_MKP_SPEC8 | P.FLAG_MKP_L2):
        with pytest.raises(P.SaimError) as ei:                              # unknown / conflicting flags
            P.Solver(None, [0, 0], [[1, 1], [1, 0]], [3, 1], 1.0, 1.0, 1.0, flags=bad)
        assert ei.value.code == P.SAIM_EINVAL


def test_qkp_div_magic_table_is_exact():
    """The QKP hot step divides lane indices by the unsaturated width pw with the table
    kDivMagic[p] = ceil(2^16 / p) (saim_qkp.cuh): (x * m) >> 16 == x // p for every x <= 32."""
    import re
    src = open(os.path.join(os.path.dirname(__file__), "..", "paper_2501_04971_b200", "csrc", "saim_qkp.cuh")).read()
    body = re.search(r"kDivMagic\[33\]\s*=\s*\{([^}]*)\}", src).group(1)
    mag = [int(v) for v in body.replace("\n", " ").split(",") if v.strip()]
    assert len(mag) == 33
    for p in range(1, 33):
        for x in range(33):
            assert (x * mag[p]) >> 16 == x // p, (p, x)
