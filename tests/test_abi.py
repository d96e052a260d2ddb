"""The C-ABI library loads on a CPU-only host and exports every symbol the
header declares; host-side entry points run without a GPU."""

import re
from pathlib import Path

import numpy as np
import pytest

from paper_1802_03749_b200 import _native, colouring
from oracle import plans

HEADER = Path(__file__).resolve().parents[1] / "include" / "meshplan_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(mp_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = _native.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared_symbols()) == set(_native.exported_symbols())


def test_struct_layout_matches_header(tmp_path):
    """ctypes mirrors of mp_loop / mp_hier_plan agree with the C compiler."""
    import shutil
    import subprocess

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    fields = {"mp_loop": _native.MpLoop, "mp_hier_plan": _native.MpHierPlan}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, py in fields.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([cc, str(src), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n")
               if line)
    for cname, py in fields.items():
        assert int(got[cname]) == __import__("ctypes").sizeof(py)
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, (cname, f)


def test_version_string():
    assert b"sm_100a" in _native.load().mp_version()


def _random_csr(rng, n, npts, k):
    rows = [np.unique(rng.integers(0, npts, rng.integers(0, k + 1))) for _ in range(n)]
    indptr = np.concatenate(([0], np.cumsum([r.size for r in rows]))).astype(np.int64)
    return indptr, (np.concatenate(rows) if rows else np.empty(0)).astype(np.int64)


@pytest.mark.parametrize("seed", range(12))
def test_native_greedy_csr_bit_identical(seed):
    rng = np.random.default_rng(seed)
    indptr, idx = _random_csr(rng, int(rng.integers(1, 300)), int(rng.integers(1, 80)), 4)
    for ll in (True, False):
        assert np.array_equal(colouring.greedy_colour_csr(indptr, idx, 80, ll),
                              plans.greedy_colour_csr(indptr, idx, 80, ll))


@pytest.mark.parametrize("seed", range(12))
def test_native_smallest_last_and_adj(seed):
    rng = np.random.default_rng(seed)
    k = int(rng.integers(1, 120))
    dense = rng.random((k, k)) < rng.uniform(0.02, 0.3)
    dense = np.triu(dense, 1)
    dense = dense | dense.T
    indptr = np.concatenate(([0], np.cumsum(dense.sum(1)))).astype(np.int64)
    idx = np.nonzero(dense)[1].astype(np.int64)
    o_ref = plans.smallest_last_order(indptr, idx)
    assert np.array_equal(colouring.smallest_last_order(indptr, idx), o_ref)
    for ll in (False, True):
        assert np.array_equal(colouring.greedy_colour_adj(indptr, idx, o_ref, ll),
                              plans.greedy_colour_adj(indptr, idx, o_ref, ll))


def test_status_codes_map_to_reference_errors():
    from paper_1802_03749_b200 import errors

    with pytest.raises(errors.RaceError):
        errors.raise_for_status(3, "x")
    with pytest.raises(errors.CapacityError):
        errors.raise_for_status(4, "x")
    with pytest.raises(errors.KernelSpecError):
        errors.raise_for_status(2, "x")
    errors.raise_for_status(0, "")
