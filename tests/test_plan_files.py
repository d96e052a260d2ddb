"""Plan files (CPU): the reference JSON format and the binary .npz extension
round-trip every plan field, both for global and hierarchical plans (built
here from the reference's own golden plans, no GPU needed)."""

import numpy as np
import pytest

import paper_1802_03749_b200 as mp
from conftest import case_mesh, golden_cases, load_case
from helpers import reference_plan

CASES = [c for c in golden_cases() if c["reorder"] in ("none", "gps", "partition")][:12]


def _same(a, b):
    assert type(a) is type(b)
    assert a.kernel_key == b.kernel_key and a.config == b.config
    for name in a.set_perms:
        assert np.array_equal(a.set_perms[name].forward, b.set_perms[name].forward)
    for name, arr in a.mesh.data.items():
        assert np.array_equal(arr.values, b.mesh.data[name].values) and arr.layout == b.mesh.data[name].layout
    if isinstance(a, mp.GlobalPlan):
        assert np.array_equal(a.colours.colours, b.colours.colours)
        assert np.array_equal(a.colour_offsets, b.colour_offsets)
        return
    for f in ("block_offsets", "thread_colours", "thread_colour_counts", "shared_bytes"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(a.block_colours.colours, b.block_colours.colours)
    for d in ("staged", "written"):
        for k, (ip, ids) in getattr(a, d).items():
            ip2, ids2 = getattr(b, d)[k]
            assert np.array_equal(ip, ip2) and np.array_equal(ids, ids2)
            assert ip2.dtype == np.int64 and ids2.dtype == np.int64


@pytest.mark.parametrize("rec", CASES, ids=lambda c: c["file"])
@pytest.mark.parametrize("suffix", [".json", ".npz"])
def test_plan_file_round_trip(rec, suffix, tmp_path):
    z = load_case(rec)
    mesh = case_mesh(rec)
    kernel = mp.kernel_for_mesh(rec["kernel"], mesh)
    plan = reference_plan(rec, z, mesh, kernel)
    path = tmp_path / f"plan{suffix}"
    mp.save_plan(plan, path, mesh)
    _same(plan, mp.load_plan(path, mesh))


def test_binary_plan_rejects_other_mesh(tmp_path):
    rec = CASES[0]
    z = load_case(rec)
    mesh = case_mesh(rec)
    kernel = mp.kernel_for_mesh(rec["kernel"], mesh)
    path = tmp_path / "p.npz"
    mp.save_plan(reference_plan(rec, z, mesh, kernel), path, mesh)
    other = mp.generate_mesh("quad2d", (5, 4), dtype="f64")
    with pytest.raises((mp.MeshValidationError, mp.FileFormatError)):
        mp.load_plan(path, other)


def test_bad_binary_plan_is_a_format_error(tmp_path):
    path = tmp_path / "bad.npz"
    np.savez(path, x=np.arange(3))
    mesh = mp.generate_mesh("quad2d", (5, 4), dtype="f64")
    with pytest.raises(mp.FileFormatError):
        mp.load_plan(path, mesh)
