"""Pin the oracle: every oracle function against the reference's own outputs.

Golden vectors come from tests/golden/make_golden.py (the real reference,
run in the build container).  CPU only.
"""

import numpy as np
import pytest

from conftest import DIR_OF, INC_OF, READ_OF, bit_equal, case_mesh, golden_cases, load_case
from oracle import loops, plans

CASES = golden_cases()


def _ids(c):
    return f"{c['file']}-{c['family']}-{c['kernel']}-{c['dtype']}-{c['strategy']}-{c['reorder']}"


def _arrays(mesh, kernel_name):
    m = next(iter(mesh.mappings.values()))
    ind = mesh.data[READ_OF[kernel_name]].view2d() if kernel_name in READ_OF else None
    return m.table, ind, np.ascontiguousarray(mesh.data[DIR_OF[kernel_name]].view2d()), \
        np.ascontiguousarray(mesh.data[INC_OF[kernel_name]].view2d())


@pytest.mark.parametrize("rec", CASES, ids=_ids)
def test_oracle_serial_matches_reference(rec):
    z = load_case(rec)
    mesh = case_mesh(rec)
    t, ind, d, inc = _arrays(mesh, rec["kernel"])
    assert bit_equal(loops.serial_loop(rec["kernel"], t, ind, d, inc), z["serial_inc"])
    rmesh = case_mesh(rec, random=True, arrays=z)
    t, ind, d, inc = _arrays(rmesh, rec["kernel"])
    assert bit_equal(loops.serial_loop(rec["kernel"], t, ind, d, inc), z["rand_serial_inc"])


@pytest.mark.parametrize("rec", CASES, ids=_ids)
def test_oracle_same_plan_executor_bit_exact(rec):
    """Oracle global/hier executors on the reference plan reproduce the
    reference executor bit for bit on non-quantised data."""
    z = load_case(rec)
    rmesh = case_mesh(rec, random=True, arrays=z)
    t, ind, d, inc = _arrays(rmesh, rec["kernel"])
    efwd, pfwd = z["elem_fwd"], z["point_fwd"]
    einv, pinv = np.argsort(efwd), np.argsort(pfwd)
    t2 = pfwd[t[einv]]
    assert np.array_equal(t2, z["plan_table"])
    ind2 = None if ind is None else ind[pinv]
    d2, inc2 = d[einv], inc[pinv]
    if rec["strategy"] == "global":
        out = loops.global_loop(rec["kernel"], t2, ind2, d2, inc2, z["colour_offsets"])
    else:
        out = loops.hier_loop(rec["kernel"], t2, ind2, d2, inc2, z["block_offsets"], z["block_colours"],
                              z["thread_colours"], (z["staged_ptr"], z["staged_ids"]),
                              (z["written_ptr"], z["written_ids"]))
    assert bit_equal(out, z["rand_exec_inc"])


PLAN_CASES = [c for c in CASES if c["reorder"] in ("none", "gps")]


@pytest.mark.parametrize("rec", PLAN_CASES, ids=_ids)
def test_oracle_plans_match_reference(rec):
    z = load_case(rec)
    mesh = case_mesh(rec)
    m = next(iter(mesh.mappings.values()))
    npts = m.to_set.size
    wslots = list(range(m.arity))
    if rec["strategy"] == "global":
        p = plans.global_plan(m.table, npts, wslots, rec["reorder"])
        assert np.array_equal(p["colour_offsets"], z["colour_offsets"])
        assert np.array_equal(p["colours"], z["colours"])
    else:
        p = plans.hier_plan(m.table, npts, wslots, wslots, rec["block_size"], rec["reorder"])
        assert np.array_equal(p["block_offsets"], z["block_offsets"])
        assert np.array_equal(p["block_colours"], z["block_colours"])
        assert np.array_equal(p["thread_colours"], z["thread_colours"])
        assert np.array_equal(p["thread_colour_counts"], z["thread_colour_counts"])
        assert np.array_equal(p["staged"][0], z["staged_ptr"]) and np.array_equal(p["staged"][1], z["staged_ids"])
        assert np.array_equal(p["written"][1], z["written_ids"])
    assert np.array_equal(p["elem_fwd"], z["elem_fwd"])
    assert np.array_equal(p["point_fwd"], z["point_fwd"])
    assert np.array_equal(p["table"], z["plan_table"])


def test_known_answers():
    # reference known-answer tests
    assert plans.effective_block_size(480, 1.001, 0.5) == (479, 480.5 / 479)  # test_partition.py:47-52
    col = plans.thread_colours_for_block(np.array([[0, 1], [1, 2], [2, 3], [3, 0]]))
    assert col.max() + 1 == 2
    # one edge pair sharing a cell -> 2 global colours; disjoint -> 1 (test_plan.py:55-65)
    assert plans.global_plan(np.array([[0, 1], [1, 2]]), 3, [0, 1])["colour_offsets"].tolist() == [0, 1, 2]
    assert plans.global_plan(np.array([[0, 1], [2, 3]]), 4, [0, 1])["colour_offsets"].tolist() == [0, 2]
    # stable colour sort [1,0,1,0] -> order [1,3,0,2] (test_colouring.py:122-125)
    assert np.argsort(np.array([1, 0, 1, 0]), kind="stable").tolist() == [1, 3, 0, 2]


# ---- the oracle at the BASELINE config sizes ------------------------------------------


def _fingerprints():
    import json

    from conftest import GOLDEN

    return json.loads((GOLDEN / "fingerprints.json").read_text())


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_oracle_serial_matches_reference_at_config_size(name):
    """The oracle's serial loop on the full C1 / C2 mesh (seed 0, the
    package generator, bit-identical to the reference's) reproduces the
    CRC32 of the reference execute_serial result (make_fingerprints.py)."""
    import zlib

    import paper_1802_03749_b200 as mp

    rec = _fingerprints()[name]
    mesh = mp.generate_mesh(rec["family"], tuple(rec["dims"]), seed=rec["seed"], dtype=rec["dtype"],
                            arrays=mp.workloads.arrays_for_kernel(rec["kernel"]))
    t, ind, d, inc = _arrays(mesh, rec["kernel"])
    got = np.ascontiguousarray(loops.serial_loop(rec["kernel"], t, ind, d, inc))
    assert got.shape[0] == rec["n_points"]
    assert (zlib.crc32(got.tobytes()) & 0xFFFFFFFF) == rec["serial"]["crc32"]
    assert float(np.abs(got).sum()) == rec["serial_abs_sum"]
