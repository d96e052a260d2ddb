"""Block colouring on the GPU (plan.py:241-257).

``mp_plan_block_colours`` must reproduce the reference's sequential greedy
(``greedy_colour_csr``, numpy_impl.py:12-60, restated in
oracle/plans.py:18) with blocks as items, least-loaded and first-fit, and
the relabel by load (colouring.py:68-74).  Inputs are per-block ascending
unique written-point lists (what ``mp_plan_block_points`` produces).  The
golden plans (test_gpu_parity) and the BASELINE-size fingerprints
(test_gpu_configs) check it inside the planner; here it is exercised on
its own, including the paths the meshes rarely hit: more than 64 colours
(the wide pass), a block with more lower-id conflicts than a staged chunk
holds (read from global), and more blocks than the shared-memory colour
ring (old colours from L2).
"""

import numpy as np
import pytest
import torch

from oracle import plans as oracle_plans
from paper_1802_03749_b200 import gpuplan

pytestmark = pytest.mark.gpu


def _csr(lists):
    ptr = np.zeros(len(lists) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(x) for x in lists])
    ids = np.concatenate([np.asarray(sorted(set(x)), dtype=np.int64) for x in lists]) if lists else np.zeros(0)
    return ptr, ids.astype(np.int64)


def _device(ptr, ids):
    return (torch.as_tensor(ptr.astype(np.int32), device="cuda"),
            torch.as_tensor(ids.astype(np.int32), device="cuda"))


def _check(lists, least_loaded=True):
    lists = [sorted(set(x)) for x in lists]
    ptr, ids = _csr(lists)
    npts = int(ids.max()) + 1 if ids.size else 1
    want = oracle_plans.greedy_colour_csr(ptr, ids, npts, least_loaded)
    got, num, counts = gpuplan.colour_blocks_device(*_device(ptr, ids), least_loaded=least_loaded)
    got = got.cpu().numpy()
    if least_loaded and want.size:
        ref = oracle_plans.relabel_by_load(want, int(want.max()) + 1)
        want, want_counts = ref[0], ref[1]
        assert np.array_equal(counts, want_counts)
    assert num == (int(want.max()) + 1 if want.size else 0)
    assert np.array_equal(got, want)
    return num


def _random_blocks(rng, nb, npts, per_block, spread):
    out = []
    for b in range(nb):
        centre = int(b * npts / nb)
        k = int(rng.integers(1, per_block + 1))
        lo, hi = max(0, centre - spread), min(npts, centre + spread)
        out.append(rng.integers(lo, hi, size=k).tolist())
    return out


@pytest.mark.parametrize("least_loaded", [True, False])
@pytest.mark.parametrize("seed", [0, 1])
def test_random_banded_blocks(seed, least_loaded):
    rng = np.random.default_rng(seed)
    _check(_random_blocks(rng, 3000, 20000, 40, 300), least_loaded)


def test_more_blocks_than_the_colour_ring():
    # 40K blocks > GC_RING (16384): neighbours far back are read from L2
    rng = np.random.default_rng(3)
    lists = _random_blocks(rng, 40000, 200000, 30, 200)
    # long-range conflicts: every 1000th block also writes point 0..9
    for b in range(0, 40000, 1000):
        lists[b] = lists[b] + [b % 10]
    _check(lists)


def test_wide_pass_over_64_colours():
    # 100 blocks all writing point 0 -> 100 colours (the 1024-colour pass)
    lists = [[0, 1 + b] for b in range(100)] + [[1 + b, 500 + b] for b in range(300)]
    assert _check(lists) == 100
    assert _check(lists, least_loaded=False) == 100


def test_block_with_more_conflicts_than_a_chunk():
    # block N conflicts with all N earlier blocks (N > GC_PCAP = 12288)
    N = 20000
    lists = [[1 + b] for b in range(N)]
    lists.append([1 + b for b in range(N)])
    lists.append([1, 2])
    assert _check(lists) == 3


def test_empty_blocks_and_single_block():
    assert _check([[5]]) == 1
    assert _check([[], [1], [], [1], []]) >= 2


def test_golden_block_colourings():
    """Every hierarchical golden case: the device colouring of the
    reference's own written lists equals the reference's block colours."""
    from conftest import golden_cases, load_case

    n = 0
    for rec in golden_cases():
        if rec["strategy"] != "hier":
            continue
        z = load_case(rec)
        if "written_ptr" not in z or z["written_ptr"].size <= 1:
            continue
        ptr, ids = z["written_ptr"].astype(np.int64), z["written_ids"].astype(np.int64)
        got, num, _ = gpuplan.colour_blocks_device(*_device(ptr, ids))
        assert np.array_equal(got.cpu().numpy(), z["block_colours"]), rec["file"]
        n += 1
    assert n >= 20
