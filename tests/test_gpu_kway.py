"""GPU heavy-edge matching (mp_heavy_edge_matching_device) against the native
sequential sweep (itself checked against the oracle in test_kway_native.py),
and the whole k-way partition with either matching."""

import os

import numpy as np
import pytest
import torch

import paper_1802_03749_b200 as mp
from paper_1802_03749_b200 import _native, kway
from test_kway_native import _graph, p

pytestmark = pytest.mark.gpu


def _device_match(ip, ix, w, nw, visit, maxc):
    d = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
    return kway._match_device(d(ip), d(ix), d(w), d(nw), visit, maxc).cpu().numpy()


def _host_match(ip, ix, w, nw, visit, maxc):
    out = np.empty(len(nw), dtype=np.int64)
    _native.call("mp_heavy_edge_matching", len(nw), p(ip), p(ix), p(w), p(nw), p(visit), maxc, p(out))
    return out


@pytest.mark.parametrize("seed", range(20))
def test_device_matching_random_graphs(seed):
    ip, ix, w, rng = _graph(seed, n=int(np.random.default_rng(seed).integers(2, 400)))
    n = len(ip) - 1
    nw = rng.integers(1, 4, n).astype(np.int64)
    visit = rng.permutation(n).astype(np.int64)
    for maxc in (1, 2, 4, 8):
        assert np.array_equal(_device_match(ip, ix, w, nw, visit, maxc), _host_match(ip, ix, w, nw, visit, maxc))


@pytest.mark.parametrize("dims,family", [((300, 300), "quad2d"), ((24, 24, 24), "hex3d-faces")])
def test_device_matching_mesh_thread_graph(dims, family):
    mesh = mp.generate_mesh(family, dims, dtype="f64")
    m = next(iter(mesh.mappings.values()))
    g = kway.build_thread_graph([m])
    rng = np.random.default_rng(7)
    nw = rng.integers(1, 3, g.n).astype(np.int64)
    visit = rng.permutation(g.n).astype(np.int64)
    args = (g.indptr.astype(np.int64), g.indices.astype(np.int64), g.weights.astype(np.int64), nw, visit, 4)
    assert np.array_equal(_device_match(*args), _host_match(*args))


def test_partition_device_matching_equals_host(monkeypatch):
    mesh = mp.generate_mesh("quad2d", (120, 120), dtype="f64")
    m = next(iter(mesh.mappings.values()))
    g = kway.build_thread_graph([m])
    cfg = mp.PlanConfig(reorder="partition").partition_config()
    a = kway.partition_kway(g, cfg)
    monkeypatch.setenv("MESHPLAN_HOST_MATCHING", "1")
    b = kway.partition_kway(g, cfg)
    assert np.array_equal(a.assignment, b.assignment) and a.cut == b.cut


@pytest.mark.parametrize("cap", ["1", "2", "5"])
def test_device_matching_host_finish_after_round_cap(cap, monkeypatch):
    """Past the round cap the remaining turns run on the host in visit order:
    still the sequential matching."""
    monkeypatch.setenv("MESHPLAN_MATCH_ROUNDS", cap)
    for seed in range(6):
        ip, ix, w, rng = _graph(seed + 50, n=int(np.random.default_rng(seed).integers(40, 300)))
        n = len(ip) - 1
        nw = rng.integers(1, 3, n).astype(np.int64)
        visit = rng.permutation(n).astype(np.int64)
        assert np.array_equal(_device_match(ip, ix, w, nw, visit, 4), _host_match(ip, ix, w, nw, visit, 4))


def test_device_matching_path_graph_in_order():
    """An adversarial order (a path visited end to end: one ready node per
    round) still matches the sequential greedy."""
    n = 3000
    ip = np.concatenate(([0], np.cumsum([1] + [2] * (n - 2) + [1]))).astype(np.int64)
    ix = np.concatenate([[1]] + [[u - 1, u + 1] for u in range(1, n - 1)] + [[n - 2]]).astype(np.int64)
    w = np.ones(len(ix), dtype=np.int64)
    nw = np.ones(n, dtype=np.int64)
    visit = np.arange(n, dtype=np.int64)
    assert np.array_equal(_device_match(ip, ix, w, nw, visit, 2), _host_match(ip, ix, w, nw, visit, 2))
