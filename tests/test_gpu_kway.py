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
