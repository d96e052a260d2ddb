"""Shared fixtures: golden cases produced by the real reference, helpers."""

import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

GOLDEN = REPO / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")
    config.addinivalue_line("markers", "slow: full-size BASELINE configs (minutes; -m gpu runs them)")


def pytest_collection_modifyitems(config, items):
    """gpu-marked tests skip (instead of failing) on a host without CUDA."""
    if has_gpu() or os.environ.get("MESHPLAN_FORCE_GPU_TESTS"):
        return
    skip = pytest.mark.skip(reason="needs a CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def golden_cases():
    return json.loads((GOLDEN / "manifest.json").read_text())


def load_case(rec):
    with np.load(GOLDEN / rec["file"]) as z:
        return {k: z[k] for k in z.files}


INC_OF = {"flux": "res", "flux-noread": "res", "scatter8": "force", "face-flux": "flux", "face-flux-heavy": "flux"}
READ_OF = {"flux": "q", "face-flux": "state", "face-flux-heavy": "state"}
DIR_OF = {"flux": "w", "flux-noread": "w", "scatter8": "stress", "face-flux": "facew", "face-flux-heavy": "facew"}
OP_WSLOTS = {"scatter8": list(range(8))}


def case_mesh(rec, random=False, arrays=None):
    """The case's mesh from this package's generator (bit-equal to the
    reference generator), optionally with the stored random values."""
    from paper_1802_03749_b200 import workloads
    from paper_1802_03749_b200.mesh import DataArray

    mesh = workloads.generate_mesh(rec["family"], tuple(rec["dims"]), seed=rec["seed"], dtype=rec["dtype"])
    if random:
        arrays = arrays if arrays is not None else load_case(rec)
        new = []
        for name, a in mesh.data.items():
            v2 = arrays[f"rand_{name}"]
            new.append(DataArray(a.name, a.set, a.components, np.ascontiguousarray(v2).ravel(), "aos"))
        mesh = mesh.with_data(*new)
    return mesh


def bit_equal(a, b) -> bool:
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if a.dtype.kind == "f":
        return np.array_equal(a.view(np.uint8), b.view(np.uint8))
    return np.array_equal(a, b)


@pytest.fixture(scope="session")
def cases():
    return golden_cases()


gpu = pytest.mark.skipif(not has_gpu() and not os.environ.get("MESHPLAN_FORCE_GPU_TESTS"), reason="needs a CUDA device")
