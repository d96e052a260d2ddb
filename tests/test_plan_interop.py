"""Plan-file interoperability with the reference (plan.py:619-755).

``tests/golden/plans/*.json`` were written by the REAL reference's
``save_plan`` (tests/golden/make_plan_json.py).  Checked here:

* CPU: this package's ``load_plan`` reads each reference file against the
  mesh from this package's generator, and its ``save_plan`` writes the loaded
  plan back byte for byte identical -- the two formats are the same format;
* CPU, where the reference package is importable (the build container, or
  ``baseline/_ref`` staged by tools/stage_reference.sh): the reference's own
  ``load_plan`` reads a file this package wrote;
* GPU: the GPU planner's plan of the same mesh and config, saved by this
  package, has the reference file's content in every field except the
  hardware descriptor (plans built here describe the B200, the reference's
  default is its P100 model), and the reference loads it.
"""

import importlib
import json
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1802_03749_b200 as mp
from conftest import REPO, gpu

PLANS = REPO / "tests" / "golden" / "plans"
MANIFEST = json.loads((PLANS / "manifest.json").read_text())


def _mesh(rec):
    return mp.generate_mesh(rec["family"], tuple(rec["dims"]), seed=0, dtype=rec["dtype"])


def _reference():
    """The reference package (a separate module tree), or None."""
    for root in (REPO / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (root / "meshplan" / "__init__.py").exists():
            saved = {k: v for k, v in sys.modules.items() if k == "meshplan" or k.startswith("meshplan.")}
            for k in saved:
                del sys.modules[k]
            sys.path.insert(0, str(root))
            try:
                ref = importlib.import_module("meshplan")
                importlib.import_module("meshplan.bench_kernels")
                return ref
            except Exception:
                return None
            finally:
                sys.path.remove(str(root))
    return None


@pytest.mark.parametrize("name", sorted(MANIFEST))
def test_reference_plan_file_loads_and_rewrites_identically(name, tmp_path):
    rec = MANIFEST[name]
    mesh = _mesh(rec)
    src = PLANS / f"{name}.json"
    plan = mp.load_plan(src, mesh)
    assert plan.config.strategy == rec["config"]["strategy"]
    data = json.loads(src.read_text())
    if "hier" in data:
        assert np.array_equal(plan.block_offsets, data["hier"]["block_offsets"])
        assert np.array_equal(plan.thread_colours, data["hier"]["thread_colours"])
    else:
        assert np.array_equal(plan.colour_offsets, data["global"]["colour_offsets"])
    out = tmp_path / "again.json"
    mp.save_plan(plan, out, mesh=mesh)
    assert out.read_bytes() == src.read_bytes()


def test_reference_reads_a_plan_file_written_here(tmp_path):
    ref = _reference()
    if ref is None:
        pytest.skip("reference package not importable here")
    from meshplan.bench_kernels import generate_mesh as ref_generate

    for name, rec in sorted(MANIFEST.items()):
        mesh = _mesh(rec)
        plan = mp.load_plan(PLANS / f"{name}.json", mesh)
        out = tmp_path / f"{name}.json"
        mp.save_plan(plan, out, mesh=mesh)
        rmesh = ref_generate(rec["family"], tuple(rec["dims"]), seed=0, dtype=rec["dtype"])
        rplan = ref.load_plan(out, rmesh)
        for s, perm in plan.set_perms.items():
            assert np.array_equal(rplan.set_perms[s].forward, perm.forward)
        if "hier" in rec["config"]["strategy"]:
            assert np.array_equal(rplan.block_colours.colours, plan.block_colours.colours)


@gpu
@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(MANIFEST))
def test_gpu_planner_writes_the_reference_plan_file(name, tmp_path):
    rec = MANIFEST[name]
    mesh = _mesh(rec)
    kernel = mp.kernel_for_mesh(rec["kernel"], mesh)
    cfg = mp.PlanConfig(**rec["config"])
    plan = (mp.build_global_plan if cfg.strategy == "global" else mp.build_hierarchical_plan)(mesh, kernel, cfg)
    out = tmp_path / "gpu.json"
    mp.save_plan(plan, out, mesh=mesh)
    got, want = json.loads(out.read_text()), json.loads((PLANS / f"{name}.json").read_text())
    assert got.pop("hw")["name"] == "b200" and want.pop("hw")["name"] == "p100"
    assert set(got) == set(want)
    for key in want:
        assert got[key] == want[key], key
    ref = _reference()
    if ref is not None:
        from meshplan.bench_kernels import generate_mesh as ref_generate

        rplan = ref.load_plan(out, ref_generate(rec["family"], tuple(rec["dims"]), seed=0, dtype=rec["dtype"]))
        assert rplan.kernel_key == plan.kernel_key
