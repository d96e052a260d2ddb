"""Execution plans: configuration, plan objects, the two builders, plan files.

Public names, plan fields, error texts and the JSON file format are the
reference's (pkg/src/meshplan/plan.py:51-755), so plans interchange with
``meshplan`` and existing callers keep working.  What differs is where the
work happens: the builders run the planner on the GPU (``gpuplan``) and the
sequential greedy colourings in native C++, and every plan keeps its
execution structures resident on the device (``plan._device``) so the
executors launch without re-uploading or re-deriving anything.
"""

import json
import zlib
from dataclasses import dataclass, field, replace

import numpy as np

from .colouring import ColourAssignment, colour_csr_least_loaded
from .errors import CapacityError, FileFormatError, KernelSpecError, MeshValidationError
from .hardware import B200, HardwareDescriptor
from .kernelspec import KernelSpec
from .mesh import DataArray, Mapping, Mesh, apply_permutation, transform_layout, validate_mesh
from .partition import PartitionConfig, chunk_partition, compute_effective_block_size, partition_structured_hex
from .permutation import Permutation

PLAN_HEADER = "meshplan-plan 1"
STRATEGIES = ("global", "hier")
REORDER_MODES = ("none", "gps", "partition", "cluster")  # "cluster": GPU extension (cluster.py)
STAGING_MODES = ("all-indirect", "increment-only")
MAPPING_ENTRY_BYTES = 4  # device mapping entries are int32


@dataclass(frozen=True)
class PlanConfig:
    strategy: str = "hier"
    reorder: str = "none"
    layout: str = "aos"
    staging: str = "all-indirect"
    block_size: int = 128
    tolerance: float = 1.001
    epsilon: float = 0.5
    seed: int = 0
    unweighted_cut: bool = False
    wide_transfers: bool = False

    def __post_init__(self):
        if self.strategy not in STRATEGIES:
            raise MeshValidationError(f"unknown strategy {self.strategy!r}")
        if self.layout not in ("aos", "soa"):
            raise MeshValidationError(f"unknown layout {self.layout!r}")
        if self.staging not in STAGING_MODES:
            raise MeshValidationError(f"unknown staging mode {self.staging!r}")
        if self.reorder.split(":", 1)[0] not in REORDER_MODES + ("structured",):
            raise MeshValidationError(f"unknown reorder mode {self.reorder!r}")

    def partition_config(self) -> PartitionConfig:
        return PartitionConfig(self.block_size, self.tolerance, self.epsilon, self.seed, self.unweighted_cut)

    def structured_shape(self):
        if not self.reorder.startswith("structured"):
            return None
        parts = self.reorder.partition(":")[2].replace(",", " ").split()
        if len(parts) not in (2, 3):  # bx,by: quad2d tiles (extension)
            raise MeshValidationError(f"structured reorder needs bx,by,bz, got {self.reorder!r}")
        return tuple(int(p) for p in parts)


@dataclass(frozen=True)
class GlobalPlan:
    mesh: Mesh
    kernel_key: str
    config: PlanConfig
    hw: HardwareDescriptor
    set_perms: dict
    colours: ColourAssignment
    colour_offsets: np.ndarray
    array_layouts: dict
    mapping_layout: str = "aos"

    @property
    def num_colours(self) -> int:
        return self.colours.num_colours

    def colour_range(self, c: int) -> tuple:
        return int(self.colour_offsets[c]), int(self.colour_offsets[c + 1])

    def restore_data(self, result: Mesh) -> Mesh:
        return restore(self, result)


@dataclass(frozen=True)
class HierarchicalPlan:
    mesh: Mesh
    kernel_key: str
    config: PlanConfig
    hw: HardwareDescriptor
    set_perms: dict
    block_offsets: np.ndarray
    block_colours: ColourAssignment
    thread_colours: np.ndarray
    thread_colour_counts: np.ndarray
    staged: dict
    written: dict
    shared_bytes: np.ndarray
    refs_per_element: int
    partition_meta: dict = field(default_factory=dict)
    array_layouts: dict = field(default_factory=dict)
    mapping_layout: str = "soa"

    @property
    def num_blocks(self) -> int:
        return len(self.block_offsets) - 1

    def block_range(self, b: int) -> tuple:
        return int(self.block_offsets[b]), int(self.block_offsets[b + 1])

    def working_threads(self) -> np.ndarray:
        return np.diff(self.block_offsets)

    def staged_slots(self, set_name: str, block: int, points) -> np.ndarray:
        """Shared slot of each point: its position in the block's staged list."""
        indptr, ids = self.staged[set_name]
        lst = ids[indptr[block]: indptr[block + 1]]
        points = np.asarray(points)
        if lst.size == 0:
            if points.size == 0:
                return np.empty(0, dtype=np.int64)
            raise CapacityError(f"block {block}: nothing staged on set {set_name!r} but accesses exist")
        pos = np.searchsorted(lst, points)
        ok = (pos < lst.size) & (lst[np.minimum(pos, lst.size - 1)] == points)
        if not np.all(ok):
            raise CapacityError(f"block {block}: access to a point missing from its staging list on set {set_name!r}")
        return pos

    def restore_data(self, result: Mesh) -> Mesh:
        return restore(self, result)


def reuse_factor(plan: HierarchicalPlan) -> float:
    """Indirect references per staged point (plan.py:188-198)."""
    staged = sum(int(indptr[-1]) for indptr, _ in plan.staged.values())
    if staged == 0:
        return 1.0
    return plan.refs_per_element * int(plan.block_offsets[-1]) / staged


def restore(plan, result: Mesh) -> Mesh:
    """Map a plan-numbered result back to the original numbering."""
    out = result
    for name, perm in plan.set_perms.items():
        if not perm.is_identity():
            out = apply_permutation(out, name, perm.inverted())
    return out


# ------------------------------------------------------------------------------
# builders
# ------------------------------------------------------------------------------


def _check_valid(mesh: Mesh, kernel: KernelSpec) -> None:
    rep = validate_mesh(mesh)
    if not rep.valid:
        raise MeshValidationError(f"invalid mesh:\n{rep}")
    kernel.validate_against(mesh)


def _layouts(mesh: Mesh, kernel: KernelSpec, config: PlanConfig) -> dict:
    ind = {a.array for a in kernel.indirect_args}
    direct = {a.array for a in kernel.direct_args}
    if ind & direct:
        raise KernelSpecError(f"arrays accessed both directly and indirectly: {sorted(ind & direct)}")
    out = {}
    for name, arr in mesh.data.items():
        out[name] = config.layout if name in ind else ("soa" if name in direct else arr.layout)
    return out


def _refs_per_element(mesh, kernel) -> int:
    total = 0
    for mname in kernel.mapping_names():
        slots = set()
        for a in kernel.indirect_args:
            if a.mapping == mname:
                slots.update(kernel.arg_slots(mesh, a))
        total += len(slots)
    return total


def written_refs(mesh: Mesh, kernel: KernelSpec):
    """Per-element distinct written (set, point) references as a namespaced
    CSR: ``(indptr, indices, set_offsets, total_points)`` -- each to-set's
    points offset by the sizes of the sets before it, in increment-argument
    order (plan.py:201-229).  The conflict relation every colouring and race
    check here is built on."""
    offsets, total, cols = {}, 0, []
    for a in kernel.increment_args:
        to = mesh.mappings[a.mapping].to_set
        if to.name not in offsets:
            offsets[to.name] = total
            total += to.size
    for a in kernel.increment_args:
        m = mesh.mappings[a.mapping]
        cols.append(m.table[:, list(kernel.arg_slots(mesh, a))] + offsets[m.to_set.name])
    n = mesh.sets[kernel.iter_set_name(mesh)].size
    rows = np.hstack(cols) if cols else np.empty((n, 0), dtype=np.int64)
    srt = np.sort(rows, axis=1)
    keep = np.ones_like(srt, dtype=bool)
    keep[:, 1:] = srt[:, 1:] != srt[:, :-1]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(keep.sum(axis=1), out=indptr[1:])
    return indptr, srt[keep].astype(np.int64), offsets, max(total, 1)


def build_global_plan(mesh: Mesh, kernel: KernelSpec, config: PlanConfig | None = None,
                      hw: HardwareDescriptor = B200) -> GlobalPlan:
    """Reorder, colour elements, range-split by colour (plan.py:408-448)."""
    from . import builder

    config = config or PlanConfig(strategy="global")
    if config.strategy != "global":
        config = replace(config, strategy="global")
    if config.reorder.startswith("structured"):
        raise MeshValidationError("structured blocks only apply to the hierarchical strategy")
    _check_valid(mesh, kernel)
    return builder.build_global(mesh, kernel, config, hw)


def build_hierarchical_plan(mesh: Mesh, kernel: KernelSpec, config: PlanConfig | None = None,
                            hw: HardwareDescriptor = B200) -> HierarchicalPlan:
    """Block, two-level colour, colour-sort and stage the loop (plan.py:467-579)."""
    from . import builder

    config = config or PlanConfig(strategy="hier")
    if config.strategy != "hier":
        config = replace(config, strategy="hier")
    _check_valid(mesh, kernel)
    compute_effective_block_size(config.partition_config())
    return builder.build_hier(mesh, kernel, config, hw)


# ------------------------------------------------------------------------------
# plan files (format of plan.py:619-755)
# ------------------------------------------------------------------------------


def mesh_fingerprint(mesh: Mesh) -> dict:
    return {
        "sets": {s.name: s.size for s in mesh.sets.values()},
        "mappings": {
            m.name: [m.from_set.name, m.to_set.name, m.arity, zlib.crc32(np.ascontiguousarray(m.table).tobytes())]
            for m in mesh.mappings.values()
        },
        "data": {a.name: [a.set.name, a.components, a.elem_type] for a in mesh.data.values()},
    }


def plan_to_dict(plan, as_lists: bool = True) -> dict:
    """The plan file content; arrays as lists (JSON) or numpy arrays (binary)."""
    c = plan.config
    L = (lambda a: np.asarray(a).tolist()) if as_lists else (lambda a: np.asarray(a))  # noqa: E731
    out = {
        "format": PLAN_HEADER,
        "strategy": c.strategy,
        "config": {k: getattr(c, k) for k in ("strategy", "reorder", "layout", "staging", "block_size", "tolerance",
                                               "epsilon", "seed", "unweighted_cut", "wide_transfers")},
        "hw": plan.hw.to_dict(),
        "kernel_key": plan.kernel_key,
        "set_perms": {n: L(p.forward) for n, p in plan.set_perms.items() if not p.is_identity()},
        "array_layouts": dict(plan.array_layouts),
    }
    if isinstance(plan, GlobalPlan):
        out["global"] = {"colours": L(plan.colours.colours), "num_colours": plan.colours.num_colours,
                         "colour_offsets": L(plan.colour_offsets)}
        return out

    def csr(d):
        return {k: {"indptr": L(v[0]), "ids": L(v[1])} for k, v in d.items()}

    out["hier"] = {
        "block_offsets": L(plan.block_offsets),
        "block_colours": L(plan.block_colours.colours),
        "num_block_colours": plan.block_colours.num_colours,
        "thread_colours": L(plan.thread_colours),
        "thread_colour_counts": L(plan.thread_colour_counts),
        "staged": csr(plan.staged),
        "written": csr(plan.written),
        "shared_bytes": L(plan.shared_bytes),
        "refs_per_element": plan.refs_per_element,
        "partition_meta": plan.partition_meta,
    }
    return out


# Binary plan files (extension): the same content as the
# JSON format with every array stored raw in an uncompressed .npz (C5 plans
# are ~1.5 GB as JSON text).  The header is the JSON dict with each array
# replaced by a reference into the archive.
_NPZ_REF = "__npz__"


def _to_binary(data: dict, arrays: dict, prefix: str = "") -> dict:
    out = {}
    for k, v in data.items():
        key = f"{prefix}{k}"
        if isinstance(v, dict):
            out[k] = _to_binary(v, arrays, key + "/")
        elif isinstance(v, np.ndarray):
            a = v.astype(np.int32) if v.dtype == np.int64 and (v.size == 0 or (v.min() >= -2**31 and v.max() < 2**31)) else v
            arrays[key] = np.ascontiguousarray(a)
            out[k] = {_NPZ_REF: key, "dtype": str(v.dtype)}
        else:
            out[k] = v
    return out


def _from_binary(data: dict, arrays) -> dict:
    out = {}
    for k, v in data.items():
        if isinstance(v, dict) and _NPZ_REF in v:
            out[k] = np.asarray(arrays[v[_NPZ_REF]]).astype(v["dtype"])
        elif isinstance(v, dict):
            out[k] = _from_binary(v, arrays)
        else:
            out[k] = v
    return out


def save_plan(plan, path, mesh: Mesh | None = None, binary: bool | None = None) -> None:
    """Write a plan file: the reference's JSON format (plan.py:619-755), or the
    binary .npz form when ``binary`` (default: the path ends with .npz)."""
    binary = str(path).endswith(".npz") if binary is None else binary
    data = plan_to_dict(plan, as_lists=not binary)
    if mesh is not None:
        data["mesh_fingerprint"] = mesh_fingerprint(mesh)
    if binary:
        arrays = {}
        header = _to_binary(data, arrays)
        arrays["__header__"] = np.frombuffer(json.dumps(header, sort_keys=True).encode(), dtype=np.uint8)
        with open(path, "wb") as fh:
            np.savez(fh, **arrays)
        return
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(data, fh, sort_keys=True, separators=(",", ":"))
        fh.write("\n")


def load_plan(path, mesh: Mesh):
    with open(path, "rb") as fh:
        magic = fh.read(2)
    if magic == b"PK":  # binary plan (.npz)
        try:
            with np.load(path, allow_pickle=False) as z:
                header = json.loads(bytes(z["__header__"]).decode())
                data = _from_binary(header, z)
        except (ValueError, KeyError, OSError) as exc:
            raise FileFormatError(f"{path}: bad binary plan: {exc}") from None
        return _plan_from_dict(data, mesh, path)
    with open(path, "r", encoding="utf-8") as fh:
        try:
            data = json.load(fh)
        except ValueError as exc:
            raise FileFormatError(f"{path}: bad plan JSON: {exc}") from None
    return _plan_from_dict(data, mesh, path)


def _plan_from_dict(data: dict, mesh: Mesh, path):
    if data.get("format") != PLAN_HEADER:
        raise FileFormatError(f"{path}: not a meshplan plan file")
    fp = data.get("mesh_fingerprint")
    if fp is not None and fp != mesh_fingerprint(mesh):
        raise MeshValidationError(f"{path}: plan was built for a different mesh")
    config = PlanConfig(**data["config"])
    hw = HardwareDescriptor.from_dict(data["hw"])
    perms = {name: Permutation.identity(s.size) for name, s in mesh.sets.items()}
    m2 = mesh
    for name, fwd in data["set_perms"].items():
        perms[name] = Permutation.from_forward(np.asarray(fwd, dtype=np.int64))
        m2 = apply_permutation(m2, name, perms[name])
    layouts = data["array_layouts"]
    m2 = m2.with_data(*[transform_layout(a, layouts.get(n, a.layout)) for n, a in m2.data.items()])
    i64 = lambda v: np.asarray(v, dtype=np.int64)  # noqa: E731
    if "global" in data:
        g = data["global"]
        col = i64(g["colours"])
        return GlobalPlan(m2, data["kernel_key"], config, hw, perms,
                          ColourAssignment(col, g["num_colours"], np.bincount(col, minlength=g["num_colours"])),
                          i64(g["colour_offsets"]), layouts)
    h = data["hier"]
    bc = i64(h["block_colours"])
    csr = lambda d: {k: (i64(v["indptr"]), i64(v["ids"])) for k, v in d.items()}  # noqa: E731
    return HierarchicalPlan(
        m2, data["kernel_key"], config, hw, perms, i64(h["block_offsets"]),
        ColourAssignment(bc, h["num_block_colours"], np.bincount(bc, minlength=h["num_block_colours"])),
        i64(h["thread_colours"]), i64(h["thread_colour_counts"]), csr(h["staged"]), csr(h["written"]),
        i64(h["shared_bytes"]), h["refs_per_element"], h["partition_meta"], layouts,
    )
