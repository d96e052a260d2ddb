"""Synthetic meshes and the five registered indirect-increment loops.

Generators reproduce the reference families bit for bit
(reference: pkg/src/meshplan/bench_kernels.py:26-144): same table
enumeration, same ``np.random.default_rng(seed)`` draw order
(q, res=0, w, state, flux=0, facew for edge/face families; stress,
force=0 for hex nodes) and the same 1/1024-grid values.  ``arrays=`` limits
which arrays are materialised: arrays drawn before the last requested one
are still drawn (and dropped) so the RNG stream, and therefore every value,
is unchanged.  That keeps the 64M-edge and 8M-cell configs inside memory
(the full reference generator materialises an unused 28-component state).

Kernel specs carry a ``device_op``; the element arithmetic itself lives in
``csrc/mp_ops.cuh`` (device) and ``oracle/loops.py`` (the CPU checker, test-only).
"""

import numpy as np

from . import structured
from .errors import MeshValidationError
from .kernelspec import KernelArg, KernelSpec
from .mesh import ELEM_TYPES, DataArray, Mapping, Mesh, MeshSet

FAMILIES = ("quad2d", "tri2d", "hex3d-nodes", "hex3d-faces")
KERNEL_NAMES = ("flux", "flux-noread", "scatter8", "face-flux", "face-flux-heavy")

# (array, on_set, components, zero-initialised) in reference draw order
_EDGE_ARRAYS = (("q", "to", 4, False), ("res", "to", 4, True), ("w", "from", 2, False),
                ("state", "to", 28, False), ("flux", "to", 5, True), ("facew", "from", 4, False))
_NODE_ARRAYS = (("stress", "from", 4, False), ("force", "to", 3, True))


def _draw(rng, rows, comps, dt):
    if dt.kind == "i":
        return rng.integers(-9, 10, size=(rows, comps)).astype(dt)
    return (rng.integers(-1024, 1025, size=(rows, comps)) / 1024.0).astype(dt)


def _make_arrays(rng, spec, from_set, to_set, dt, arrays):
    wanted = set(spec_name for spec_name, *_ in spec) if arrays is None else set(arrays)
    last = max((i for i, s in enumerate(spec) if s[0] in wanted), default=-1)
    out = []
    for i, (name, where, comps, zero) in enumerate(spec[: last + 1]):
        s = to_set if where == "to" else from_set
        if zero:
            vals = np.zeros((s.size, comps), dtype=dt)
        else:
            vals = _draw(rng, s.size, comps, dt)  # always drawn: keeps the stream aligned
        if name in wanted:
            out.append(DataArray(name, s, comps, vals.reshape(-1), "aos"))
    return out


def _dt(dtype):
    if dtype not in ELEM_TYPES:
        raise MeshValidationError(f"unknown dtype {dtype!r}")
    return ELEM_TYPES[dtype]


def gen_quad2d(nx: int, ny: int, seed: int = 0, dtype: str = "f64", arrays=None) -> Mesh:
    """Quad grid, interior edges -> 2 cells; y-edges first, then x-edges."""
    if nx < 1 or ny < 1:
        raise MeshValidationError("dims must be >= 1")
    dt = _dt(dtype)
    cell = np.arange(nx * ny, dtype=np.int64).reshape(nx, ny)
    ylo = cell[:, :-1].reshape(-1)
    xlo = cell[:-1, :].reshape(-1)
    table = np.concatenate([np.stack([ylo, ylo + 1], 1), np.stack([xlo, xlo + ny], 1)]).reshape(-1, 2)
    edges, cells = MeshSet("edges", table.shape[0]), MeshSet("cells", nx * ny)
    data = _make_arrays(np.random.default_rng(seed), _EDGE_ARRAYS, edges, cells, dt, arrays)
    meta = {"family": "quad2d", "dims": f"{nx} {ny}", "seed": str(seed), "dtype": dtype}
    return Mesh.build([edges, cells], [Mapping("e2c", edges, cells, table)], data, meta)


def gen_tri2d(nx: int, ny: int, seed: int = 0, dtype: str = "f64", arrays=None) -> Mesh:
    """Each quad q splits into triangles 2q, 2q+1; diagonals, then y, then x edges."""
    if nx < 1 or ny < 1:
        raise MeshValidationError("dims must be >= 1")
    dt = _dt(dtype)
    quad = np.arange(nx * ny, dtype=np.int64).reshape(nx, ny)
    diag = quad.reshape(-1)
    yq = quad[:, :-1].reshape(-1)
    xq = quad[:-1, :].reshape(-1)
    table = np.concatenate([
        np.stack([2 * diag, 2 * diag + 1], 1),
        np.stack([2 * yq + 1, 2 * (yq + 1)], 1),
        np.stack([2 * xq + 1, 2 * (xq + ny)], 1),
    ]).reshape(-1, 2)
    edges, cells = MeshSet("edges", table.shape[0]), MeshSet("cells", 2 * nx * ny)
    data = _make_arrays(np.random.default_rng(seed), _EDGE_ARRAYS, edges, cells, dt, arrays)
    meta = {"family": "tri2d", "dims": f"{nx} {ny}", "seed": str(seed), "dtype": dtype}
    return Mesh.build([edges, cells], [Mapping("e2c", edges, cells, table)], data, meta)


def gen_hex3d(nx, ny, nz, target="nodes", seed=0, dtype="f64", arrays=None) -> Mesh:
    if nx < 1 or ny < 1 or nz < 1:
        raise MeshValidationError("dims must be >= 1")
    if target not in ("nodes", "faces"):
        raise MeshValidationError(f"unknown hex target {target!r}")
    dt = _dt(dtype)
    dims = (nx, ny, nz)
    rng = np.random.default_rng(seed)
    cells = MeshSet("cells", structured.cell_count(dims))
    meta = {"dims": f"{nx} {ny} {nz}", "seed": str(seed), "dtype": dtype}
    if target == "nodes":
        nodes = MeshSet("nodes", structured.node_count(dims))
        data = _make_arrays(rng, _NODE_ARRAYS, cells, nodes, dt, arrays)
        meta["family"] = "hex3d-nodes"
        return Mesh.build([cells, nodes], [Mapping("c2n", cells, nodes, structured.hex_cell_nodes(dims))], data, meta)
    table, _ = structured.hex_internal_faces(dims)
    faces = MeshSet("faces", table.shape[0])
    data = _make_arrays(rng, _EDGE_ARRAYS, faces, cells, dt, arrays)
    meta["family"] = "hex3d-faces"
    return Mesh.build([faces, cells], [Mapping("f2c", faces, cells, table)], data, meta)


def _dims(dims, k):
    d = tuple(int(v) for v in dims)
    if len(d) != k:
        raise MeshValidationError(f"expected {k} dims, got {d}")
    return d


def generate_mesh(family: str, dims, seed: int = 0, dtype: str = "f64", arrays=None) -> Mesh:
    if family == "quad2d":
        return gen_quad2d(*_dims(dims, 2), seed=seed, dtype=dtype, arrays=arrays)
    if family == "tri2d":
        return gen_tri2d(*_dims(dims, 2), seed=seed, dtype=dtype, arrays=arrays)
    if family in ("hex3d-nodes", "hex3d-faces"):
        return gen_hex3d(*_dims(dims, 3), target=family[6:], seed=seed, dtype=dtype, arrays=arrays)
    raise MeshValidationError(f"unknown mesh family {family!r}; expected one of {FAMILIES}")


def arrays_for_kernel(name: str) -> tuple:
    """Data arrays a named kernel touches (what ``arrays=`` needs)."""
    return {
        "flux": ("q", "res", "w"),
        "flux-noread": ("res", "w"),
        "scatter8": ("stress", "force"),
        "face-flux": ("state", "flux", "facew"),
        "face-flux-heavy": ("state", "flux", "facew"),
    }[name]


# --- kernel specs --------------------------------------------------------------


def kernel_flux_increment(dtype="f64", mapping="e2c", unit=False, no_indirect_read=False) -> KernelSpec:
    """Edge flux (bench_kernels.py:154-189): left=(q1-q0)*w0, right=-left."""
    _dt(dtype)
    name = "flux-noread" if no_indirect_read else "flux"
    args = [] if no_indirect_read else [KernelArg("q", "q", "read", mapping=mapping)]
    args += [KernelArg("w", "w", "read"), KernelArg("res", "res", "increment", mapping=mapping)]
    return KernelSpec(name, tuple(args), None, 48, name + (":unit" if unit else ""))


def kernel_scatter8(dtype="f64", mapping="c2n", unit=False) -> KernelSpec:
    """Cell -> 8 nodes (bench_kernels.py:192-207): [s0+s1, s1*s2, s3-s0] to every corner."""
    _dt(dtype)
    args = (KernelArg("stress", "stress", "read"), KernelArg("force", "force", "increment", mapping=mapping))
    return KernelSpec("scatter8", args, None, 96, "scatter8" + (":unit" if unit else ""))


def kernel_face_flux(dtype="f64", mapping="f2c", heavy=False, unit=False) -> KernelSpec:
    """Face flux (bench_kernels.py:210-246): phi=(sr[:5]-sl[:5])*fw0 (heavy: sqrt scaling)."""
    dt = _dt(dtype)
    if heavy and dt.kind != "f":
        raise MeshValidationError("heavy face flux needs float data")
    name = "face-flux-heavy" if heavy else "face-flux"
    args = (
        KernelArg("state", "state", "read", mapping=mapping),
        KernelArg("facew", "facew", "read"),
        KernelArg("flux", "flux", "increment", mapping=mapping),
    )
    return KernelSpec(name, args, None, 165, name + (":unit" if unit else ""))


def kernel_for_mesh(name: str, mesh: Mesh, unit: bool = False) -> KernelSpec:
    """Bind a registered kernel to a generated single-mapping mesh."""
    if len(mesh.mappings) != 1:
        raise MeshValidationError("bench kernels expect a single-mapping mesh")
    m = next(iter(mesh.mappings.values()))

    def elem_type(array):
        arr = mesh.data.get(array)
        if arr is None:
            raise MeshValidationError(f"kernel {name!r} needs data array {array!r}, mesh has {sorted(mesh.data)}")
        return arr.elem_type

    if name in ("flux", "flux-noread"):
        if m.arity != 2:
            raise MeshValidationError(f"kernel {name!r} needs an arity-2 mapping")
        return kernel_flux_increment(elem_type("res"), m.name, unit, name == "flux-noread")
    if name == "scatter8":
        if m.arity != 8:
            raise MeshValidationError("kernel 'scatter8' needs an arity-8 mapping")
        return kernel_scatter8(elem_type("force"), m.name, unit)
    if name in ("face-flux", "face-flux-heavy"):
        if m.arity != 2:
            raise MeshValidationError(f"kernel {name!r} needs an arity-2 mapping")
        return kernel_face_flux(elem_type("flux"), m.name, name == "face-flux-heavy", unit)
    raise MeshValidationError(f"unknown kernel {name!r}; expected one of {KERNEL_NAMES}")


def kernels_for_family(family: str) -> tuple:
    return ("scatter8",) if family == "hex3d-nodes" else ("flux", "face-flux")


# --- counter-based synthetic values (benchmark-scale meshes) --------------------------


def hashed_grid_values(index, seed: int, salt: int):
    """Values on the 1/1024 grid in [-1, 1] from a 32-bit integer hash of
    (index, seed, salt).  Any row of any array can be produced independently
    (on the GPU, on any rank of a decomposition) -- unlike the reference's
    sequential RNG stream, which takes ~30 s to draw at 64M edges.  ``index``
    is an int64 torch tensor or numpy array; returns float64 of its shape."""
    mask = 0xFFFFFFFF
    x = (index * 1664525 + (seed * 1013904223 + salt * 40503 + 12345)) & mask
    for _ in range(2):
        x = x ^ (x >> 16)
        x = (x * 0x45D9F3B) & mask
    x = x ^ (x >> 16)
    v = (x % 2049) - 1024
    v = v.to(__import__("torch").float64) if hasattr(v, "to") else v.astype(np.float64)
    return v / 1024.0


def quad2d_table(nx: int, ny: int, xlo: int = 0, xhi: int | None = None):
    """Edges of gen_quad2d restricted to owner cells with x in [xlo, xhi)
    (owner = first cell), in global enumeration order, plus their global
    edge ids.  With the full range this is exactly gen_quad2d's table."""
    xhi = nx if xhi is None else xhi
    x = np.arange(xlo, xhi, dtype=np.int64)
    y = np.arange(ny - 1, dtype=np.int64)
    ylo = (x[:, None] * ny + y[None, :]).reshape(-1)
    y_ids = (x[:, None] * (ny - 1) + y[None, :]).reshape(-1)
    xs = x[x < nx - 1]
    xlo_c = (xs[:, None] * ny + np.arange(ny, dtype=np.int64)[None, :]).reshape(-1)
    x_ids = nx * (ny - 1) + xlo_c
    table = np.concatenate([np.stack([ylo, ylo + 1], 1), np.stack([xlo_c, xlo_c + ny], 1)]).reshape(-1, 2)
    return table, np.concatenate([y_ids, x_ids])
