"""Blocking of the iteration set: configuration, chunking, structured blocks.

Names and the Eq. (1)-(2) arithmetic follow the reference
(pkg/src/meshplan/partition.py:98-170, 353-375).  The multilevel k-way
partitioner lives in :mod:`.kway`.
"""

import math
from dataclasses import dataclass, field

import numpy as np

from . import structured
from .errors import FileFormatError, MeshValidationError

PART_HEADER = "meshplan-part 1"


@dataclass(frozen=True)
class PartitionConfig:
    block_size: int = 128
    tolerance: float = 1.001
    epsilon: float = 0.5
    seed: int = 0
    unweighted_cut: bool = False

    def __post_init__(self):
        if self.block_size < 1:
            raise MeshValidationError("block size must be >= 1")
        if self.tolerance < 1.0:
            raise MeshValidationError("tolerance must be >= 1")
        if self.epsilon < 0.0:
            raise MeshValidationError("epsilon must be >= 0")


def compute_effective_block_size(cfg: PartitionConfig) -> tuple:
    """Eq. (1)-(2): S' = floor(S / l), l' = (S + eps) / S'."""
    eff = int(math.floor(cfg.block_size / cfg.tolerance))
    if eff < 1:
        raise MeshValidationError(
            f"unsatisfiable config: block size {cfg.block_size} with tolerance {cfg.tolerance} floors to zero"
        )
    return eff, (cfg.block_size + cfg.epsilon) / eff


@dataclass(frozen=True)
class Partition:
    assignment: np.ndarray
    num_blocks: int
    over_tolerance: bool = False
    cut: int | None = None
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        a = np.ascontiguousarray(self.assignment, dtype=np.int64)
        a.setflags(write=False)
        object.__setattr__(self, "assignment", a)
        if a.size and (a.min() < 0 or a.max() >= self.num_blocks):
            raise ValueError("block ids out of range")

    def block_sizes(self) -> np.ndarray:
        return np.bincount(self.assignment, minlength=self.num_blocks)

    def imbalance(self) -> float:
        n = self.assignment.size
        if n == 0 or self.num_blocks == 0:
            return 1.0
        return self.num_blocks * int(self.block_sizes().max()) / n


def chunk_partition(n: int, chunk: int) -> Partition:
    if chunk < 1:
        raise ValueError("chunk size must be >= 1")
    return Partition(np.arange(n, dtype=np.int64) // chunk, max(0, -(-n // chunk)))


def partition_structured_hex(dims, block_shape, target: str) -> Partition:
    if target not in ("cells-nodes", "faces-cells"):
        raise MeshValidationError(f"unknown structured target {target!r}")
    try:
        cell_block = structured.hex_block_assignment(dims, block_shape)
    except ValueError as exc:
        raise MeshValidationError(str(exc)) from None
    nb = int(np.prod([d // s for d, s in zip(dims, block_shape)]))
    meta = {"dims": tuple(dims), "block_shape": tuple(block_shape), "target": target}
    if target == "faces-cells":
        _, owners = structured.hex_internal_faces(dims)
        cell_block = cell_block[owners]
    return Partition(cell_block, nb, meta=meta)


def save_partition(part: Partition, path) -> None:
    with open(path, "w", encoding="ascii") as fh:
        fh.write(f"{PART_HEADER}\nblocks {part.num_blocks}\n")
        fh.write("".join(f"{int(b)}\n" for b in part.assignment))


def load_partition(path) -> Partition:
    with open(path, "r", encoding="ascii") as fh:
        lines = [t for t in (ln.strip() for ln in fh) if t]
    if not lines or lines[0] != PART_HEADER:
        raise FileFormatError(f"{path}: not a partition file")
    if len(lines) < 2 or not lines[1].startswith("blocks "):
        raise FileFormatError(f"{path}: missing blocks header")
    return Partition(np.array([int(v) for v in lines[2:]], dtype=np.int64), int(lines[1].split()[1]))


def __getattr__(name):
    # the reference keeps the k-way partitioner in this module (partition.py:28-350)
    if name in ("ThreadGraph", "build_thread_graph", "partition_kway"):
        from . import kway

        return getattr(kway, name)
    raise AttributeError(name)
