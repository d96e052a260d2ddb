"""Multi-GPU owner-compute decomposition.

* CPU, world_size 2 over gloo: the exchange protocol end to end with real
  torch.distributed transports; the local loop is the oracle and pack /
  unpack are torch ops (test-only stand-ins for the device kernels).
* GPU, N ranks simulated in threads on one device: the full device path
  (local GPU plans, sm_100a executors, halo kernels) against the oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch

from paper_1802_03749_b200 import decomp, workloads
from oracle import loops


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torch_pack(src, rows, comps, out):
    out.copy_(src.reshape(-1, comps)[rows.long()].reshape(-1))


def _torch_unpack(dst, rows, comps, src, mode):
    v = dst.view(-1, comps)
    if mode == decomp.ZERO:
        v[rows.long()] = 0
    elif mode == decomp.ADD:
        v[rows.long()] += src.view(-1, comps)
    else:
        v[rows.long()] = src.view(-1, comps)


def _global_case(nx=12, ny=10):
    mesh = workloads.gen_quad2d(nx, ny, seed=5, dtype="f64")
    m = mesh.mappings["e2c"]
    q = mesh.data["q"].view2d()
    w = np.ascontiguousarray(mesh.data["w"].view2d())
    want = loops.serial_loop("flux", m.table, q, w, np.zeros((m.to_set.size, 4)))
    return mesh, want


def _rank_main(rank, world, port, result_file):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    decomp.pack_rows, decomp.unpack_rows = _torch_pack, _torch_unpack
    nx, ny = 12, 10
    mesh, want = _global_case(nx, ny)
    q = mesh.data["q"].view2d()
    w = np.ascontiguousarray(mesh.data["w"].view2d())
    bounds, xs = decomp.slab_bounds(nx, ny, world)
    table, gids = workloads.quad2d_table(nx, ny, int(xs[rank]), int(xs[rank + 1]))

    def allgather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    dec = decomp.decompose(table, gids, bounds, rank, world, allgather)
    assert np.array_equal(mesh.mappings["e2c"].table[gids], table)
    qt = torch.zeros(dec.n_local * 4, dtype=torch.float64)
    qt.view(-1, 4)[: dec.n_owned] = torch.as_tensor(q[dec.lo:dec.hi])  # halo q arrives by exchange
    res = torch.zeros(dec.n_local * 4, dtype=torch.float64)
    hx = decomp.HaloExchange(dec, decomp.TorchDistTransport(), "cpu")
    for _ in range(2):  # two steps: halo rows must be re-zeroed in between
        hx.import_rows(qt, 4)
        assert np.array_equal(qt.view(-1, 4).numpy(), q[dec.local_points])
        res.view(-1, 4)[:] = torch.as_tensor(
            loops.serial_loop("flux", dec.local_table, qt.view(-1, 4).numpy(), w[dec.elem_ids],
                              res.view(-1, 4).numpy()))
        hx.export_increments(res, 4)
        assert not res.view(-1, 4)[dec.n_owned:].any()
    owned = res.view(-1, 4)[: dec.n_owned].numpy()
    parts = [None] * world
    dist.all_gather_object(parts, (dec.lo, owned))
    if rank == 0:
        full = np.zeros_like(want)
        for lo, block in parts:
            full[lo: lo + block.shape[0]] = block
        np.save(result_file, full)
    dist.destroy_process_group()


def test_gloo_two_ranks_exchange_matches_serial(tmp_path):
    import torch.multiprocessing as tmp

    out = str(tmp_path / "full.npy")
    tmp.spawn(_rank_main, args=(2, _free_port(), out), nprocs=2, join=True)
    _, want = _global_case()
    assert np.array_equal(np.load(out), 2 * want)


def test_decompose_lists_consistent():
    nx, ny, world = 9, 7, 3
    bounds, xs = decomp.slab_bounds(nx, ny, world)
    tables = [workloads.quad2d_table(nx, ny, int(xs[r]), int(xs[r + 1])) for r in range(world)]
    halos = []
    for t, _ in tables:
        pts = np.unique(t)
        halos.append(pts[(pts < bounds[0]) | (pts >= bounds[1])])  # placeholder, recomputed below

    def make_allgather():
        store = {}

        def run(rank):
            t, g = tables[rank]
            pts = np.unique(t)
            lo, hi = bounds[rank], bounds[rank + 1]
            store[rank] = pts[(pts < lo) | (pts >= hi)]
        for r in range(world):
            run(r)
        return lambda obj: [store[r] for r in range(world)]

    ag = make_allgather()
    decs = [decomp.decompose(tables[r][0], tables[r][1], bounds, r, world, ag) for r in range(world)]
    full = workloads.quad2d_table(nx, ny)[0]
    assert sum(d.elem_ids.size for d in decs) == full.shape[0]
    for d in decs:
        assert np.array_equal(d.local_points[d.local_table], full[d.elem_ids])
        for peer, rows in d.halo_rows.items():
            other = decs[peer]
            assert np.array_equal(d.local_points[rows], other.local_points[other.export_rows[d.rank]])


@pytest.mark.gpu
@pytest.mark.parametrize("world,reorder,schedule,overlap", [
    (2, "gps", "dataflow", False), (3, "none", "dataflow", False), (4, "gps", "stream", False),
    (2, "none", "stream-pull", False), (4, "gps", "stream", True), (2, "none", "stream-pull", True),
    (3, "gps", "colour", True), (2, "gps", "pipelined", True)])
def test_threaded_ranks_on_one_gpu_match_serial(world, reorder, schedule, overlap):
    """Decomposed steps (halo import, local loop, increment export) equal the
    serial loop; with ``overlap`` the core blocks (no halo point) run while the
    import is in flight and the boundary blocks after it."""
    import threading

    import paper_1802_03749_b200 as mp

    nx, ny = 64, 48
    mesh, _ = _global_case(nx, ny)
    m = mesh.mappings["e2c"]
    q = mesh.data["q"].view2d()
    w = np.ascontiguousarray(mesh.data["w"].view2d())
    want = loops.serial_loop("flux", m.table, q, w, np.zeros((m.to_set.size, 4)))
    bounds, xs = decomp.slab_bounds(nx, ny, world)
    tables = [workloads.quad2d_table(nx, ny, int(xs[r]), int(xs[r + 1])) for r in range(world)]
    halos = []
    for r, (t, _) in enumerate(tables):
        pts = np.unique(t)
        halos.append(pts[(pts < bounds[r]) | (pts >= bounds[r + 1])])
    hub = decomp.ThreadHub()
    out, errors = {}, []

    def rank_main(r):
        torch.cuda.set_device(0)
        # each simulated rank on its own stream (separate processes each have
        # their own default stream; threads would share the legacy one)
        with torch.cuda.stream(torch.cuda.Stream()):
            rank_body(r)

    def rank_body(r):
        try:
            t, g = tables[r]
            dec = decomp.decompose(t, g, bounds, r, world, lambda obj: halos)
            res0 = np.zeros((dec.n_local, 4))
            local = decomp.local_flux_mesh(t, g, dec, q[dec.local_points], w[g], res0)
            kernel = mp.kernel_for_mesh("flux", local)
            dl = decomp.DistributedLoop(local, kernel, dec, decomp.ThreadTransport(hub, r),
                                        mp.PlanConfig(reorder=reorder, block_size=64), schedule, overlap=overlap)
            if overlap:
                core = dl.core_blocks().cpu().numpy()
                dp = dl.plan._device
                halo = np.zeros(dec.n_local, dtype=bool)
                for rows in dl.dec.halo_rows.values():
                    halo[rows] = True
                bo = dp.block_offsets.cpu().numpy()
                tab = dp.map.cpu().numpy()
                for b in range(len(bo) - 1):
                    assert core[b] == (not halo[tab[bo[b]:bo[b + 1]]].any())
                assert dl.core.num_blocks + dl.boundary.num_blocks == dl.plan.num_blocks
                assert (dl.boundary.num_blocks > 0) == bool(halo.any())  # the last slab imports nothing
            for _ in range(3):
                dl.step()
            torch.cuda.synchronize()
            out[r] = (dec.lo, dl.owned_result())
        except Exception as exc:  # pragma: no cover - surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=300)
    assert not errors, errors
    full = np.zeros_like(want)
    for lo, block in out.values():
        full[lo: lo + block.shape[0]] = block
    assert np.array_equal(full, 3 * want)


# ---- peer-memory exchange (device-side puts / waits, graph-capturable) ------------------


def _peer_rank(r, world, nx, ny, reorder, schedule, overlap, publish, steps, graph, barrier=lambda: None,
               capture_lock=None, fused=None):
    """One rank's share with the peer-memory exchange; returns (lo, owned rows).
    ``barrier`` separates setup from stepping: ranks sharing one device must
    not synchronise the whole device (plan building does) while a peer's
    exchange kernel waits for them."""
    import paper_1802_03749_b200 as mp

    mesh, _ = _global_case(nx, ny)
    q = mesh.data["q"].view2d()
    w = np.ascontiguousarray(mesh.data["w"].view2d())
    bounds, xs = decomp.slab_bounds(nx, ny, world)
    tables = [workloads.quad2d_table(nx, ny, int(xs[k]), int(xs[k + 1])) for k in range(world)]
    halos = []
    for k, (t, _) in enumerate(tables):
        pts = np.unique(t)
        halos.append(pts[(pts < bounds[k]) | (pts >= bounds[k + 1])])
    t, g = tables[r]
    dec = decomp.decompose(t, g, bounds, r, world, lambda obj: halos)
    local = decomp.local_flux_mesh(t, g, dec, q[dec.local_points], w[g], np.zeros((dec.n_local, 4)))
    kernel = mp.kernel_for_mesh("flux", local)
    dl = decomp.DistributedLoop(local, kernel, dec, publish, mp.PlanConfig(reorder=reorder, block_size=64),
                                schedule, overlap=overlap, fused_export=fused)
    assert dl.peer
    assert dl.fused == (schedule in ("stream", "stream-pull") if fused is None else fused)
    barrier()
    if graph:
        dl.warmup_step()
        barrier()
        if capture_lock is not None:  # threads of one process capture one at a time
            with capture_lock:
                gr = dl.capture(warmup=False)
        else:
            gr = dl.capture(warmup=False)
        barrier()
        for _ in range(steps):
            gr.replay()
    else:
        for _ in range(steps):
            dl.step()
    torch.cuda.current_stream().synchronize()
    barrier()
    res = (dec.lo, dl.owned_result())
    return res, dl


def _ipc_rank_main(rank, world, port, result_file, case):
    """One rank as its own process (gloo rendezvous, mailboxes through CUDA
    IPC).  Ranks sharing one device must be processes: threads of one
    process share its hardware work queues, so one rank's waiting exchange
    kernel can stall another rank's queued put (a cross-rank deadlock that
    separate GPUs, or separate processes time-slicing one GPU, never see)."""
    import torch.distributed as dist

    nx, ny, reorder, schedule, overlap, graph, fused, steps = case
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)

    def allgather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    (lo, owned), dl = _peer_rank(rank, world, nx, ny, reorder, schedule, overlap, decomp.ipc_connector(allgather),
                                 steps, graph=graph, barrier=dist.barrier, fused=fused)
    parts = [None] * world
    dist.all_gather_object(parts, (lo, owned))
    dist.barrier()
    dl.halo.close()
    if rank == 0:
        _, want = _global_case(nx, ny)
        full = np.zeros_like(want)
        for lo_, block in parts:
            full[lo_: lo_ + block.shape[0]] = block
        np.save(result_file, np.stack([full, steps * want]))
    dist.destroy_process_group()


PEER_CASES = [  # world, reorder, schedule, overlap, graph, fused (None: the default, fused under stream schedules)
    (2, "gps", "stream", False, False, None), (3, "none", "stream", True, False, None),
    (4, "gps", "stream", True, True, None), (3, "gps", "stream", True, True, False),
    (2, "none", "colour", True, True, None), (3, "gps", "pipelined", False, True, None),
    (2, "gps", "stream-pull", True, True, None), (2, "none", "stream-pull", False, False, None)]


@pytest.mark.gpu
@pytest.mark.parametrize("world,reorder,schedule,overlap,graph,fused", PEER_CASES)
def test_peer_exchange_processes_on_one_gpu_match_serial(world, reorder, schedule, overlap, graph, fused, tmp_path):
    """N processes (gloo rendezvous only) on one device exchanging through
    each other's IPC-mapped mailboxes: direct steps and CUDA-graph replays of
    a whole step equal the serial loop; under the streamed colour schedules
    the increment export is fused into the loop's write-back (the halo rows'
    last writers store them into the owners' mailboxes)."""
    import torch.multiprocessing as tmp

    out = str(tmp_path / "full.npy")
    case = (32, 24, reorder, schedule, overlap, graph, fused, 3)
    tmp.spawn(_ipc_rank_main, args=(world, _free_port(), out, case), nprocs=world, join=True)
    got, want = np.load(out)
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_peer_exchange_two_processes_larger_mesh(tmp_path):
    """The bench's configuration in miniature: two processes, GPS plans, the
    core/boundary overlap, the fused export, graph-replayed steps."""
    import torch.multiprocessing as tmp

    out = str(tmp_path / "full.npy")
    case = (96, 80, "gps", "stream", True, True, None, 2)
    tmp.spawn(_ipc_rank_main, args=(2, _free_port(), out, case), nprocs=2, join=True)
    got, want = np.load(out)
    assert np.array_equal(got, want)
