"""Small runs of the round-2 kernels for compute-sanitizer: GPU block
colouring, the gather-form executor (all families), the fused-export
streamed executor (one process, export rows into a local stand-in mailbox),
the peer put / get / signal kernels on one device."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1802_03749_b200 as mp  # noqa: E402
from paper_1802_03749_b200 import _native, gpuplan  # noqa: E402

# block colouring (random blocks, both choosers)
rng = np.random.default_rng(0)
lists = [sorted(set(rng.integers(max(0, b - 40), b + 40, size=12).tolist())) for b in range(3000)]
ptr = np.zeros(len(lists) + 1, dtype=np.int32)
ptr[1:] = np.cumsum([len(x) for x in lists])
ids = np.concatenate([np.asarray(x, dtype=np.int32) for x in lists])
for ll in (True, False):
    gpuplan.colour_blocks_device(torch.as_tensor(ptr, device="cuda"), torch.as_tensor(ids, device="cuda"), ll)

# gather form on every family
cases = [("quad2d", (40, 30), "flux", "all-indirect", "gps"), ("hex3d-nodes", (6, 5, 4), "scatter8", "all-indirect", "none"),
         ("hex3d-faces", (6, 5, 4), "face-flux", "increment-only", "none"), ("tri2d", (20, 16), "flux", "all-indirect", "gps"),
         ("quad2d", (48, 40), "flux", "all-indirect", "structured:8,8")]
for fam, dims, kname, staging, reorder in cases:
    mesh = mp.generate_mesh(fam, dims, dtype="f64")
    kernel = mp.kernel_for_mesh(kname, mesh)
    plan = mp.build_hierarchical_plan(mesh, kernel, mp.PlanConfig(reorder=reorder, staging=staging, block_size=32))
    lp = mp.bind(plan, kernel, schedule="gather")
    lp.run()
    lp.run()

# peer kernels on one device: put into a local "peer" mailbox, get back, signal
rows = torch.arange(0, 64, 2, dtype=torch.int32, device="cuda")
src = torch.rand(128 * 4, dtype=torch.float64, device="cuda")
dst = torch.zeros_like(src)
box = ctypes.c_void_p()
_native.call("mp_mailbox_alloc", 4096 + 256, ctypes.byref(box))
base = box.value
slot, flag, counter, epoch = base, base + 2048, base + 2048 + 64, base + 2048 + 128
_native.call("mp_epoch_bump", epoch, _native.stream_ptr())
_native.call("mp_halo_put", _native.MP_F64, src.data_ptr(), rows.data_ptr(), rows.numel(), 4, slot, rows.numel() * 4,
             flag, epoch, counter, _native.stream_ptr())
_native.call("mp_halo_get", _native.MP_F64, dst.data_ptr(), rows.data_ptr(), rows.numel(), 4, slot, rows.numel() * 4,
             flag, epoch, 1, _native.stream_ptr())
_native.call("mp_halo_signal", flag, epoch, _native.stream_ptr())
torch.cuda.synchronize()
assert torch.equal(dst.view(-1, 4)[rows.long()], src.view(-1, 4)[rows.long()])
_native.load().mp_free(ctypes.c_void_p(base))
print("sanitize r2 run ok")
