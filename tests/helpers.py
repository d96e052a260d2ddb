"""Test helpers: rebuild reference plans (from golden arrays) as package objects."""

import numpy as np

import paper_1802_03749_b200 as mp
from paper_1802_03749_b200.colouring import ColourAssignment
from paper_1802_03749_b200.mesh import apply_permutation, transform_layout


def config_of(rec):
    return mp.PlanConfig(strategy=rec["strategy"], reorder=rec["reorder"], layout=rec["layout"],
                         staging=rec["staging"], block_size=rec["block_size"])


def layouts_of(mesh, kernel, layout):
    ind = {a.array for a in kernel.indirect_args}
    direct = {a.array for a in kernel.direct_args}
    return {n: (layout if n in ind else ("soa" if n in direct else a.layout)) for n, a in mesh.data.items()}


def reference_plan(rec, z, mesh, kernel):
    """The reference's plan for this case as a package plan object (no device state)."""
    m = next(iter(mesh.mappings.values()))
    perms = {m.from_set.name: mp.Permutation.from_forward(z["elem_fwd"]),
             m.to_set.name: mp.Permutation.from_forward(z["point_fwd"])}
    pm = mesh
    for name, p in perms.items():
        pm = apply_permutation(pm, name, p)
    lay = layouts_of(mesh, kernel, rec["layout"])
    pm = pm.with_data(*[transform_layout(a, lay[n]) for n, a in pm.data.items()])
    cfg = config_of(rec)
    if rec["strategy"] == "global":
        col = z["colours"]
        return mp.GlobalPlan(pm, kernel.signature_key(), cfg, mp.B200, perms, ColourAssignment.from_colours(col),
                             z["colour_offsets"], lay)
    bc = z["block_colours"]
    return mp.HierarchicalPlan(
        pm, kernel.signature_key(), cfg, mp.B200, perms, z["block_offsets"],
        ColourAssignment(bc, rec["num_block_colours"], np.bincount(bc, minlength=rec["num_block_colours"])),
        z["thread_colours"], z["thread_colour_counts"], {m.to_set.name: (z["staged_ptr"], z["staged_ids"])},
        {m.to_set.name: (z["written_ptr"], z["written_ids"])}, z["shared_bytes"], rec["refs_per_element"],
        rec.get("partition_meta", {}), lay,
    )
