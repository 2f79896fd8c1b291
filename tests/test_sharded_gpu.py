"""SURVEY §8e single-GPU check of the multi-GPU decomposition: shard the views
G ways on one device exactly as G ranks would (parallel.view_shard), project
each shard, backproject each shard into its own partial volume, and sum the
partials in a fixed order. The result must equal the one-launch result within
float32 reassociation (1e-6), and the z-slabs a reduce-scatter would hand out
are the contiguous k-ranges of that sum."""
import numpy as np
import pytest

from conftest import make_case, rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G", [2, 4, 8])
def test_view_shards_sum_to_the_full_launch(G):
    import torch
    import paper_2110_09841_b200 as cb
    from paper_2110_09841_b200.parallel import slab_elems, view_shard
    geom, det, views, _ = make_case((64, 64, 64), (0.72, 0.72, 0.72), 480, 616, 0.154, 0.154,
                                    749.0, 1198.0, 64)
    scene = cb.DeviceScene(geom, det, views)
    x = torch.from_numpy(cb.fill_uniform01(geom.voxel_count(), 7).astype(np.float32)).reshape(
        geom.shape()).cuda()
    b = torch.from_numpy(cb.fill_uniform01(det.pixel_count() * 64, 8).astype(np.float32)).reshape(
        64, det.rows, det.cols).cuda()
    p_full = scene.project_cvp(x)
    bp_full = scene.backproject_cvp(b)
    parts, total = [], torch.zeros_like(bp_full)
    for r in range(G):
        vb, vc = view_shard(64, G, r)
        parts.append(scene.project_cvp(x, view_begin=vb, view_count=vc))
        total += scene.backproject_cvp(b[vb:vb + vc].contiguous(), view_begin=vb, view_count=vc)
    p_cat = torch.cat(parts)
    assert rel_l2(p_cat.cpu().numpy(), p_full.cpu().numpy()) < 1e-6
    assert rel_l2(total.cpu().numpy(), bp_full.cpu().numpy()) < 1e-6
    n = slab_elems(geom.voxel_count(), G)
    flat = total.reshape(-1)
    for r in range(G):
        slab = flat[r * n:(r + 1) * n].reshape(-1, 64, 64)
        assert slab.shape[0] == 64 // G  # z-slabs: contiguous k ranges
