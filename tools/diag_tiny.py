"""Diagnostic: forward projection through the fixed-point tile vs the
float-atomic fallback (a 1e-30-scaled volume overflows the tile scale) against
the reference, same 32^3 scene as tests/test_config_parity_gpu.py."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_09841_b200 as cb
from oracle.pyoracle import Reference, Scene

det = cb.DetectorGeometry.make(48, 48, 1.0, 1.0)
geom = cb.VolumeGeometry.make((32, 32, 32), (1.0, 1.0, 1.0))
views = cb.make_circular_trajectory(60.0, 100.0, 6, 360.0, det)
scene = cb.DeviceScene(geom, det, views)
x64 = cb.fill_uniform01(geom.voxel_count(), 5).astype(np.float32)
x = torch.from_numpy(x64).reshape(geom.shape()).cuda()
ref = Reference().project_cvp(Scene((32,) * 3, (1.0,) * 3, 48, 48, 1.0, 1.0, cb.views_to_array(views)),
                              x64.astype(np.float64))
for name, scale in (("tile", 1.0), ("fallback", 1e-30), ("mid", 1e-20)):
    p = scene.project_cvp(x * scale).double().cpu().numpy() / scale
    d = p - ref
    print(name, "rel-L2", np.linalg.norm(d) / np.linalg.norm(ref), "max", np.abs(d).max() / np.abs(ref).max())

# the global path at unit scale (CVPB_NO_TILE is read per launch)
os.environ["CVPB_NO_TILE"] = "1"
for name, scale in (("no-tile P", 1.0),):
    p = scene.project_cvp(x * scale).double().cpu().numpy() / scale
    d = p - ref
    print(name, "rel-L2", np.linalg.norm(d) / np.linalg.norm(ref), "max", np.abs(d).max() / np.abs(ref).max())
b64 = cb.fill_uniform01(det.pixel_count() * 6, 8).astype(np.float32)
bref = Reference().backproject_cvp(Scene((32,) * 3, (1.0,) * 3, 48, 48, 1.0, 1.0, cb.views_to_array(views)),
                                   b64.astype(np.float64))
bd = scene.backproject_cvp(torch.from_numpy(b64).reshape(6, 48, 48).cuda()).double().cpu().numpy()
print("no-tile BP rel-L2", np.linalg.norm(bd.ravel() - bref.ravel()) / np.linalg.norm(bref))
os.environ["CVPB_NO_TILE"] = "0"
bd = scene.backproject_cvp(torch.from_numpy(b64).reshape(6, 48, 48).cuda()).double().cpu().numpy()
print("tile BP rel-L2", np.linalg.norm(bd.ravel() - bref.ravel()) / np.linalg.norm(bref))
