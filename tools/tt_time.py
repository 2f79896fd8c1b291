"""TT pair timing at a BASELINE config geometry (A/B of TT kernel variants):
python tools/tt_time.py [c2|c3|c4|c5] [views]  (library from CVPB_LIB if set)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_09841_b200 as cb
from tools.bench_configs import CFG

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 64
c = CFG[cfg]
det = cb.DetectorGeometry.make(c["R"], c["C"], c["px"], c["px"])
geom = cb.VolumeGeometry.make((c["n"],) * 3, (c["a"],) * 3)
views = cb.make_circular_trajectory(c["sid"], c["sdd"], nv, c["arc"], det)
sc = cb.DeviceScene(geom, det, views)
x = torch.rand(geom.shape(), device="cuda")
b = torch.rand((nv, c["R"], c["C"]), device="cuda")
p, v = sc.new_stack(), sc.new_volume()
for amp in (1, 0):
    o = cb.TTOptions(amplitude=amp)
    sc.project_tt(x, p, o); sc.backproject_tt(b, v, o)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); sc.project_tt(x, p, o); e[1].record(); sc.backproject_tt(b, v, o); e[2].record()
    torch.cuda.synchronize()
    w = geom.voxel_count() * nv / 1e9
    print(f"TT A{2 if amp else 1} {cfg} views={nv}: P {w / e[0].elapsed_time(e[1]) * 1e3:.1f} "
          f"BP {w / e[1].elapsed_time(e[2]) * 1e3:.1f} Gvox-view/s")
