"""B200-native cone-beam projector pair (arXiv 2110.09841, "Cutting Voxel
Projector"): exact/relaxed CVP, its gather backprojector, Siddon-K and TT
footprint comparison projectors, and device-resident CGLS — hand-written
sm_100a kernels behind the C-ABI of include/cvpb200.h.

The Python API mirrors the reference's C++ operator API
(/root/reference/proj/include/cbct/*.hpp); see INTEGRATION.md.
"""
from ._native import (CvpbRuntimeError, DomainError, InvalidArgument, NoDevice, OutOfRange,
                      LIB_PATH)
from .geometry import (AttenuationVolume, DetectorGeometry, ProjectionStack, ViewGeometry,
                       VolumeGeometry, make_circular_trajectory, read_camera_matrices,
                       views_to_array, write_camera_matrices)
from .operators import (CutVolumeRecord, CvpOptions, CvpPrecision, DeviceScene, ExecPolicy, GroupScene,
                        PixelRoi, PixelScaling, RadiusEstimate, TTOptions, backproject_cvp,
                        backproject_cvp_into, backproject_siddon_k, backproject_siddon_k_into,
                        collect_cut_records, pixel_scale_cos, pixel_scale_exact, project_cvp,
                        project_cvp_into, project_siddon_k, project_siddon_k_into, scene_for)
from .solver import (CglsResult, LinearOperatorPair, SartResult, adjoint_test, cgls, cvp_pair,
                     extinction_from_intensity, fill_uniform01, os_sart, relative_projector_error,
                     siddon_pair, tt_pair)

__all__ = [n for n in dir() if not n.startswith("_")]
