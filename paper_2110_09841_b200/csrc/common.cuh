// Shared device-side definitions for the cvpb200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace cvpb {

// Per-view constants, precomputed on the host in float64 (the reference
// rebuilds the same numbers per call in ViewCtx::make, cvp.cpp:38-56, and
// DetectorPlane::of, siddon.cpp:138-147). Resident in device memory: 720 views
// x 256 B would not fit the 64 KB __constant__ bank.
struct ViewConst {
    // horizontal reduction of the camera (cvp.cpp:26-36)
    double sx, sy, s3;      // source
    double w1x, w1y;        // camera row 0, xy part (chi1 numerator)
    double w3x, w3y;        // camera row 2, xy part (depth)
    double pp1, pp2;        // principal point [px]
    double f_over_b2, b2_over_f;
    // full pinhole model for ray-driven projectors (siddon.cpp:135-150)
    double base[3], du[3], dv[3];
    double eu[3], ev[3], ew[3];
    double f, b1, b2;
    int scale_slot;         // index of this view's pixel-scale image
    int pad_;
};

// Launch-wide scene description.
struct Scene {
    int n1, n2, n3;         // volume counts
    double a1, a2, a3;      // voxel size [mm]
    double minx, miny, minz;  // min corner (= -extent/2, geometry.hpp:29)
    int rows, cols;         // detector
    double pw, ph;
};

// Backprojection fused with a reduce-scatter (cvpb_backproject_cvp_scatter):
// planes [plane_begin[t], plane_begin[t + 1]) of the volume go to slab[t]
// (element 0 = first voxel of plane plane_begin[t]) — stored (store = 1:
// each rank writes its own receive region, the owner sums them) or added with
// atomics; slab[t] may live in another GPU's memory (peer access).
constexpr int kMaxSlabTargets = 16;
struct SlabTargets {
    int n = 0;
    int plane_begin[kMaxSlabTargets + 1] = {};
    float* slab[kMaxSlabTargets] = {};
    int store = 0;  // 1: plain stores (the launch's result overwrites the regions)
};

// Error flags raised by kernels (checked by the host after the launch).
enum DeviceError : int {
    kDevOk = 0,
    kDevSourcePlane = 1,   // "voxel base reaches the source plane" (cvp.cpp:82-84)
    kDevDegenerate = 2,    // degenerate polygon centroid (polygon.hpp:94)
};

}  // namespace cvpb
