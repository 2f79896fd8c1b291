/* ORACLE TEST INFRASTRUCTURE — not product code; parity pinned against
 * oracle/_ref (the reference compiled from /root/reference/proj/src) and the
 * committed golden vectors in tests/golden/.
 *
 * Plain-C restatement of the reference CPU algorithm for the hot path
 * (cbctproj: cvp.cpp, siddon.cpp, solver.cpp, geometry.cpp). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and
 * only as the checker / CPU baseline — never as the product path.
 *
 * Conventions (same as include/cvpb200.h):
 *   view  = 17 doubles: source[3], frame rows e_u,e_v,e_w [9], f, pp1, pp2, b1, b2
 *   volume index (k*N2 + j)*N1 + i          (geometry.hpp:34-36)
 *   stack  index v*R*C + m*C + n             (volume.hpp:23-46)
 *   opts  = {scaling(0 cos,1 exact), elevation(0/1), precision(0 double,1 single),
 *            r_estimate(0 voxel-center, 1 cut-centroid)}  (cvp.hpp:13-22)
 * Return codes: 0 ok, 1 invalid_argument, 2 runtime_error, 3 out_of_range,
 * 4 domain_error.
 */
#ifndef CVP_ORACLE_H
#define CVP_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

void orc_fill_uniform01(double* out, size_t n, uint64_t seed);

int orc_make_circular_trajectory(double sid, double sdd, int n_views, double arc_deg, int rows,
                                 int cols, double pw, double ph, double* out17);

int orc_pixel_scale(const double* view17, int rows, int cols, double pw, double ph, int exact,
                    int m, int n, double* out);

int orc_project_cvp(const int* counts, const double* voxel, int rows, int cols, double pw,
                    double ph, int n_views, const double* views17, const int* opts4,
                    const double* vol, double* out);

int orc_backproject_cvp(const int* counts, const double* voxel, int rows, int cols, double pw,
                        double ph, int n_views, const double* views17, const int* opts4,
                        const double* proj, double* out);

int orc_collect_cut_records(const int* counts, const double* voxel, const double* view17,
                            int rows, int cols, double pw, double ph, const int* opts4, int i,
                            int j, int k, int cap, int* rows_out, int* cols_out,
                            double* vol_out, double* invr2_out, int* n_out);

int orc_project_siddon(const int* counts, const double* voxel, int rows, int cols, double pw,
                       double ph, int n_views, const double* views17, int k_per_edge,
                       const int* roi4, const double* vol, double* out);

int orc_backproject_siddon(const int* counts, const double* voxel, int rows, int cols, double pw,
                           double ph, int n_views, const double* views17, int k_per_edge,
                           const double* proj, double* out);

/* SF-TT separable-footprint pair (tt_oracle.c; Long, Fessler & Balter 2010),
 * amplitude 0 = A1 (voxel-centre elevation), 1 = A2 (per detector row). */
int orc_project_tt(const int* counts, const double* voxel, int rows, int cols, int n_views,
                   const double* views17, int amplitude, const double* vol, double* out);
int orc_backproject_tt(const int* counts, const double* voxel, int rows, int cols, int n_views,
                       const double* views17, int amplitude, const double* proj, double* out);

/* Kahan-compensated dot (solver.cpp:15-24). */
double orc_dot_kahan(const double* a, const double* b, size_t n);

#ifdef __cplusplus
}
#endif
#endif
