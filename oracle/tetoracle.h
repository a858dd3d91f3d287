/*
 * tetoracle.h -- CPU restatement of the reference traversal (TEST
 * INFRASTRUCTURE ONLY).
 *
 * This is the parity oracle for the sm_100a kernels in
 * paper_2103_02309_b200/csrc.  It is imported only by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg, as the checker --
 * never by the product path.  Parity pinning: checked against the golden
 * vectors generated from the reference itself (tests/golden/, made by
 * tests/golden/make_golden.py) and against the reference's compiled kernels
 * built by oracle/build_ref.sh (oracle/_ref/).
 *
 * Every function cites the reference file:line it restates.  Floating point
 * follows the reference's expression order; build with -ffp-contract=off
 * (the reference's own flag, pkg/setup.py:17-20).
 */
#ifndef TETORACLE_H
#define TETORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int layout;               /* 32, 20, 16 (CompactMesh.layout) or 80 */
  int64_t n_points;
  int64_t n_tets;
  const float* pts;         /* (p, 3) */
  const uint32_t* recs;     /* (t, layout/4) = records_u32(); tet80: to_build_tet80 output */
  const int32_t* sv;        /* (t, 4) side_verts */
  const uint32_t* sn;       /* (t, 4) side_neighbors */
  const int32_t* cf_tri;    /* (c,) */
  const int32_t* cf_tets;   /* (c, 2) */
  const double* tri;        /* (n_tri, 3, 3) */
} to_mesh;

/* _kernels.pyx:271-370 + batch.py:57-71 (triangle/t/tet_back may be NULL). */
int to_cast_rays(const to_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start,
                 uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle,
                 double* t, int32_t* tet_back, int n_threads);
/* visits_sink path, _kernels.pyx:307-341: CSR by offsets (exclusive scan of visited). */
int to_cast_rays_visits(const to_mesh* m, int64_t n, const float* o, const float* d,
                        const int32_t* start, const int64_t* offsets, int32_t* seq);
/* _kernels.pyx:416-492 */
int to_locate_points(const to_mesh* m, int64_t n, const double* q, const int32_t* hints, int32_t* tet,
                     int32_t* visited, int n_threads);
/* _kernels.pyx:527-614 */
int to_shadow_rays(const to_mesh* m, int64_t n, const double* p, const double* light, int light_stride,
                   const int32_t* p_tet, const int32_t* light_tet, int light_tet_stride, double eps,
                   uint8_t* occluded, int32_t* visited, int n_threads);
/* ScTP walk around traversal.sctp_exit_face (traversal.py:484-511). */
int to_sctp_cast_rays(const to_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start,
                      uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle,
                      double* t, int32_t* tet_back, int n_threads);
/* Single-tet ScTP predicate on arbitrary fp64 vertices (for the reference's
 * own sctp_exit_face golden cases). */
int to_sctp_exit_face(const double* verts12, const double* o3, const double* d3, int entry);
/* TetMesh-80 records from the side tables: 20 u32 per tet. */
void to_build_tet80(const int32_t* sv, const uint32_t* sn, const float* pts, int64_t n_tets,
                    uint32_t* out);
/* fp64 ray/triangle t, _kernels_py._mt_t (_kernels_py.py:435-454). */
double to_mt_t(const double* o, const double* d, const double* tri9);

#ifdef __cplusplus
}
#endif

#endif
