/*
 * tetb200.h -- C ABI of the B200-native tetrahedral-mesh ray traversal engine.
 *
 * This is the drop-in boundary for the reference package's "kernel module"
 * protocol (BACKEND_NAME / cast_rays / locate_points / shadow_rays,
 * /root/reference/pkg/src/tetray/_kernels.pyx:15,271,416,527, selected by
 * backend.get_kernels, backend.py:35-45, and passed as `kernels=` by every
 * batch entry point, batch.py:45,84,140,152).  Plain pointers and sizes only:
 * no torch or numpy types cross this boundary.
 *
 * Pointer conventions
 *   - tb_mesh_create / tb_mesh_create_tet80: HOST pointers (the mesh is copied
 *     into HBM once and is immutable afterwards).
 *   - tb_cast_rays, tb_cast_rays_visits, tb_locate_points, tb_shadow_rays,
 *     tb_sctp_cast_rays: DEVICE pointers on the mesh's device, enqueued on
 *     `stream` (a cudaStream_t; NULL = legacy default stream).  Nothing is
 *     synchronised; the caller owns ordering.
 *   - *_host variants: HOST pointers (pageable or pinned); the call stages
 *     the inputs to HBM, launches, copies the outputs back and synchronises.
 *
 * Errors: every function returns 0 on success and a negative TB_E* code on
 * failure; tb_last_error() returns a thread-local message for the last
 * failure on the calling thread.  Per-ray problems are not errors: they are
 * reported through the per-ray status (TB_STATUS_ERROR = the reference's
 * cycle guard, _kernels.pyx:365-368).
 *
 * Thread safety: a tb_mesh is immutable after creation; concurrent calls on
 * the same mesh from several host threads are allowed (the reference's tile
 * pool calls cast_rays concurrently, render.py:538-541).
 */
#ifndef TETB200_H
#define TETB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TB_ABI_VERSION 1

/* Record layouts (tetmesh.py:34-46); 80 = TetMesh-80 (4 ids + 4 refs + 4
 * inline float3 vertices, no separate point fetch; not in the reference). */
#define TB_LAYOUT_TET32 32
#define TB_LAYOUT_TET20 20
#define TB_LAYOUT_TET16 16
#define TB_LAYOUT_TET80 80

/* Per-ray status codes (_kernels.pyx:17-19). */
#define TB_STATUS_MISS 0
#define TB_STATUS_HIT 1
#define TB_STATUS_ERROR 2

/* Neighbour-reference encoding (tetmesh.py:29-32). */
#define TB_CONSTRAINED_BIT 0x80000000u
#define TB_PAYLOAD_MASK 0x7FFFFFFFu
#define TB_BOUNDARY_REF 0x7FFFFFFFu

/* Error codes. */
#define TB_OK 0
#define TB_E_ARG -1
#define TB_E_CUDA -2
#define TB_E_OOM -3
#define TB_E_LAYOUT -4

typedef struct tb_mesh tb_mesh;

/* Upload a CompactMesh (tetmesh.py:147-195) to HBM on `device`.
 * Replaces: the arrays _kernels.cast_rays reads per call
 *   (_kernels.pyx:276-282: mesh.points, records_u32(), side_verts,
 *   side_neighbors) plus what batch.cast_rays' epilogue reads
 *   (batch.py:63-71: cf_triangle, cf_tets, triangle_coords()).
 *   points_xyz      (n_points, 3) float32
 *   records         (n_tets, layout/4) uint32 = CompactMesh.records_u32()
 *   side_verts      (n_tets, 4) int32, ascending per row
 *   side_neighbors  (n_tets, 4) uint32, sorted-slot references
 *   cf_triangle     (n_cf,) int32      scene triangle per constrained face
 *   cf_tets         (n_cf, 2) int32    [front, back], back = -1 on the hull
 *   tri_coords      (n_tri, 3, 3) float64 = triangle_coords()
 * layout is TB_LAYOUT_TET32/20/16 (records must match it) or TB_LAYOUT_TET80,
 * for which `records` is ignored and the 80-byte records are built from the
 * side tables and the points on the device. */
int tb_mesh_create(int device, int layout, int64_t n_points, const float* points_xyz,
                   int64_t n_tets, const uint32_t* records, const int32_t* side_verts,
                   const uint32_t* side_neighbors, int64_t n_cf, const int32_t* cf_triangle,
                   const int32_t* cf_tets, int64_t n_tri, const double* tri_coords,
                   tb_mesh** out);
int tb_mesh_destroy(tb_mesh* mesh);
/* Bytes of HBM the mesh occupies, and the hot bytes the walk gathers from on
 * the device: records + the six axis-permuted float4 point copies (96 B per
 * point; TetMesh-80: records only).  The reference's own accelerator count
 * (records + 12 B points, CompactMesh.accelerator_bytes, tetmesh.py:182-185)
 * is records + 12 * n_points. */
int tb_mesh_info(const tb_mesh* mesh, int* device, int* layout, int64_t* n_points,
                 int64_t* n_tets, int64_t* n_cf, int64_t* hbm_bytes, int64_t* hot_bytes);

/* 1 when the uploaded records passed the upload-time consistency check
 * (records equal the encoding of side_verts / side_neighbors,
 * tetmesh.py:299-320; neighbours symmetric and face-sharing): the walk then
 * provably stays in bounds and runs without its per-step index clamp.
 * 0 for meshes that fail it (e.g. records mutated in place): those keep the
 * clamp, so no read leaves the mesh arrays (results on such meshes are
 * undefined, as in the reference). */
int tb_mesh_validated(const tb_mesh* mesh, int* validated);

/* The batch epilogue alone (batch.py:57-71, _kernels_py._mt_t) from stored
 * results: triangle = cf_triangle[cf], fp64 t, tet_back, for rays whose
 * status / cf / tet came from a launch without the epilogue (the multi-GPU
 * frame assembly ships 13 B per ray and the root derives the other 16).
 * o, d, cf, tet, outputs: device pointers; identical to tb_cast_rays' fused
 * epilogue bit for bit. */
int tb_cast_epilogue(tb_mesh* mesh, int64_t n, const float* o, const float* d, const int32_t* cf,
                     const int32_t* tet, int32_t* triangle, double* t, int32_t* tet_back, void* stream);

/* Copy an uploaded mesh to another device (or the same one) peer to peer:
 * every device array, nothing rebuilt or revalidated (SURVEY 8 e: the mesh
 * is replicated per GPU; from HBM over NVLink instead of a second host
 * upload).  The replica is an independent handle (tb_mesh_destroy it). */
int tb_mesh_replicate(const tb_mesh* src, int device, tb_mesh** out);

/* Single-process multi-GPU trace (SURVEY 8 b's proposed tb_trace_multi; no
 * reference counterpart -- the reference renderer's tile pool,
 * render.py:496-541, is one process on CPU threads).  meshes[0..n_meshes)
 * are replicas of one mesh (same layout and size), each resident on its own
 * device (replicas may share a device).  The frame's width x height rays
 * (o, d, start: device pointers on meshes[0]'s device, pixel-major) are split
 * into 16 x 16-pixel tiles in render.py order, tile k to meshes[k % n].
 * Every device walks its tiles reading the rays from meshes[0]'s device and
 * stores each result into the output arrays there (also on meshes[0]'s
 * device, same layout as tb_cast_rays; triangle / t / tet_back may be NULL):
 * P2P loads and stores over NVLink, no staging copies, no collective.
 * Asynchronous on `stream` (a stream of meshes[0]'s device): the other
 * devices wait for the rays on it and `stream` waits for their results.
 * Fails (TB_E_CUDA) when a device cannot access meshes[0]'s device.  The
 * per-replica tile index arrays (8 B per pixel) are built once per (device,
 * frame size, replica count) and kept for the process. */
int tb_trace_multi(int n_meshes, tb_mesh* const* meshes, int64_t width, int64_t height, const float* o,
                   const float* d, const int32_t* start, uint8_t* status, int32_t* cf, int32_t* tet,
                   int32_t* visited, int32_t* triangle, double* t, int32_t* tet_back, void* stream);

/* Measurement helper (no reference counterpart; SURVEY 8 d asks the roofline
 * to be reported against a measured L2 gather bandwidth when the hot arrays
 * fit in L2).  Gathers n_pairs (record, point) pairs of this mesh at
 * independent pseudo-random indices -- the loads of one walk step, 8 pairs
 * in flight per thread -- so (layout + 12) * n_pairs / kernel time is the
 * random-gather roof of this mesh's working set.  Layouts 16/20/32 only.
 * sink: one device uint32 (practically never written).  Asynchronous on
 * stream; time it with events on that stream. */
int tb_probe_gather(tb_mesh* mesh, int64_t n_pairs, uint32_t seed, uint32_t* sink, void* stream);

/* Batch traversal with the batch-layer epilogue fused.
 * Replaces: _kernels.cast_rays (_kernels.pyx:271-370) -> (status, cf, tet,
 *   visited), plus batch.cast_rays' host epilogue (batch.py:57-71 and
 *   _kernels_py._mt_t, _kernels_py.py:435-454) -> (triangle, t, tet_back).
 *   o, d     (n, 3) float32; start (n,) int32
 *   status   (n,) uint8; cf, tet, visited (n,) int32
 *   triangle (n,) int32, t (n,) float64, tet_back (n,) int32 -- each may be
 *   NULL to skip that part of the epilogue.  Misses: triangle -1, t +inf,
 *   tet_back -1.  Start tets are NOT range-checked on the device: the caller
 *   validates them (the reference does not either). */
int tb_cast_rays(tb_mesh* mesh, int64_t n, const float* o, const float* d, const int32_t* start,
                 uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle,
                 double* t, int32_t* tet_back, void* stream);
/* tb_cast_rays with an explicit per-call ray schedule (tb_set_schedule's
 * modes; 0 = the process-wide setting).  Results are identical in every
 * mode.  Block compaction (3 / 4) is the faster choice for incoherent batches
 * (diffuse secondaries: rays starting all over the mesh), one ray per lane
 * (1) for coherent primaries and for tb_cast_rays_host, whose zero-copy path
 * is PCIe-bound and relies on one-ray-per-lane coalesced ray loads. */
int tb_cast_rays_sched(tb_mesh* mesh, int64_t n, const float* o, const float* d, const int32_t* start,
                       uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle,
                       double* t, int32_t* tet_back, int schedule, void* stream);
/* Rays per block of the cast kernels (the unit of tb_cast_rays_ordered). */
int tb_cast_block_size(void);
/* The schedule "auto" (mode 0) resolves to for a device-resident batch of n
 * rays on `device`: 7 (sampled longest-first) for launches of 6 to 48 waves
 * of blocks (a wave = SMs x 10 blocks), else 1 (one ray per lane). */
int tb_auto_schedule(int device, int64_t n);
/* Schedule 7's split for n rays on `device`: the number of leading blocks
 * that walk in launch order while the pre-pass orders the rest (0: no split,
 * every block ordered after the pre-pass).  At least 3 waves, the rest
 * ~65 % of the launch and at most 16 waves; TETB200_ORDER_TAIL (percent)
 * overrides.  Lets a caller count the launches (4 kernels split, 3 not). */
int64_t tb_sampled_head_blocks(int device, int64_t n);
/* Schedule 6 ("binned") for n device-resident rays without a scatter index:
 * 2 when the batch spans two or more 262144-ray sorting segments -- the
 * segments' first half is binned and walks on the caller's stream while the
 * second half is binned on a high-priority internal stream beside that walk
 * and walks there (config-2 secondaries +7.6 %, config 4 neutral; the sort is
 * segment-local, so the permutation is unchanged) -- else 1.
 * TETB200_BIN_SPLIT=0 disables the split. */
int tb_binned_pieces(int64_t n);
/* tb_cast_rays with a caller-chosen launch order of whole blocks: launch slot
 * b walks the tb_cast_block_size() rays of block block_order[b] (a
 * permutation of the n_blocks = ceil(n / block) blocks); rays are read and
 * results written in place, so outputs equal tb_cast_rays' bit for bit.  A
 * renderer tracing frame after frame orders a frame's blocks longest first by
 * the previous frame's walk lengths (visited), which removes most of the
 * launch's SM-idle tail (profiles/r02_experiments.md).  No reference
 * counterpart: the reference's tile pool (render.py:538-541) takes tiles in
 * order. */
int tb_cast_rays_ordered(tb_mesh* mesh, int64_t n, const float* o, const float* d, const int32_t* start,
                         const int32_t* block_order, int64_t n_blocks, uint8_t* status, int32_t* cf, int32_t* tet,
                         int32_t* visited, int32_t* triangle, double* t, int32_t* tet_back, void* stream);
/* block_order for tb_cast_rays_ordered from a previous similar batch's
 * per-ray visited counts (n rays, device memory): the batch's n_blocks
 * blocks, longest walk first (a block's key is its largest visited count,
 * bucketed at 4095), stream-ordered, no host round trip. */
int tb_block_order(int64_t n, const int32_t* visited, int32_t* order, int64_t n_blocks, void* stream);
/* tb_cast_rays whose ray r writes its seven results to index out_index[r]
 * (int64, device) of the output arrays: the multi-GPU frame assembly with
 * no separate collective -- every rank traces its image tiles and its trace
 * epilogue stores each finished ray straight into the root GPU's full-frame
 * arrays, mapped into this process with tb_ipc_open (CUDA IPC; P2P stores
 * over NVLink).  The caller synchronises the stream and then the ranks
 * (a barrier) before the root reads the frame.  No reference counterpart
 * (the reference is single-process, render.py:496-541). */
int tb_cast_rays_scatter(tb_mesh* mesh, int64_t n, const float* o, const float* d,
                         const int32_t* start, const int64_t* out_index, uint8_t* status,
                         int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle, double* t,
                         int32_t* tet_back, void* stream);
/* tb_cast_rays_scatter with an explicit schedule: 1 one ray per lane, 6 the
 * direction-binned walk (its permutation composed with out_index, so rays
 * are walked in binned order and still land at out_index[r]); 0 = the
 * process-wide setting; 2-4 (refill / compaction) have no scatter variant
 * and run one ray per lane.  Same results in every mode. */
int tb_cast_rays_scatter_sched(tb_mesh* mesh, int64_t n, const float* o, const float* d,
                               const int32_t* start, const int64_t* out_index, uint8_t* status,
                               int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle, double* t,
                               int32_t* tet_back, int schedule, void* stream);
/* The ScTP fallback walk (tb_sctp_cast_rays) with scattered outputs, as
 * tb_cast_rays_scatter: the multi-GPU frame assembly of a ScTP job. */
int tb_sctp_cast_rays_scatter(tb_mesh* mesh, int64_t n, const float* o, const float* d,
                              const int32_t* start, const int64_t* out_index, uint8_t* status,
                              int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle, double* t,
                              int32_t* tet_back, void* stream);

/* CUDA IPC of device allocations between the ranks of one node: the
 * 64-byte handle of the allocation holding dev_ptr (which must be the start
 * of a cudaMalloc'd block, e.g. from tb_device_alloc), its mapping into this
 * process on `device` (peer access enabled), and the unmapping. */
int tb_device_alloc(size_t bytes, int device, void** out);
int tb_device_free(void* ptr);
int tb_ipc_get_handle(const void* dev_ptr, void* handle_out);
int tb_ipc_open(const void* handle, int device, void** dev_ptr_out);
int tb_ipc_close(void* dev_ptr);

int tb_cast_rays_host(tb_mesh* mesh, int64_t n, const float* o, const float* d,
                      const int32_t* start, uint8_t* status, int32_t* cf, int32_t* tet,
                      int32_t* visited, int32_t* triangle, double* t, int32_t* tet_back);

/* Visit-sequence recording (the visits_sink path of _kernels.pyx:307-341,
 * consumed by batch.cast_rays_visits, batch.py:83-137).  Second pass of a
 * two-pass scheme: `offsets` (n+1,) int64 is the exclusive scan of the
 * `visited` output of a prior tb_cast_rays on the same rays; ray i's visited
 * tets are written to seq[offsets[i] : offsets[i+1]] (start tet first). */
int tb_cast_rays_visits(tb_mesh* mesh, int64_t n, const float* o, const float* d,
                        const int32_t* start, const int64_t* offsets, int32_t* seq, void* stream);

/* Batch point location.
 * Replaces: _kernels.locate_points (_kernels.pyx:416-492).
 *   q (n, 3) float64; hints (n,) int32; tet (n,) int32 (-1 = outside);
 *   visited (n,) int32. */
int tb_locate_points(tb_mesh* mesh, int64_t n, const double* q, const int32_t* hints,
                     int32_t* tet, int32_t* visited, void* stream);
int tb_locate_points_host(tb_mesh* mesh, int64_t n, const double* q, const int32_t* hints,
                          int32_t* tet, int32_t* visited);

/* Pinhole camera rays generated on the device (current device).
 * Replaces: render.camera_rays (render.py:169-185) for primary rays.
 *   frame: 14 float64 device values = fwd[3], right[3], up2[3], pos[3],
 *   half_w, half_h (computed on the host as render.camera_rays does);
 *   pixels (n,) int64 row-major pixel ids (y * width + x) or NULL for
 *   0..n-1; o, d (n, 3) float32 outputs, bit-identical to the host's. */
int tb_camera_rays(int64_t width, int64_t height, const double* frame, const int64_t* pixels, int64_t n,
                   float* o, float* d, void* stream);

/* A frame's primary pass in one launch: render.camera_rays (render.py:169-185)
 * fused with the cast from the camera tet (batch.cast_rays, batch.py:39-71)
 * -- each lane forms its pixel's ray exactly as tb_camera_rays does and
 * walks it; no rays are stored.  frame: 14 float64 HOST values (as for
 * tb_camera_rays, passed by value to the kernel); cam_tet: the located
 * camera tet (render.py:478-482); outputs (width * height,) as for
 * tb_cast_rays, device or mapped pinned host memory.  Results are
 * bit-identical to tb_camera_rays + tb_cast_rays. */
int tb_trace_camera(tb_mesh* mesh, int64_t width, int64_t height, const double* frame, int32_t cam_tet,
                    uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle, double* t,
                    int32_t* tet_back, void* stream);

/* Hull clipping for ray origins outside the mesh.
 * Replaces: the brute-force boundary-face search of traversal.cast_ray_auto
 *   (traversal.py:545-589, hull_faces traversal.py:530-542).
 *   o, d (n_all, 3) float32; rays (n,) int32 row indices into o/d, or NULL
 *   for rows 0..n-1; hull (n_hull, 4) int32 = (tet, v0, v1, v2) per
 *   boundary face in the reference's hull order.  Outputs, per ray: the
 *   index of the nearest hull face hit (fp64 Moller-Trumbore with u, v, t
 *   bounds; -1 = none) and its t. */
int tb_hull_clip(tb_mesh* mesh, int64_t n, const float* o, const float* d, const int32_t* rays,
                 int64_t n_hull, const int32_t* hull, int32_t* best_face, double* best_t, void* stream);

/* Batch occlusion (shadow) walks.
 * Replaces: _kernels.shadow_rays (_kernels.pyx:527-614).
 *   p (n, 3) float64; light (n,3) float64 when light_stride == 3, or a single
 *   (3,) point when light_stride == 0; p_tet (n,) int32; light_tet (n,) int32
 *   when light_tet_stride == 1 or a single value when 0; occluded (n,) uint8;
 *   visited (n,) int32. */
int tb_shadow_rays(tb_mesh* mesh, int64_t n, const double* p, const double* light,
                   int light_stride, const int32_t* p_tet, const int32_t* light_tet,
                   int light_tet_stride, double eps, uint8_t* occluded, int32_t* visited,
                   void* stream);
int tb_shadow_rays_host(tb_mesh* mesh, int64_t n, const double* p, const double* light,
                        int light_stride, const int32_t* p_tet, const int32_t* light_tet,
                        int light_tet_stride, double eps, uint8_t* occluded, int32_t* visited);

/* Fallback traversal with the fp64 scalar-triple-product exit test (ScTP).
 * Replaces: traversal.sctp_exit_face (traversal.py:484-511) applied per tet
 * (the reference has the predicate only, no walk).  Same
 * outputs and epilogue as tb_cast_rays. */
int tb_sctp_cast_rays(tb_mesh* mesh, int64_t n, const float* o, const float* d,
                      const int32_t* start, uint8_t* status, int32_t* cf, int32_t* tet,
                      int32_t* visited, int32_t* triangle, double* t, int32_t* tet_back,
                      void* stream);
int tb_sctp_cast_rays_host(tb_mesh* mesh, int64_t n, const float* o, const float* d,
                           const int32_t* start, uint8_t* status, int32_t* cf, int32_t* tet,
                           int32_t* visited, int32_t* triangle, double* t, int32_t* tet_back);

/* Ray scheduling of tb_cast_rays / tb_cast_rays_host (no reference
 * counterpart: the reference walks one ray per loop iteration,
 * _kernels.pyx:343-369).  Results are identical in every mode; only the
 * mapping of rays to lanes changes.
 *   mode 0 = auto (= one ray per lane), 1 = one ray per lane, 2 = per-lane
 *   persistent refill,
 *   3 / 4 = block compaction (256 / 512 threads per block) for incoherent
 *   batches; steps_per_round = walk steps between compactions (>= 1),
 *   6 = direction binning: a stable counting sort of the ray indices by
 *   direction cell (cube-map face of the dominant axis x 4 x 4 cells, 96
 *   bins; stream-ordered scratch, 9 B / ray), then one ray per lane in
 *   binned order, each ray read and its results stored by index --
 *   for incoherent device-resident batches (n < 2^31; host-ray zero-copy
 *   calls run one ray per lane), 5 = dynamic warp chunks (kept for
 *   comparison), 7 = sampled longest-first: one ray per block walked at most
 *   32 steps orders the blocks longest first, then the full walk launches
 *   them in that order (tb_cast_rays_ordered's kernel) -- for coherent
 *   device-resident primaries, whose launch otherwise ends on a few late
 *   long rays.  Split launches (tb_sampled_head_blocks > 0): the leading
 *   blocks walk in launch order on the caller's stream while a
 *   high-priority internal stream probes, orders and launches the rest; the
 *   caller's stream waits for it before the call's later work.  Results are
 *   identical in every mode. 
 * Process-wide; overrides TETB200_SCHED / TETB200_ROUND.  A negative
 * argument leaves that setting unchanged. */
int tb_set_schedule(int mode, int steps_per_round);
int tb_get_schedule(int* mode, int* steps_per_round);

/* Host-side mesh building (plain C++, no GPU; csrc/host_mesh.cpp) -- the
 * native backing of the Python mesh layer, bit-identical to the reference's
 * numpy code paths it replaces.
 *   tb_hilbert_keys      3-D Hilbert keys of (n,3) int64 grid cells, order
 *                        1..20 (hilbert.py:14-58).
 *   tb_hilbert_quantize  (n,3) float64 points -> grid cells of [lo, hi]
 *                        (hilbert.py:66-73).
 *   tb_tet_centroids     float64 centroid of each (t,4) quad, numpy mean order
 *                        (tetmesh.py:466).
 *   tb_build_side_tables sorted-slot side tables: row i of the output is row
 *                        row_of[i] (NULL = i) of (verts, refs), vertex ids
 *                        mapped through vert_map and plain tet references
 *                        through tet_map (NULL = identity), slots stably
 *                        sorted by vertex id (tetmesh.py:350-352, :482-491).
 *   tb_pack_records      Tet32/20/16 records from the side tables
 *                        (tetmesh.py:299-320).
 * All return 0 or TB_E_ARG / TB_E_LAYOUT. */
int tb_hilbert_keys(const int64_t* cells, int64_t n, int order, uint64_t* keys);
int tb_hilbert_quantize(const double* pts, int64_t n, const double* lo, const double* hi, int order,
                        int64_t* cells);
int tb_tet_centroids(const double* pts, int64_t n_points, const int32_t* quads, int64_t n, double* out);
int tb_build_side_tables(int64_t n, const int32_t* verts, const uint32_t* refs, const int64_t* row_of,
                         const int64_t* vert_map, int64_t n_vert_map, const int64_t* tet_map,
                         int64_t n_tet_map, int32_t* sv_out, uint32_t* sn_out);
int tb_pack_records(int layout, int64_t n, const int32_t* sv, const uint32_t* sn, uint32_t* words);

/* Pinned host memory helpers for end-to-end callers. */
int tb_host_alloc(size_t bytes, void** out);
int tb_host_free(void* ptr);

const char* tb_last_error(void);
int tb_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TETB200_H */
