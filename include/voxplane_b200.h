/* voxplane_b200 — C ABI of the B200-native voxel-map / plane-segmentation path.
 *
 * Drop-in for the hot path of the reference C++ library `voxplane`
 * (/root/reference/proj/core): the per-frame update
 *   clear_rays -> integrate_frame -> recenter -> estimate_normals ->
 *   classify_steppable -> build_adjacency + label_components ->
 *   filter_clusters -> fit_planes -> refine_plane -> make_polygon
 * driven by run_frames (pipeline.cpp:199-213) and voxel_frame_polygons
 * (pipeline.cpp:43-85). Every entry point below names the reference
 * interface it replaces. Plain pointers and sizes only; no C++ or torch types.
 *
 * Conventions
 *   - return value: VP_OK or a VP_E* code; vp_last_error() gives the message
 *     (thread-local). VP_EINVAL corresponds to the reference's
 *     std::invalid_argument, VP_EEMPTY to estimate_normals on an empty grid.
 *   - rotations are 9 doubles row-major (r00 r01 r02 r10 ...), translations 3.
 *   - points are n x 3 float32 sensor-frame xyz (SensorFrame::points).
 *   - voxel indices are window (logical) coordinates, as the reference's.
 *   - arrays returned through vp_*_t** are owned by the library; free them
 *     with the matching vp_*_free.
 *   - every call is synchronous on return (the grid's CUDA stream is drained).
 */
#ifndef VOXPLANE_B200_H
#define VOXPLANE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VP_OK 0
#define VP_EINVAL 1    /* std::invalid_argument in the reference            */
#define VP_EEMPTY 2    /* estimate_normals: empty grid (segmentation.cpp:22) */
#define VP_ENOMEM 3    /* device allocation failed                          */
#define VP_ECUDA 4     /* CUDA runtime / launch error                       */
#define VP_ENODEV 5    /* no usable sm_100 device                           */

typedef struct vp_grid vp_grid;         /* VoxelGrid (voxel_grid.hpp:17-91)  */
typedef struct vp_pipeline vp_pipeline; /* run_frames state (pipeline.cpp:157-245) */

/* types.hpp:63-76 */
typedef struct { uint64_t voxels_touched, points_discarded; } vp_update_stats;
typedef struct { uint64_t voxels_cleared, voxels_freed; } vp_clear_stats;
typedef struct { int32_t shift[3]; uint64_t voxels_dropped; } vp_shift_stats;

/* SegmentationParams (segmentation.hpp:11-19) */
typedef struct {
  int32_t neighbor_radius;     /* 1 */
  int32_t min_neighbors;       /* 3 */
  double max_angle_deg;        /* 15 */
  double adjacency_angle_deg;  /* 15 */
  double distance_th;          /* 0.05 */
  int32_t min_cluster_size;    /* 30 */
  double up[3];                /* (0,0,1) */
} vp_seg_params;

/* RansacParams (plane_fit.hpp:28-34); execution: 0 ClusterParallel, 1 PerClusterSerial */
typedef struct {
  int32_t iterations;  /* 100 */
  double inlier_eps;   /* 0.01 */
  uint64_t seed;       /* 0 (RunConfig.seed is synced in by the config loader) */
  double up[3];
  int32_t execution;
} vp_ransac_params;

/* Everything voxel_frame_polygons reads from PipelineConfig (pipeline.cpp:43-85). */
typedef struct {
  vp_seg_params seg;
  vp_ransac_params ransac;
  int32_t refine;            /* RunConfig.refine, default 1 */
  double min_polygon_area;   /* OutputConfig.min_polygon_area, default 0.002 */
  int32_t refine_exact;      /* 1: sequential refine sums (bit-identical to the
                                reference); 0: deterministic tree reduction
                                (within the 1e-4 rad / 1e-4 m tolerance) */
} vp_pipeline_params;

/* PlaneModel (plane_fit.hpp:13-18) */
typedef struct {
  double normal[3];
  double offset;
  int32_t inlier_count;
  int32_t cluster_label;
} vp_plane;

/* PlanePolygon (polygonize.hpp:49-54) */
typedef struct {
  vp_plane plane;
  uint32_t nverts;
  const double* v2d; /* nverts x 2 */
  const double* v3d; /* nverts x 3 */
  double area;
} vp_polygon;

typedef struct {
  size_t count;
  vp_polygon* polys;
} vp_polygons_t;

/* OccupiedVoxel list (types.hpp:19-24), lexicographic window order */
typedef struct {
  size_t count;
  int32_t* idx;     /* count x 3 */
  double* mean;     /* count x 3 */
  uint32_t* npts;   /* count     */
  uint8_t* status;  /* count     */
} vp_occupied_t;

/* SurfaceEstimate list (segmentation.hpp:24-31) */
typedef struct {
  size_t count;
  int32_t* idx;            /* count x 3 */
  double* mean;            /* count x 3 */
  double* normal;          /* count x 3 */
  int32_t* neighbor_count;
  double* angle_to_up_deg; /* host libm acos of normal.up (segmentation.cpp:62-63) */
  uint8_t* valid;
} vp_estimates_t;

/* SteppablePoint list (segmentation.hpp:33-42), ordinal = position */
typedef struct {
  size_t count;
  int32_t* idx;    /* count x 3 */
  double* mean;    /* count x 3 */
  double* normal;  /* count x 3 */
} vp_steppable_t;

/* ClusterFit list (plane_fit.hpp:36-39); inliers of fit f are
   inliers[offsets[f] .. offsets[f+1]) (x3 doubles) */
typedef struct {
  size_t count;
  vp_plane* models;
  uint64_t* offsets;  /* count + 1 */
  double* inliers;
  uint64_t clusters_skipped_small; /* FitStats (plane_fit.hpp:41-44) */
  uint64_t clusters_unfit;
} vp_fits_t;

/* FrameTiming stage spans (metrics.hpp:51-62), CUDA-event milliseconds */
typedef struct {
  double mapping_ms, classify_ms, cluster_ms, ransac_ms, hull_ms, total_ms;
  uint64_t points, voxels, clusters;
} vp_frame_timing;

const char* vp_last_error(void);
const char* vp_version(void);

/* ---- defaults (segmentation.hpp:11-19, plane_fit.hpp:28-34, config.hpp:13-28) */
void vp_default_params(vp_pipeline_params* p);

/* ---- VoxelGrid ------------------------------------------------------- */
/* VoxelGrid::VoxelGrid (voxel_grid.cpp:19-25); throws invalid_argument -> VP_EINVAL */
int vp_grid_create(double resolution, const int32_t extent[3], const double center[3],
                   int device, vp_grid** out);
void vp_grid_destroy(vp_grid* g);
/* origin() / extent() / resolution() / occupied_count() (voxel_grid.hpp:32-52) */
int vp_grid_info(const vp_grid* g, double origin[3], int32_t extent[3], double* resolution,
                 uint64_t* occupied_count);
/* VoxelGrid::integrate_frame (voxel_grid.cpp:59-115) */
int vp_integrate_frame(vp_grid* g, const float* xyz, uint64_t n, const double rotation[9],
                       const double translation[3], vp_update_stats* stats);
/* VoxelGrid::clear_rays (voxel_grid.cpp:182-215) */
int vp_clear_rays(vp_grid* g, const float* xyz, uint64_t n, const double rotation[9],
                  const double translation[3], vp_clear_stats* stats);
/* clear_rays followed by integrate_frame on one frame (pipeline.cpp:200-201)
   with a single staging of the points; xyz may be a host or device pointer. */
int vp_update_frame(vp_grid* g, const float* xyz, uint64_t n, const double rotation[9],
                    const double translation[3], vp_clear_stats* cleared, vp_update_stats* updated);
/* VoxelGrid::recenter (voxel_grid.cpp:217-252) */
int vp_recenter(vp_grid* g, const double new_center[3], vp_shift_stats* stats);
/* VoxelGrid::merge_point (voxel_grid.cpp:49-57), idx in window coordinates */
int vp_merge_point(vp_grid* g, const int32_t idx[3], const double p[3]);
/* VoxelGrid::cell(idx) (voxel_grid.hpp:49): sums, count, status of one cell */
int vp_get_cell(vp_grid* g, const int32_t idx[3], double sum[3], uint32_t* count,
                uint8_t* status);
/* VoxelGrid::set_status (voxel_grid.hpp:78) */
int vp_set_status(vp_grid* g, const int32_t idx[3], uint8_t status);
/* set_status for n voxels (idx n x 3) in one transfer (classify_steppable writeback) */
int vp_set_statuses(vp_grid* g, const int32_t* idx, const uint8_t* status, size_t n);
/* VoxelGrid::occupied_voxels (voxel_grid.cpp:254-263) */
int vp_occupied_voxels(vp_grid* g, vp_occupied_t** out);
void vp_occupied_free(vp_occupied_t* o);

/* ---- segmentation.hpp -------------------------------------------------- */
/* estimate_normals (segmentation.cpp:19-67) */
int vp_estimate_normals(vp_grid* g, const vp_seg_params* p, vp_estimates_t** out);
void vp_estimates_free(vp_estimates_t* e);
/* classify_steppable (segmentation.cpp:69-85) on the grid's current estimates
   (fused on device with estimate_normals); writes statuses back to the grid.
   objects_idx (optional) receives V_obj x 3 indices. */
int vp_classify_steppable(vp_grid* g, const vp_seg_params* p, vp_steppable_t** steppable,
                          int32_t** objects_idx, size_t* n_objects);
void vp_steppable_free(vp_steppable_t* s);
void vp_free(void* p);
/* build_adjacency + label_components (segmentation.cpp:87-194) for a host
   steppable list: labels[i] = canonical component minimum ordinal. */
int vp_label_components(const vp_steppable_t* steppable, const vp_seg_params* p,
                        double resolution, int device, int32_t* labels);
/* build_adjacency (segmentation.cpp:87-132) materialised as CSR (ascending
   neighbour lists) for API completeness; not used on the fused path. */
int vp_build_adjacency(const vp_steppable_t* steppable, const vp_seg_params* p,
                       double resolution, int device, uint64_t** row_offsets,
                       int32_t** cols, uint64_t* n_edges);

/* ---- plane_fit.hpp / polygonize.hpp ------------------------------------ */
/* fit_planes (plane_fit.cpp:55-131). Clusters in CSR form: cluster c has
   label labels[c] and member means means[offsets[c] .. offsets[c+1]) (x3). */
int vp_fit_planes(size_t n_clusters, const int32_t* labels, const uint64_t* offsets,
                  const double* means, const vp_ransac_params* p, int device,
                  vp_fits_t** out);
void vp_fits_free(vp_fits_t* f);
/* refine_plane (plane_fit.cpp:133-154) for every fit; exact!=0 reproduces
   the sequential sums bit-for-bit. */
int vp_refine_planes(const vp_fits_t* fits, const double up[3], int exact, int device,
                     vp_plane* refined);
/* make_polygon (polygonize.cpp:166-182) for every (plane, inlier set);
   polygons that are nullopt in the reference come back with nverts == 0. */
int vp_make_polygons(size_t n, const vp_plane* planes, const uint64_t* offsets,
                     const double* inliers, int filter_directions, int device,
                     vp_polygons_t** out);
void vp_polygons_free(vp_polygons_t* p);

/* ---- reference-named utilities on the device ----------------------------- */
/* jacobi_eigen_sym3 (jacobi.hpp:10-18, jacobi.cpp:46-81) for n symmetric 3x3
   matrices a (row-major, 9 each): eigenvalues ascending (3 each),
   eigenvectors column-major (9 each; column k pairs with eigenvalue k,
   right-handed). The kernel is the one estimate_normals runs. */
int vp_jacobi_eigen_sym3(size_t n, const double* a, double* eigenvalues, double* eigenvectors, int device);
/* hull_filter (polygonize.hpp:32-33, polygonize.cpp:50-114): the points
   (n x 2) not strictly inside the polygon of the extremes along `directions`
   directions, in input order; *out (m x 2) is freed with vp_free. */
int vp_hull_filter(const double* pts, uint64_t n, int directions, int device, double** out, uint64_t* m);
/* monotone_chain (polygonize.hpp:34-37, polygonize.cpp:116-139): strict CCW
   hull from the lexicographic minimum, empty when collinear. */
int vp_monotone_chain(const double* pts, uint64_t n, int device, double** out, uint64_t* m);
/* convex_hull (polygonize.hpp:38-39, polygonize.cpp:141-144): hull_filter
   then monotone_chain. */
int vp_convex_hull(const double* pts, uint64_t n, int directions, int device, double** out, uint64_t* m);
/* label_components(steppable, adjacency) (segmentation.hpp:74-75,
   segmentation.cpp:147-194) over explicit adjacency lists in CSR form
   (row_offsets n + 1, cols): labels[i] = component-minimum ordinal. */
int vp_label_components_adjacency(uint64_t n, const uint64_t* row_offsets, const int32_t* cols, int device,
                                  int32_t* labels);
/* classify_steppable(grid, estimates, params) (segmentation.hpp:68-70,
   segmentation.cpp:69-85) over caller-provided estimates (voxel indices
   n x 3, neighbor_count, angle_to_up_deg, valid): status[i] = 2 (Steppable)
   or 1 (Occupied), written to the grid's cells as well. */
int vp_classify_estimates(vp_grid* g, const vp_seg_params* p, size_t n, const int32_t* idx,
                          const int32_t* neighbor_count, const double* angle_to_up_deg, const uint8_t* valid,
                          uint8_t* status);

/* ---- composite ----------------------------------------------------------- */
/* segment(): voxel_frame_polygons (pipeline.cpp:43-85) on the device-resident
   grid: polygons in ascending cluster-label order, area-filtered. */
int vp_segment(vp_grid* g, const vp_pipeline_params* p, vp_polygons_t** out,
               vp_frame_timing* timing);

/* ---- spatial slabs --------------------------------------
   A window of window_extent voxels is split along x; a slab grid owns window
   x in [x_begin, x_end) and stores one halo plane on each side. Clear and
   integrate run on every slab with the full window's arithmetic (rays are
   clipped to the whole window and walked from their start) and keep only
   owned cells and points; halo planes are filled from the neighbours
   (vp_grid_plane) before estimate_normals; the per-slab steppable lists,
   concatenated in slab order, are exactly the single-grid list (ordinals
   are x-major), and vp_segment_steppable runs CCL .. make_polygon on it.
   Slab windows are fixed (no recenter), as for SURVEY §8(d) C5. */
int vp_slab_create(double resolution, const int32_t window_extent[3], const double center[3],
                   int32_t x_begin, int32_t x_end, int device, vp_grid** out);
/* Device pointers to the cell records and occupancy-bitmap words of window
   plane x (owned or halo) of a grid; the halo exchange copies owned boundary
   planes of one slab onto the halo planes of its neighbour. */
int vp_grid_plane(vp_grid* g, int32_t window_x, void** cells, uint64_t* cell_bytes, void** bits,
                  uint64_t* bit_bytes);
/* estimate_normals + classify_steppable over the owned voxels; returns the
   steppable list (window indices) as device arrays owned by the grid, valid
   until the next call on it. */
int vp_slab_steppable(vp_grid* g, const vp_seg_params* p, uint64_t* count, int32_t** idx,
                      double** mean, double** normal);
/* build_adjacency .. make_polygon (voxel_frame_polygons after classify) on a
   steppable list in window coordinates (device or host arrays). */
int vp_segment_steppable(vp_grid* g, const vp_pipeline_params* p, uint64_t n, const int32_t* idx,
                         const double* mean, const double* normal, int device_ptrs,
                         vp_polygons_t** out);

/* ---- distributed segmentation over slabs -----------------
   build_adjacency + label_components (segmentation.cpp:87-194) run per slab
   on its own steppable voxels plus the w = max(1, ceil(distance_th / res))
   planes either side (segmentation.cpp:89), received from the slabs that own
   them; a boundary-label merge makes the labels the single-grid canonical
   ones (component-minimum global ordinal); every cluster's members are sent
   to the slab owning its label, which runs filter_clusters .. make_polygon
   (pipeline.cpp:43-85) for the clusters it owns. Per frame, after
   vp_slab_steppable:
     vp_slab_plane_counts -> (all-gather) -> vp_slab_extend -> (halo lists)
     -> vp_slab_label -> (all-gather of triples) -> vp_slab_merge
     -> vp_slab_export -> (members to owners) -> vp_slab_segment_owned
   All arrays are device arrays owned by the grid unless stated. */
typedef struct {
  int32_t n_slabs;
  const int32_t* x_begin;        /* n_slabs + 1: first window x of every slab, then window extent x */
  const uint32_t* plane_counts;  /* window_extent[0]: steppable voxels per window x-plane, all slabs */
} vp_slab_layout;
/* A cluster member on its way to the slab that owns the cluster (32 B). */
typedef struct {
  double mean[3];
  int32_t label;   /* canonical label = global ordinal of the cluster's minimum */
  int32_t pad;
} vp_member_rec;

/* segmentation.cpp:89 */
int vp_adjacency_window(const vp_seg_params* p, double resolution, int32_t* w);
/* Steppable voxels per owned x-plane (n_planes = owned planes), from the
   last vp_slab_steppable. */
int vp_slab_plane_counts(vp_grid* g, uint32_t** counts, int32_t* n_planes);
/* Extended list of window planes [x_lo, x_hi) = owned planes +- w (clipped):
   the own list is copied into place; the caller fills the halo entries
   (entries of plane x start at index P[x] - P[x_lo], P = prefix sum of the
   layout's plane counts) from the owning slabs' lists. */
int vp_slab_extend(vp_grid* g, const vp_seg_params* p, const vp_slab_layout* layout, int32_t** idx,
                   double** mean, double** normal, uint64_t* n_ext, int32_t* x_lo, int32_t* x_hi);
/* Local union-find over the extended list; returns this slab's boundary
   triples (3 x int32: zone index of an entry in the boundary zone, zone
   index of its local component's smallest zone entry, local label) and the
   zone size (same on every slab). */
int vp_slab_label(vp_grid* g, const vp_seg_params* p, int32_t** triples, uint64_t* n_triples,
                  uint64_t* zone_size);
/* Merge the triples of all slabs (device; triples with a negative first
   entry are padding); labels = canonical label of every owned entry. */
int vp_slab_merge(vp_grid* g, const int32_t* triples, uint64_t n_triples, int32_t** labels);
/* Members of clusters owned by lower slabs, sorted by destination slab
   (ascending ordinal within each); dest_counts (host, n_slabs entries). */
int vp_slab_export(vp_grid* g, uint64_t* dest_counts, void** records);
/* filter_clusters .. make_polygon for the clusters this slab owns: its own
   members followed by the records received from the higher slabs in slab
   order (device vp_member_rec array). Polygons in ascending label order. */
int vp_slab_segment_owned(vp_grid* g, const vp_pipeline_params* p, const void* recv, uint64_t n_recv,
                          vp_polygons_t** out);

/* End-to-end latency of the last vp_pipeline_frame / _device call (SURVEY
   §8(d) unit of work): CUDA events from before the points' H2D copy to after
   the frame's polygons are assembled in host memory, in milliseconds. */
int vp_pipeline_latency_ms(const vp_pipeline* pl, double* ms);

/* ---- one slab frame, orchestrated in the library --------
   The whole per-frame exchange sequence above (frame broadcast, halo planes,
   plane counts, halo steppable lists, boundary triples, cluster members,
   polygon gather to rank 0) as ONE call per rank, over a communicator given
   as a table of stream-ordered collectives on device buffers -- the library's
   own NCCL communicator (vp_comm_nccl_create: NVLink / NVSwitch between the
   GPUs of a node) or any caller-provided implementation with the same
   semantics (e.g. torch.distributed). */
typedef struct {
  int32_t peer;
  int32_t send;   /* 1 send, 0 receive */
  void* ptr;      /* device buffer */
  uint64_t bytes;
} vp_p2p_op;
typedef struct {
  void* ctx;
  int32_t rank;
  int32_t nranks;
  /* stream = the slab grid's cudaStream_t; all buffers are device memory;
     each returns 0 on success */
  int (*broadcast)(void* ctx, void* buf, uint64_t bytes, int32_t root, void* stream);
  int (*allgather)(void* ctx, const void* send, void* recv, uint64_t bytes_per_rank, void* stream);
  /* point-to-point sends / receives as one group (matched in call order per peer pair) */
  int (*group)(void* ctx, int32_t n, const vp_p2p_op* ops, void* stream);
} vp_comm_ops;
/* NCCL communicator of nranks GPUs (libnccl.so.2 is loaded at run time; one
   rank per GPU, one process per rank). Rank 0 creates the 128-byte id and the
   caller hands it to every rank (any host channel). */
int vp_comm_nccl_unique_id(uint8_t id[128]);
int vp_comm_nccl_create(const uint8_t id[128], int32_t nranks, int32_t rank, int device, vp_comm_ops* out);
int vp_comm_nccl_destroy(vp_comm_ops* comm);
/* One frame on this rank's slab (rank k of the communicator owns slab k; the
   slabs' x ranges tile the window in rank order): points are rank 0's (host
   or device; the other ranks pass the same n and NULL); polygons of the
   whole window in ascending label order on rank 0 (NULL elsewhere) -- equal
   to run_frames' voxel_frame_polygons on one grid. */
int vp_slab_frame(vp_grid* slab, const vp_comm_ops* comm, const float* xyz, uint64_t n,
                  const double rotation[9], const double translation[3], const vp_pipeline_params* p,
                  vp_polygons_t** out);
/* The same with n_slabs slabs in this process (virtual slabs, e.g. on one
   GPU): one host thread per slab runs vp_slab_frame over an in-process
   communicator (device-to-device copies). */
int vp_slab_frame_local(vp_grid* const* slabs, int32_t n_slabs, const float* xyz, uint64_t n,
                        const double rotation[9], const double translation[3], const vp_pipeline_params* p,
                        vp_polygons_t** out);

/* run_frames state: a grid plus the global-cell recenter trigger
   (pipeline.cpp:165, 174, 199-213). */
int vp_pipeline_create(double resolution, const int32_t extent[3],
                       const double start_center[3], const vp_pipeline_params* p,
                       int device, vp_pipeline** out);
void vp_pipeline_destroy(vp_pipeline* pl);
/* Empty the map and re-centre it (the state of a freshly constructed
   VoxelGrid plus run_frames' last_cell), keeping every device allocation. */
int vp_pipeline_reset(vp_pipeline* pl, const double start_center[3]);
vp_grid* vp_pipeline_grid(vp_pipeline* pl);
/* The cudaStream_t the pipeline's kernels run on (for external event timing). */
void* vp_pipeline_stream(vp_pipeline* pl);
/* Counters of the last frame: cleared, freed, touched, discarded, dropped,
   occupied, V_occ, V_step, clusters, fits, padded members, inliers,
   polygon vertices, newly occupied, largest hull-survivor set, overflow flags. */
int vp_pipeline_counters(vp_pipeline* pl, uint64_t out[16]);
/* The same counters for a grid driven through the grid / slab entry points
   (values of the last call that read them back). */
int vp_grid_counters(vp_grid* g, uint64_t out[16]);
/* One frame of run_frames: clear_rays, integrate_frame, recenter-if-moved,
   voxel_frame_polygons. out may be NULL (polygons stay on the device);
   timing may be NULL (the per-stage device times cost six event queries,
   ~17 us of host time per frame). */
int vp_pipeline_frame(vp_pipeline* pl, const float* xyz, uint64_t n, const double rotation[9],
                      const double translation[3], vp_polygons_t** out,
                      vp_frame_timing* timing);
/* Same frame step, device-resident input (xyz_dev is a device pointer). */
int vp_pipeline_frame_device(vp_pipeline* pl, const float* xyz_dev, uint64_t n,
                             const double rotation[9], const double translation[3],
                             vp_polygons_t** out, vp_frame_timing* timing);
/* run_frames (pipeline.cpp:157-245) over n_frames frames: frame k's points
   are xyz[k] (n[k] x 3 floats; device pointers when device_ptrs != 0), pose
   rotations[9k..], translations[3k..]. Consecutive frames overlap on the
   device (frame k+1's mapping runs beside frame k's fitting and polygon
   stages); outputs are those of calling vp_pipeline_frame per frame. out
   receives the final frame's polygons (PipelineResult::polygons); timings
   (optional, n_frames entries) the per-frame device spans. */
int vp_pipeline_run(vp_pipeline* pl, size_t n_frames, const float* const* xyz, const uint64_t* n,
                    const double* rotations, const double* translations, int device_ptrs,
                    vp_polygons_t** out, vp_frame_timing* timings);
/* Per-frame outputs of a pipelined run; every member is optional (NULL) and
   points at n_frames entries. per_frame[k] receives frame k's polygons
   (run_frames' per_frame_polygons, pipeline.cpp:223-227; free each with
   vp_polygons_free); timings[k] its FrameTiming stage spans (pipeline.cpp:
   181-219, CUDA-event ms); traces[k] / trace_lens[k] its stage trace
   (voxplane_trace.h, as vp_pipeline_frame_trace; free with vp_free). */
typedef struct {
  vp_polygons_t** per_frame;
  vp_frame_timing* timings;
  uint8_t** traces;
  uint64_t* trace_lens;
} vp_run_outputs;
/* vp_pipeline_run with per-frame outputs: the body of run_frames
   (pipeline.cpp:157-245) with frames in flight; every frame's polygons are
   packed on the device into mapped host memory (no copy, no stream wait). */
int vp_pipeline_run_frames(vp_pipeline* pl, size_t n_frames, const float* const* xyz, const uint64_t* n,
                           const double* rotations, const double* translations, int device_ptrs,
                           vp_polygons_t** out, const vp_run_outputs* extra);
/* Same frame step, returning the stage trace (voxplane_trace.h); buf is
   freed with vp_free. */
int vp_pipeline_frame_trace(vp_pipeline* pl, const float* xyz, uint64_t n,
                            const double rotation[9], const double translation[3],
                            uint8_t** buf, uint64_t* len);

/* ---- height-map baseline (heightmap.hpp:10-55, heightmap.cpp:9-89) -------
   The paper's Table I 2.5-D baseline: one height per (x, y) cell, latest
   measurement wins in point order; segment = BFS region growing over
   4-neighbours with |dh| < distance_th from seeds in lexicographic order
   (region id = seed flat index, members in BFS order), then fit_planes,
   refine_plane (p->refine, p->refine_exact) and make_polygon as the voxel
   path. Polygons with area < p->min_polygon_area are dropped (run_frames'
   filter, pipeline.cpp:190-193; pass -inf for plain hm_segment). */
typedef struct vp_heightmap vp_heightmap;
int vp_heightmap_create(double resolution, const int32_t extent[2], const double center[2], int device,
                        vp_heightmap** out);
void vp_heightmap_destroy(vp_heightmap* hm);
int vp_hm_integrate(vp_heightmap* hm, const float* xyz, uint64_t n, const double rotation[9],
                    const double translation[3]);
/* heights / valid flags of all cells (x-major), host arrays of extent[0]*extent[1] */
int vp_hm_cells(vp_heightmap* hm, double* heights, uint8_t* valid);
int vp_hm_segment(vp_heightmap* hm, const vp_pipeline_params* p, vp_polygons_t** out);
/* The last segment's regions: the visit sequence (all region cells, BFS
   order per region, host array of >= extent cells) and every cell's region
   root (its seed's flat index; own index for invalid cells). */
int vp_hm_regions(vp_heightmap* hm, uint32_t* visit, int32_t* root, uint64_t* nv);

/* ---- plane IoU scoring (metrics.cpp:19-185; the paper's Table I metric) --
   match_planes: every (truth, detected) pair within the 20 deg normal gate is
   projected into the truth plane and rasterised at raster_res (plane_iou,
   default 0.005 m; one block per pair on the device, integer counts), pairs
   matched greedily by IoU; matches (capacity min(#detected, #truth)) in
   truth order. write_iou_report writes the reference's report text. */
typedef struct {
  int32_t detected_id, truth_id;
  double iou;
} vp_plane_match;
typedef struct {
  uint64_t truth_count, detected_count, matched, unmatched_truth, unmatched_detected;
  double mean_iou, area_weighted_iou;
} vp_iou_report;
int vp_match_planes(const vp_polygons_t* detected, const vp_polygons_t* truth, double raster_res, int device,
                    vp_iou_report* report, vp_plane_match* matches);
int vp_write_iou_report(const char* path, const vp_iou_report* report, const vp_plane_match* matches);

/* ---- frame and polygon formats on the GPU path (frame_io.cpp:91-116,
   polygon_io.cpp:30-47) ---------------------------------------------------
   A VXPF stream (magic "VXPF", u32 version 1, per frame u32 n, 12 f32 pose
   [R|t] row-major, n x 3 f32 xyz) is read once into pinned host memory, so
   replay feeds run_frames with asynchronous H2D copies and no per-frame
   host staging. Errors as the reference: a missing file, bad magic or
   version, or a truncated frame -> VP_EINVAL with the reference's message. */
typedef struct vp_stream vp_stream;
int vp_stream_open(const char* path, vp_stream** out);
void vp_stream_close(vp_stream* s);
uint64_t vp_stream_count(const vp_stream* s);
/* Frame i: pinned xyz (n x 3 f32), pose as doubles (f32 values, as read). */
int vp_stream_frame(const vp_stream* s, uint64_t i, const float** xyz, uint64_t* n, double rotation[9],
                    double translation[3]);
/* run_frames over frames [first, first + count) of a stream (replay_pipeline,
   pipeline.cpp:291-302): out = the last frame's polygons, timings optional. */
int vp_pipeline_replay(vp_pipeline* pl, const vp_stream* s, uint64_t first, uint64_t count,
                       vp_polygons_t** out, vp_frame_timing* timings);
/* write_frames_binary (frame_io.cpp:74-89): frames given as host arrays. */
int vp_write_frames_binary(const char* path, size_t n_frames, const float* const* xyz, const uint64_t* n,
                           const double* rotations, const double* translations);
/* write_polygons (polygon_io.cpp:30-47): the golden-file text, %.9g. */
int vp_write_polygons(const char* path, const vp_polygons_t* polygons);

/* ---- cluster-parallel ablation (pipeline.cpp:304-381, Fig. 9) -------------
   Per trial (trial-major, alternating mode order as the reference): M drawn
   from CounterRng(seed, count, trial) in [points_min, points_max], `count`
   clusters of exactly M synthetic points (the reference's generator, bit for
   bit, on the host), staged on the device, then fit_planes timed with CUDA
   events in both RansacExecution modes; the two modes' fits must be
   bitwise identical (checked every measurement; VP_ECUDA otherwise). Rows:
   10 % trimmed means and medians over trials. */
typedef struct {
  const int32_t* cluster_counts;
  int32_t n_counts;
  int32_t trials;
  int32_t points_min, points_max;
  uint64_t seed;
  int32_t iterations;
  double inlier_eps;
  int32_t device;
} vp_ablation_config;
typedef struct {
  int32_t clusters, trials;
  double parallel_ms, serial_ms, parallel_median_ms, serial_median_ms;
} vp_ablation_row;
/* AblationConfig defaults (pipeline.hpp:65-74): counts {1,2,4,8,16} need the
   caller's array; trials 1000, M in [10000, 30000], seed 1234, 100
   iterations, eps 0.01. */
void vp_default_ablation_config(vp_ablation_config* c);
int vp_run_ablation(const vp_ablation_config* c, vp_ablation_row* rows);
/* The synthetic clusters of one (trial, count): *m points per cluster,
   points = count * m * 3 doubles (host, free with vp_free). */
int vp_ablation_clusters(const vp_ablation_config* c, int32_t trial, int32_t count, int32_t* m,
                         double** points);
/* write_ablation_csv (pipeline.cpp:383-396). */
int vp_write_ablation_csv(const char* path, const vp_ablation_row* rows, size_t n);

/* label_components algorithm (identical labels): 0 = min-neighbour hooking +
   forward-window unions (default), 1 = neighbour-sampling unions + whole-window
   unions outside the sampled giant component, 2 = hooking + the same giant
   skip. Set before creating pipelines (captured graphs keep their variant). */
int vp_set_ccl_mode(int mode);
/* Count of this library's kernel launches since process start (bench evidence). */
uint64_t vp_kernel_launch_count(void);
/* Per-kernel CUDA-event timing of every launch (serialising; for profiling
   runs only). vp_profile_read returns the kernel count and fills up to cap. */
void vp_profile_enable(int on);
int vp_profile_read(const char** names, double* ms, uint64_t* calls, int cap);

#ifdef __cplusplus
}
#endif
#endif
