/* Per-frame stage trace: the byte format shared by the CPU oracle
 * (oracle/voxplane_oracle.c), the compiled reference (oracle/_ref, built from
 * /root/reference/proj/core/src by oracle/Makefile) and the B200 library
 * (vp_pipeline_frame_trace), so parity tests compare every stage of
 * pipeline.cpp:199-213 / :43-85 field by field.
 *
 * Little-endian, no padding; sections in this order:
 *   "VPTR" u32 version(=1) u32 frame_index
 *   mapping:  u64 clear.cleared u64 clear.freed u64 upd.touched u64 upd.discarded
 *             u8 recentered i32 shift[3] u64 dropped f64 origin[3] u64 occupied_count
 *   occupied: u64 V; i32 idx[V*3] f64 mean[V*3] u32 count[V] u8 status[V]
 *             (status as stored before classify_steppable of this frame)
 *   normals:  f64 normal[V*3] i32 neighbor_count[V] u8 valid[V]
 *             (angle_to_up_deg is NOT traced: it is acos() of normal.up, which the
 *              host recomputes with libm; the device only evaluates the predicate)
 *   steppable:u64 S; i32 idx[S*3] f64 mean[S*3] f64 normal[S*3]
 *   labels:   i32 label[S]
 *   clusters: u64 K; per cluster i32 label, u64 size   (after filter_clusters)
 *   fits:     u64 skipped_small u64 unfit u64 F; per fit
 *             f64 normal[3] f64 offset i32 inlier_count i32 label u64 M f64 inliers[M*3]
 *   refined:  per fit f64 normal[3] f64 offset (equals the fit when refine is off)
 *   polygons: u64 P; per polygon f64 normal[3] f64 offset i32 inlier_count i32 label
 *             u64 nv f64 v2d[nv*2] f64 v3d[nv*3] f64 area
 * When the grid has no occupied voxel the segmentation sections are empty
 * (pipeline.cpp:48 returns before estimate_normals).
 */
#ifndef VOXPLANE_TRACE_H
#define VOXPLANE_TRACE_H
#define VP_TRACE_VERSION 1u
#endif
