/* Synthetic frame source for the benchmarks and parity tests.
 *
 * Restates the reference's analytic scene simulator
 * (/root/reference/proj/core/src/scene_sim.cpp) and default trajectories
 * (pipeline.cpp:89-155) so the GPU box can generate the exact frames the
 * reference would render (tests pin this against oracle/_ref's render_frame
 * byte for byte). Host C++; not part of the timed path.
 */
#ifndef VOXPLANE_SCENE_H
#define VOXPLANE_SCENE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Box (scene_sim.hpp:12-15) */
typedef struct {
  double min[3];
  double max[3];
} vp_box;

/* Rect (scene_sim.hpp:19-23): pose rotation row-major, translation, half extents */
typedef struct {
  double R[9];
  double t[3];
  double half_u, half_v;
} vp_rect;

/* SensorSpec (scene_sim.hpp:54-67); kind 0 = pinhole depth, 1 = ray pattern */
typedef struct {
  int32_t kind;
  int32_t width, height;
  double hfov_deg, vfov_deg;
  const float* pattern; /* npattern x 3, sensor-frame directions */
  uint64_t npattern;
  double rate_hz;
  double max_range;
  double noise_sigma;
} vp_sensor;

/* build_scene (scene_sim.cpp:43-114) for SceneKind 0 Stair5, 1 SingleStage,
   2 Overhang, 3 SmallObstacle with SceneParams defaults. Capacities: 16 each. */
int vp_stock_scene(int kind, vp_box* boxes, size_t* nb, vp_rect* rects, size_t* nr);

/* default_trajectory (pipeline.cpp:89-155) with SceneParams defaults; poses
   are 12 doubles (R row-major, t). Returns the pose count (<= frames). */
int vp_default_trajectory(int kind, int frames, double rate_hz, double* poses);

/* scripted_trajectory (scene_sim.cpp:252-298); kind 0 Straight, 1 Orbit,
   2 StairAscent. spec = {duration, rate, start xyz, end xyz, pitch0, pitch1,
   center xyz, radius, height, start_angle, revolutions, rise, run, x0}. */
int vp_scripted_trajectory(int kind, const double spec[21], double* poses, int cap);

/* make_spherical_pattern / make_rosette_pattern (scene_sim.cpp:161-184) */
int vp_spherical_pattern(int n, float* out);
int vp_rosette_pattern(int n, double cone_deg, double freq_ratio, float* out);

/* render_frame (scene_sim.cpp:186-236): points (library-allocated, free with
   vp_free) in ray order, misses dropped; the returned pose is quantised
   through f32 (frame_io.cpp:64-72). threads <= 0: hardware concurrency. */
int vp_render_frame(const vp_box* boxes, size_t nb, const vp_rect* rects, size_t nr,
                    const vp_sensor* sensor, const double R[9], const double t[3], uint64_t seed,
                    uint64_t frame_index, int threads, float** points, uint64_t* n,
                    double qR[9], double qt[3]);

/* build_scene's ground-truth regions (scene_sim.cpp:23-30, 43-114) for a
   stock SceneKind: per region the plane (normal xyz, offset; plane_through)
   and its 4 corners (12 doubles); make_polygon of the corners
   (vp_make_polygons) gives the truth polygon. Capacity 16 regions. */
int vp_scene_truth(int kind, double* planes, double* corners, size_t* n);

/* quantize_pose (frame_io.cpp:64-72) + the orthonormality check of
   render_frame (scene_sim.cpp:188-190); returns VP_EINVAL (voxplane_b200.h) if invalid. */
int vp_quantize_pose(const double R[9], const double t[3], double qR[9], double qt[3]);

/* ---- device frame source ---------------------------
   render_frame on the GPU: one thread per ray (pinhole pixel or pattern
   direction), the reference's ray/box and ray/rect arithmetic in FP64
   without FMA, CounterRng(seed, frame, ray) range noise, and an ordered
   compaction of the hits (misses dropped, ray order kept). The frame stays
   in device memory (feed it to vp_pipeline_frame_device / slabs). The noise
   uses the device log/cos (<= 1-2 ulp from glibc): points equal the host
   source's bytes unless such an ulp survives the f32 rounding
   (tests/test_frame_source.py measures it). */
typedef struct vp_frame_source vp_frame_source;
int vp_frame_source_create(const vp_box* boxes, size_t nb, const vp_rect* rects, size_t nr,
                           const vp_sensor* sensor, uint64_t seed, int device, vp_frame_source** out);
void vp_frame_source_destroy(vp_frame_source* s);
/* The cudaStream_t the source renders on. */
void* vp_frame_source_stream(vp_frame_source* s);
/* Render frame `frame_index` at pose (R, t): xyz_dev = device points (n x 3
   f32, valid until the next render), qR/qt = the f32-quantised pose. */
int vp_frame_source_render(vp_frame_source* s, const double R[9], const double t[3], uint64_t frame_index,
                           const float** xyz_dev, uint64_t* n, double qR[9], double qt[3]);

#ifdef __cplusplus
}
#endif
#endif
