// Drop-in check #2: every remaining reference name of the hot path's API
// called the way a reference user calls it, with the results
// written to a record file that tests/test_gpu_dropin.py compares against the
// compiled reference (oracle/_ref ref_* wrappers):
//   CounterRng (rng.hpp), jacobi_eigen_sym3 (jacobi.hpp), hull_filter /
//   monotone_chain / convex_hull (polygonize.hpp), label_components on an
//   explicit adjacency (segmentation.hpp), quantize_pose / write_frames_binary
//   / read_frames_binary / write_frames_text / read_frames_text (frame_io.hpp),
//   read_polygons (polygon_io.hpp), replay_pipeline -> run_frames
//   (pipeline.hpp) with per-frame polygons, timing CSV and the IoU report,
//   and the height-map baseline through run_frames.
// Usage: drop_in_api records.bin tiny_frames.bin truth.txt baseline_frames.bin out_dir
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "voxplane/frame_io.hpp"
#include "voxplane/jacobi.hpp"
#include "voxplane/pipeline.hpp"
#include "voxplane/polygon_io.hpp"
#include "voxplane/polygonize.hpp"
#include "voxplane/rng.hpp"
#include "voxplane/segmentation.hpp"

using namespace voxplane;

namespace {
FILE* g_out = nullptr;
template <typename T>
void rec(const std::string& tag, const std::vector<T>& v) {
  const uint32_t tl = static_cast<uint32_t>(tag.size());
  const uint64_t nb = v.size() * sizeof(T);
  std::fwrite(&tl, 4, 1, g_out);
  std::fwrite(tag.data(), 1, tl, g_out);
  std::fwrite(&nb, 8, 1, g_out);
  if (nb) std::fwrite(v.data(), 1, nb, g_out);
}
void require(bool ok, const char* what) {
  if (!ok) throw std::runtime_error(what);
}
}  // namespace

int main(int argc, char** argv) {
  if (argc < 6) {
    std::fprintf(stderr, "usage: %s records.bin tiny_frames.bin truth.txt baseline_frames.bin out_dir\n", argv[0]);
    return 2;
  }
  g_out = std::fopen(argv[1], "wb");
  const std::string out = argv[5];
  try {
    // -- CounterRng: four fresh streams keyed (2025, 7, 3)
    {
      std::vector<uint64_t> raw;
      std::vector<double> uni, nrm;
      std::vector<uint32_t> below;
      CounterRng a(2025, 7, 3), b(2025, 7, 3), c(2025, 7, 3), d(2025, 7, 3);
      for (int i = 0; i < 257; ++i) {
        raw.push_back(a.next_u64());
        uni.push_back(b.uniform());
        below.push_back(c.below(1000003u));
        nrm.push_back(d.normal());
      }
      rec("rng_raw", raw);
      rec("rng_uniform", uni);
      rec("rng_below", below);
      rec("rng_normal", nrm);
    }
    // -- jacobi_eigen_sym3: random symmetric, diagonal, repeated, rank-1 matrices
    {
      CounterRng r(11);
      std::vector<Mat3> ms;
      for (int i = 0; i < 200; ++i) {
        Mat3 m;
        for (int p = 0; p < 3; ++p)
          for (int q = p; q < 3; ++q) m(p, q) = m(q, p) = r.uniform(-1.0, 1.0) * (i % 7 == 0 ? 1e-6 : 1.0);
        ms.push_back(m);
      }
      Mat3 dgl = Mat3::Zero();
      dgl(0, 0) = 3.0;
      dgl(1, 1) = 1.0;
      dgl(2, 2) = 2.0;
      ms.push_back(dgl);
      ms.push_back(Mat3::Identity());
      const Vec3 u(0.3, -0.5, 0.8);
      ms.push_back(u * u.transpose());
      std::vector<double> a, vals, vecs;
      const std::vector<EigenSym3> batch = jacobi_eigen_sym3(ms);
      for (size_t i = 0; i < ms.size(); ++i) {
        const EigenSym3 one = jacobi_eigen_sym3(ms[i]);  // single-matrix overload
        for (int k = 0; k < 3; ++k)
          require(one.eigenvalues[k] == batch[i].eigenvalues[k], "jacobi: single != batched");
        for (int p = 0; p < 3; ++p)
          for (int q = 0; q < 3; ++q) a.push_back(ms[i](p, q));
        for (int k = 0; k < 3; ++k) vals.push_back(batch[i].eigenvalues[k]);
        for (int k = 0; k < 3; ++k)
          for (int p = 0; p < 3; ++p) vecs.push_back(batch[i].eigenvectors(p, k));
      }
      rec("jac_a", a);
      rec("jac_vals", vals);
      rec("jac_vecs", vecs);
    }
    // -- hulls: discs, grids with duplicates, collinear sets, tiny sets
    {
      CounterRng r(5);
      const int sizes[] = {0, 1, 2, 3, 4, 5, 8, 17, 100, 1000, 3000, 20000};
      int set_id = 0;
      for (int n : sizes)
        for (int shape = 0; shape < 3; ++shape) {
          std::vector<Vec2> p;
          for (int i = 0; i < n; ++i) {
            if (shape == 0) {  // disc, points on a 1 mm lattice (ties and duplicates)
              double x, y;
              do {
                x = r.uniform(-1.0, 1.0);
                y = r.uniform(-1.0, 1.0);
              } while (x * x + y * y > 1.0);
              p.emplace_back(std::round(x * 1000.0) / 1000.0, std::round(y * 1000.0) / 1000.0);
            } else if (shape == 1) {  // square grid, every point twice
              const int s = static_cast<int>(std::sqrt(n / 2.0)) + 1;
              p.emplace_back(0.01 * ((i / 2) % s), 0.01 * ((i / 2) / s));
            } else {  // collinear (monotone_chain -> empty)
              p.emplace_back(0.5 * i, 0.25 * i - 1.0);
            }
          }
          std::vector<double> flat;
          for (const Vec2& q : p) flat.insert(flat.end(), {q.x(), q.y()});
          for (int dirs : {16, 8, 3, 0}) {
            std::vector<double> hf, mc, ch;
            for (const Vec2& q : hull_filter(p, dirs)) hf.insert(hf.end(), {q.x(), q.y()});
            for (const Vec2& q : convex_hull(p, dirs)) ch.insert(ch.end(), {q.x(), q.y()});
            const std::string id = std::to_string(set_id) + "_" + std::to_string(dirs);
            rec("hull_pts_" + id, flat);
            rec("hull_filter_" + id, hf);
            rec("hull_convex_" + id, ch);
            if (dirs == 16) {
              for (const Vec2& q : monotone_chain(p)) mc.insert(mc.end(), {q.x(), q.y()});
              rec("hull_chain_" + id, mc);
            }
          }
          ++set_id;
        }
    }
    // -- label_components(steppable, adjacency): random symmetric graphs
    {
      CounterRng r(9);
      for (int gi = 0; gi < 6; ++gi) {
        const int n = 50 + 300 * gi;
        std::vector<SteppablePoint> st(n);
        for (int i = 0; i < n; ++i) st[i].voxel = Vec3i(i, 0, 0);
        Adjacency adj(n);
        const int ne = n * (gi % 3 + 1) / 2;
        for (int e = 0; e < ne; ++e) {
          const int a = static_cast<int>(r.below(n)), b = static_cast<int>(r.below(n));
          if (a == b) continue;
          adj[a].push_back(b);
          adj[b].push_back(a);
        }
        for (auto& l : adj) std::sort(l.begin(), l.end());
        const ClusterSet set = label_components(st, adj);
        std::vector<uint64_t> rows{0};
        std::vector<int32_t> cols;
        for (const auto& l : adj) {
          cols.insert(cols.end(), l.begin(), l.end());
          rows.push_back(cols.size());
        }
        // clusters: ascending label, members ascending ordinal
        for (size_t k = 1; k < set.clusters.size(); ++k)
          require(set.clusters[k - 1].label < set.clusters[k].label, "clusters not in label order");
        size_t members = 0;
        for (const Cluster& c : set.clusters) members += c.members.size();
        require(members == static_cast<size_t>(n), "cluster members != n");
        rec("cc_rows_" + std::to_string(gi), rows);
        rec("cc_cols_" + std::to_string(gi), cols);
        rec("cc_labels_" + std::to_string(gi), set.labels);
      }
    }
    // -- frame formats: quantize_pose, binary and text round trips
    {
      std::vector<SensorFrame> frames = read_frames_binary(argv[2]);
      require(!frames.empty(), "no frames");
      Pose p;
      p.rotation = Mat3::Identity();
      p.translation = Vec3(0.1, 1.0 / 3.0, -2.0 / 7.0);
      const Pose q = quantize_pose(p);
      rec("quant_t", std::vector<double>{q.translation.x(), q.translation.y(), q.translation.z()});
      write_frames_binary(out + "/frames_rt.bin", frames);
      const std::vector<SensorFrame> back = read_frames_binary(out + "/frames_rt.bin");
      require(back.size() == frames.size(), "binary round trip: frame count");
      for (size_t k = 0; k < frames.size(); ++k) {
        require(back[k].points.size() == frames[k].points.size(), "binary round trip: points");
        for (size_t i = 0; i < frames[k].points.size(); ++i)
          require(back[k].points[i] == frames[k].points[i], "binary round trip: xyz");
        require(back[k].pose.translation == frames[k].pose.translation, "binary round trip: pose");
      }
      std::vector<SensorFrame> small(frames.begin(), frames.begin() + 1);
      small[0].points.resize(std::min<size_t>(small[0].points.size(), 500));
      write_frames_text(out + "/frames_rt.txt", small);
      const std::vector<SensorFrame> tback = read_frames_text(out + "/frames_rt.txt");
      require(tback.size() == 1 && tback[0].points.size() == small[0].points.size(), "text round trip");
      for (size_t i = 0; i < small[0].points.size(); ++i)
        require(tback[0].points[i] == small[0].points[i], "text round trip: xyz");
    }
    // -- replay_pipeline -> run_frames (test_pipeline.cpp tiny_config), truth file
    {
      PipelineConfig c = default_config();
      c.output.dir = out + "/replay";
      c.output.per_frame_polygons = true;
      c.output.dump_labels = true;
      c.grid_extent = Vec3i(140, 140, 140);
      c.run.seed = 77;
      c.ransac.seed = 77;
      c.refine_exact = true;
      const PipelineResult r = replay_pipeline(c, argv[2], argv[3]);
      require(r.iou.has_value(), "replay: no IoU report");
      require(r.frames_processed == r.timing.frames.size(), "timing rows");
      // read_polygons -> write_polygons reproduces the file
      write_polygons(out + "/replay/polygons_reread.txt", read_polygons(r.polygons_path));
      rec("replay_frames", std::vector<uint64_t>{r.frames_processed});
      std::vector<double> tm;
      for (const FrameTiming& f : r.timing.frames)
        tm.insert(tm.end(), {static_cast<double>(f.points), static_cast<double>(f.voxels),
                             static_cast<double>(f.clusters), f.total_ms});
      rec("replay_timing", tm);
    }
    // -- the height-map baseline through run_frames (test_pipeline.cpp:183-192)
    {
      PipelineConfig c = default_config();
      c.output.dir = out + "/baseline";
      c.grid_extent = Vec3i(140, 140, 140);
      c.ransac.seed = 77;
      c.run.baseline = true;
      c.refine_exact = true;
      run_frames(c, read_frames_binary(argv[4]), nullptr);
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "drop_in_api: %s\n", e.what());
    std::fclose(g_out);
    return 1;
  }
  std::fclose(g_out);
  std::printf("ok\n");
  return 0;
}
