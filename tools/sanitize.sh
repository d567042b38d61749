# compute-sanitizer runs (memcheck / racecheck / synccheck / initcheck) over
# small end-to-end workloads: the smoke stream, a pipelined C2 run of 4
# frames, the slab path with 3 virtual slabs, the device frame source.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
cat > gpurun_out/san_work.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import __graft_entry__ as ge
from paper_2510_01592_b200 import native, scenes, slabs
ge.smoke()
w = scenes.workload("c2", frames=4)
pl = native.Pipeline(w.resolution, (300, 300, 300), w.frames[0].translation, native.default_params(seed=w.seed))
pl.run(w.frames)
w4 = scenes.workload("c4", frames=2)  # incoherent rays: the brick-mask walk
pl4 = native.Pipeline(w4.resolution, (300, 300, 200), w4.frames[0].translation, native.default_params(seed=w4.seed))
pl4.run(w4.frames)
ss = [slabs.Slab(0.01, (300, 200, 150), (0.0, 0.0, 0.5), a, b) for a, b in [(0, 100), (100, 103), (103, 300)]]
comm = slabs.LocalComm(3)
for f in scenes.stair_frames(3):
    slabs.slab_frame(ss, comm, torch.from_numpy(np.ascontiguousarray(f.points)).cuda(), f.rotation, f.translation,
                     native.default_params(seed=5))
ws = scenes.workload_spec("c2", 1)
src = scenes.DeviceFrameSource(ws.scene, ws.sensor, ws.seed)
src.render(ws.poses[0], 0)
# round 2: the library-orchestrated slab frame (one host thread per slab)
ss2 = [slabs.Slab(0.01, (300, 200, 150), (0.0, 0.0, 0.5), a, b) for a, b in [(0, 120), (120, 300)]]
for f in scenes.stair_frames(2):
    slabs.frame_local(ss2, f.points, f.rotation, f.translation, native.default_params(seed=5))
# more clusters than the initial capacity (the cluster buffers grow, the chain re-runs)
from test_gpu_parity import many_patch_frame
f = many_patch_frame()
p = native.default_params(seed=3, refine_exact=False, min_area=1e-6)
p.seg.min_cluster_size = 5
pm = native.Pipeline(0.01, (400, 400, 120), f.translation, p)
pm.frame(f.points, f.rotation, f.translation)
# round 2: fits above the wide-pass threshold (k_poly_wide_ext / _keep), lattice ties
g = np.stack(np.meshgrid(np.arange(150), np.arange(140), indexing="ij"), -1).reshape(-1, 2) * 0.01
lat = np.c_[g, np.zeros(len(g))]
native.make_polygons([dict(normal=np.array([0, 0, 1.0]), offset=0.0), dict(normal=np.array([0.3, -0.2, 0.9]) / np.linalg.norm([0.3, -0.2, 0.9]), offset=0.1)],
                     [lat, np.random.default_rng(1).normal(size=(40000, 3))])
print("sanitizer workload done")
PY
for tool in memcheck racecheck synccheck; do
  VP_NO_GRAPH=1 timeout 1500 $S --tool $tool --print-limit 20 python gpurun_out/san_work.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_$tool.log
done
for f in gpurun_out/san_*.log; do tail -n 4 $f; done
