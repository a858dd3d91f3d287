#!/bin/bash
# ncu of the fused render-style pass (camera_cast_kernel<20>, config 2, hits into pinned host memory)
TAG=${1:-r02s15}; OUT=gpurun_out/$TAG; mkdir -p $OUT
cat > /tmp/cam_probe.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2103_02309_b200.trace import TraceResult, trace_camera
from paper_2103_02309_b200.device import device_mesh
cfg = bench.CONFIGS[2]
sc = bench.build_scene(cfg)
W, H = cfg["width"], cfg["height"]
cam = bench.camera_of(cfg, 0)
dm = device_mesh(sc.mesh, device=0, layout=cfg["layout"])
hres = TraceResult(*[torch.empty(W * H, dtype=dt).pin_memory() for dt in
                     (torch.uint8, torch.int32, torch.int32, torch.float64, torch.int32, torch.int32, torch.int32)])
_, ct = trace_camera(dm, cam, W, H, out=hres)
for _ in range(4):
    trace_camera(dm, cam, W, H, out=hres, cam_tet=ct)
torch.cuda.synchronize()
print("ok")
PY
timeout 600 python /tmp/cam_probe.py > $OUT/probe.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:camera_cast_kernel -s 2 -c 1 -o $OUT/prof_cam \
    python /tmp/cam_probe.py > $OUT/ncu_cam.log 2>&1
echo done
