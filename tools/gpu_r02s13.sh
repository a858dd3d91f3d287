#!/bin/bash
# fused camera pass: its parity tests, the camera tests, e2e_render A/B (fused vs two launches) and the default line
TAG=${1:-r02s13}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_cuda_parity.py -m gpu -q -k "camera" > $OUT/pytest_cam.log 2>&1; echo "rc=$?" >> $OUT/pytest_cam.log
timeout 600 python - > $OUT/render_ab.jsonl 2> $OUT/render_ab.err <<'PY'
import json, time, torch, sys
sys.path.insert(0, ".")
import bench
from paper_2103_02309_b200.trace import TraceResult, trace_camera
from paper_2103_02309_b200.device import device_mesh
cfg = bench.CONFIGS[2]
sc = bench.build_scene(cfg)
mesh = sc.mesh if hasattr(sc, "mesh") else sc[0]
W, H = cfg["width"], cfg["height"]
cam = bench.camera_of(cfg, 0)
dm = device_mesh(mesh, device=0, layout=cfg["layout"])
hres = TraceResult(*[torch.empty(W * H, dtype=dt).pin_memory() for dt in
                     (torch.uint8, torch.int32, torch.int32, torch.float64, torch.int32, torch.int32, torch.int32)])
_, ct = trace_camera(dm, cam, W, H, out=hres)
for rnd in range(3):
    for fused in (False, True):
        for _ in range(5):
            trace_camera(dm, cam, W, H, out=hres, cam_tet=ct, fused=fused); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            trace_camera(dm, cam, W, H, out=hres, cam_tet=ct, fused=fused); torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / 20 * 1e3
        print(json.dumps({"round": rnd, "fused": fused, "ms": round(ms, 4), "Mrays_s": round(W * H / ms / 1e3, 1)}), flush=True)
PY
timeout 1200 python bench.py --steps 20 --warmup 5 > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err
echo done
