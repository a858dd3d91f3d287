"""Device-resident tracing API: ``trace(mesh, origins, dirs, start)``.

PyTorch tensors are the ray and hit buffers (plumbing only): inputs are
CUDA tensors already in HBM, outputs are allocated on the same device, and
the launch is enqueued on the current torch stream with no host sync.  This
is the call the benchmark's device-side number measures; ``trace_host`` is
the end-to-end form (pinned host buffers, H2D + kernel + D2H).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from ._lib import SCHEDULES, addr, check, lib
from .device import DeviceMesh, device_mesh


@dataclass
class TraceResult:
    status: torch.Tensor  # (n,) uint8   0 miss / 1 hit / 2 cycle guard
    cf: torch.Tensor  # (n,) int32   constrained face, -1 unless hit
    triangle: torch.Tensor  # (n,) int32   scene triangle, -1 on miss
    t: torch.Tensor  # (n,) float64 hit parameter, +inf on miss
    tet: torch.Tensor  # (n,) int32   terminating (front) tet
    tet_back: torch.Tensor  # (n,) int32   tet behind the hit face, -1 on hull
    visited: torch.Tensor  # (n,) int32   tets visited (start counts 1)

    def __len__(self) -> int:
        return self.status.numel()


def empty_result(n: int, device) -> TraceResult:
    dev = torch.device(device)
    return TraceResult(
        status=torch.empty(n, dtype=torch.uint8, device=dev),
        cf=torch.empty(n, dtype=torch.int32, device=dev),
        triangle=torch.empty(n, dtype=torch.int32, device=dev),
        t=torch.empty(n, dtype=torch.float64, device=dev),
        tet=torch.empty(n, dtype=torch.int32, device=dev),
        tet_back=torch.empty(n, dtype=torch.int32, device=dev),
        visited=torch.empty(n, dtype=torch.int32, device=dev),
    )


def _check_inputs(dm: DeviceMesh, origins, dirs, start):
    n = start.numel()
    for name, x, dt, shape in (("origins", origins, torch.float32, (n, 3)), ("dirs", dirs, torch.float32, (n, 3)),
                               ("start", start, torch.int32, (n,))):
        if x.dtype != dt or tuple(x.shape) != shape or not x.is_contiguous():
            raise ValueError(f"{name} must be a contiguous {dt} tensor of shape {shape}")
        if x.device.type != "cuda" or x.device.index != dm.device:
            raise ValueError(f"{name} must live on cuda:{dm.device}")
    return n


def trace(mesh, origins: torch.Tensor, dirs: torch.Tensor, start: torch.Tensor, *, out: TraceResult | None = None,
          stream: torch.cuda.Stream | None = None, epilogue: bool = True, sctp: bool = False,
          layout: str | None = None, schedule: str | int = "auto") -> TraceResult:
    """Trace rays on the GPU; returns hit triangle id, t and terminating tet.

    ``sctp=True`` runs the fp64 scalar-triple-product fallback walk instead
    of the 2-D modified-basis walk.  ``schedule`` maps rays to lanes (results
    are identical either way): "lane" suits coherent primaries, "binned"
    (stable counting sort by direction cell -- 96 cube-map cells -- then
    the walk in binned order) incoherent batches such as diffuse
    secondaries (r01: +41 % on config 4), "compact" block compaction
    (kept for comparison); "auto" uses the process-wide setting (default:
    "lane" -- deciding from device-resident start tets would need a host
    round trip).  Start tets
    are not range-checked here (device inputs stay on the device);
    ``kernels.cast_rays`` checks them.
    """
    dm = device_mesh(mesh, device=origins.device.index, layout=layout)
    n = _check_inputs(dm, origins, dirs, start)
    res = out if out is not None else empty_result(n, origins.device)
    s = (stream or torch.cuda.current_stream(origins.device)).cuda_stream
    tri = addr(res.triangle) if epilogue else None
    tt = addr(res.t) if epilogue else None
    back = addr(res.tet_back) if epilogue else None
    ins = (dm.handle, n, addr(origins), addr(dirs), addr(start), addr(res.status), addr(res.cf), addr(res.tet),
           addr(res.visited), tri, tt, back)
    if sctp:
        check(lib.tb_sctp_cast_rays(*ins, s), "tb_sctp_cast_rays")
    else:
        mode = SCHEDULES[schedule] if isinstance(schedule, str) else int(schedule)
        check(lib.tb_cast_rays_sched(*ins, mode, s), "tb_cast_rays_sched")
    return res


def camera_rays_device(camera: dict, width: int, height: int, device, pixels: torch.Tensor | None = None,
                       stream=None):
    """Primary rays generated in HBM (bit-identical to scenes.camera_rays):
    (o, d) float32 (n, 3) CUDA tensors, row-major pixels or the given ids."""
    from .scenes import camera_frame

    dev = torch.device(device)
    frame = torch.from_numpy(camera_frame(camera["position"], camera["look_at"], camera.get("up", (0.0, 1.0, 0.0)),
                                          camera.get("fov", 68.0), width, height)).to(dev)
    n = pixels.numel() if pixels is not None else width * height
    o = torch.empty((n, 3), dtype=torch.float32, device=dev)
    d = torch.empty((n, 3), dtype=torch.float32, device=dev)
    s = (stream or torch.cuda.current_stream(dev)).cuda_stream
    with torch.cuda.device(dev):
        check(lib.tb_camera_rays(width, height, addr(frame), addr(pixels), n, addr(o), addr(d), s), "tb_camera_rays")
    return o, d


def trace_camera(mesh, camera: dict, width: int, height: int, *, device=None, out: TraceResult | None = None,
                 stream=None, sctp: bool = False, layout: str | None = None, cam_tet: int | None = None):
    """Render-style primary pass entirely on the device: locate the camera
    (render.py:478-482; skipped when ``cam_tet`` is given), generate the
    frame's rays in HBM, trace.  ``out`` may hold pinned host tensors: the
    kernel then writes the hits straight to host memory over PCIe (mapped
    pinned memory under UVA), overlapping the copy with the walk.
    Returns (TraceResult, cam_tet)."""
    dm = device_mesh(mesh, device=None if device is None else torch.device(device).index, layout=layout)
    dev = torch.device("cuda", dm.device)
    if cam_tet is None:
        q = torch.tensor([camera["position"]], dtype=torch.float64, device=dev)
        cam, _ = locate(dm, q, torch.tensor([dm.source_tet], dtype=torch.int32, device=dev))
        cam_tet = int(cam.item())
        if cam_tet < 0:
            raise ValueError("camera is outside the tetrahedralized volume")
    o, d = camera_rays_device(camera, width, height, dev, stream=stream)
    start = torch.full((o.shape[0],), cam_tet, dtype=torch.int32, device=dev)
    return trace(dm, o, d, start, out=out, stream=stream, sctp=sctp), cam_tet


def locate(mesh, q: torch.Tensor, hints: torch.Tensor, *, stream=None):
    """Device point location: (tet, visited) int32 tensors."""
    dm = device_mesh(mesh, device=q.device.index)
    n = hints.numel()
    tet = torch.empty(n, dtype=torch.int32, device=q.device)
    vis = torch.empty(n, dtype=torch.int32, device=q.device)
    s = (stream or torch.cuda.current_stream(q.device)).cuda_stream
    check(lib.tb_locate_points(dm.handle, n, addr(q), addr(hints), addr(tet), addr(vis), s), "tb_locate_points")
    return tet, vis
