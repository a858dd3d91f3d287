"""Device-resident tracing API: ``trace(mesh, origins, dirs, start)``.

PyTorch tensors are the ray and hit buffers (plumbing only): inputs are
CUDA tensors already in HBM, outputs are allocated on the same device, and
the launch is enqueued on the current torch stream with no host sync.  This
is the call the benchmark's device-side number measures; ``trace_host`` is
the end-to-end form (pinned host buffers, H2D + kernel + D2H).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
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
          layout: str | None = None, schedule: str | int = "auto",
          block_order: torch.Tensor | None = None) -> TraceResult:
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

    ``block_order`` (int32 CUDA tensor, a permutation of the batch's blocks of
    ``block_size()`` rays): launch the blocks in this order, results in place
    (tb_cast_rays_ordered).  ``longest_first(visited)`` builds it from a
    previous, similar batch's walk lengths -- the next frame of an animation:
    long blocks first leaves no late long walk to idle the SMs at the end of
    the launch (r02: config 2 frames +19-20 % ordered by the previous frame).
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
    if block_order is not None:
        if sctp or schedule not in ("auto", "lane", 0, 1):
            raise ValueError("block_order applies to the 2-D walk's one-ray-per-lane schedule")
        if block_order.dtype != torch.int32 or block_order.device != origins.device:
            raise ValueError("block_order must be an int32 tensor on the rays' device")
        bo = block_order.contiguous()
        check(lib.tb_cast_rays_ordered(dm.handle, n, addr(origins), addr(dirs), addr(start), addr(bo), bo.numel(),
                                       addr(res.status), addr(res.cf), addr(res.tet), addr(res.visited), tri, tt,
                                       back, s), "tb_cast_rays_ordered")
    elif sctp:
        check(lib.tb_sctp_cast_rays(*ins, s), "tb_sctp_cast_rays")
    else:
        mode = SCHEDULES[schedule] if isinstance(schedule, str) else int(schedule)
        check(lib.tb_cast_rays_sched(*ins, mode, s), "tb_cast_rays_sched")
    return res


def block_size() -> int:
    """Rays per block of the cast kernels (the unit of ``block_order``)."""
    return int(lib.tb_cast_block_size())


def longest_first(visited: torch.Tensor, stream=None) -> torch.Tensor:
    """Launch order for ``trace(block_order=...)``: the blocks of a batch,
    longest walk first, from the per-ray visited counts of a previous,
    similar batch (same ray layout -- e.g. the previous frame).  A block
    holds its slot until its slowest warp ends, so the key is the block's
    maximum (tb_block_order: two small kernels on the device, no host
    round trip; blocks with equal keys run in no particular order -- which
    changes where a block runs, never its results)."""
    b = block_size()
    v = visited.to(torch.int32).contiguous()
    n = v.numel()
    nb = (n + b - 1) // b
    order = torch.empty(nb, dtype=torch.int32, device=v.device)
    s = (stream or torch.cuda.current_stream(v.device)).cuda_stream
    with torch.cuda.device(v.device):
        check(lib.tb_block_order(n, addr(v), addr(order), nb, s), "tb_block_order")
    return order


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
                 stream=None, sctp: bool = False, layout: str | None = None, cam_tet: int | None = None,
                 block_order: torch.Tensor | None = None, fused: bool = True):
    """Render-style primary pass entirely on the device: locate the camera
    (render.py:478-482; skipped when ``cam_tet`` is given), generate the
    frame's rays in HBM, trace.  ``out`` may hold pinned host tensors: the
    kernel then writes the hits straight to host memory over PCIe (mapped
    pinned memory under UVA), overlapping the copy with the walk.
    ``block_order``: see ``trace`` (for an animation, ``longest_first`` of
    the previous frame's ``visited``; the pixel order is row-major here).
    ``fused`` (2-D walk without a block order): one launch that forms each
    pixel's ray in registers and walks it (tb_trace_camera) -- no rays in
    HBM; bit-identical to the two-launch path (fused=False).
    Returns (TraceResult, cam_tet)."""
    dm = device_mesh(mesh, device=None if device is None else torch.device(device).index, layout=layout)
    dev = torch.device("cuda", dm.device)
    if cam_tet is None:
        q = torch.tensor([camera["position"]], dtype=torch.float64, device=dev)
        cam, _ = locate(dm, q, torch.tensor([dm.source_tet], dtype=torch.int32, device=dev))
        cam_tet = int(cam.item())
        if cam_tet < 0:
            raise ValueError("camera is outside the tetrahedralized volume")
    if fused and not sctp and block_order is None:
        from .scenes import camera_frame

        frame = np.ascontiguousarray(camera_frame(camera["position"], camera["look_at"],
                                                  camera.get("up", (0.0, 1.0, 0.0)), camera.get("fov", 68.0), width,
                                                  height), dtype=np.float64)
        res = out if out is not None else empty_result(width * height, dev)
        if len(res) != width * height:
            raise ValueError(f"out holds {len(res)} rays, the frame {width * height}")
        s = (stream or torch.cuda.current_stream(dev)).cuda_stream
        with torch.cuda.device(dev):
            check(lib.tb_trace_camera(dm.handle, width, height, frame.ctypes.data, int(cam_tet), addr(res.status),
                                      addr(res.cf), addr(res.tet), addr(res.visited), addr(res.triangle),
                                      addr(res.t), addr(res.tet_back), s), "tb_trace_camera")
        return res, cam_tet
    o, d = camera_rays_device(camera, width, height, dev, stream=stream)
    start = torch.full((o.shape[0],), cam_tet, dtype=torch.int32, device=dev)
    return trace(dm, o, d, start, out=out, stream=stream, sctp=sctp, block_order=block_order), cam_tet


def locate(mesh, q: torch.Tensor, hints: torch.Tensor, *, stream=None):
    """Device point location: (tet, visited) int32 tensors."""
    dm = device_mesh(mesh, device=q.device.index)
    n = hints.numel()
    tet = torch.empty(n, dtype=torch.int32, device=q.device)
    vis = torch.empty(n, dtype=torch.int32, device=q.device)
    s = (stream or torch.cuda.current_stream(q.device)).cuda_stream
    check(lib.tb_locate_points(dm.handle, n, addr(q), addr(hints), addr(tet), addr(vis), s), "tb_locate_points")
    return tet, vis
