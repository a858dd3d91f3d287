"""Multi-GPU tracing: image tiles sharded across ranks, mesh replicated,
one NCCL gather of the hit buffers at the end.

Rays are independent, so the path partitions with no exchange until the
frame is assembled.  The image is cut into 16x16 tiles
in the reference renderer's order (row-major over tile origins,
render.py:496-514); tile k of the job goes to rank k mod world (interleaved,
so uneven per-tile cost spreads evenly).  A job may stack several frames;
tiles are then numbered frame-major.  Each rank traces its shard with the
mesh resident in its own HBM, then ``gather_hits`` moves every rank's hit
records to the root in one collective.
"""

from __future__ import annotations

import numpy as np


def tile_origins(width: int, height: int, tile: int = 16):
    """(x0, y0, x1, y1) per tile, row-major over tile origins (render.py:496-514)."""
    out = []
    for y0 in range(0, height, tile):
        for x0 in range(0, width, tile):
            out.append((x0, y0, min(width, x0 + tile), min(height, y0 + tile)))
    return out


def shard_pixels(width: int, height: int, rank: int, world: int, tile: int = 16, frames: int = 1) -> np.ndarray:
    """Global ray indices (frame * W * H + y * W + x) owned by ``rank``:
    tiles k = rank, rank + world, ... of the frame-major tile sequence,
    pixels row-major within each tile."""
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} not in [0, {world})")
    tiles = tile_origins(width, height, tile)
    parts = []
    for k in range(rank, len(tiles) * frames, world):
        f, t = divmod(k, len(tiles))
        x0, y0, x1, y1 = tiles[t]
        ys, xs = np.mgrid[y0:y1, x0:x1]
        parts.append(f * width * height + ys.ravel() * width + xs.ravel())
    if not parts:
        return np.zeros(0, dtype=np.int64)
    return np.concatenate(parts).astype(np.int64)


# Packed hit record moved by the gather: idx i64, t f64, cf/tet/visited/
# triangle/tet_back i32, status u8 (+3 pad) = 40 bytes per ray.
RECORD_BYTES = 40


def pack_hits(idx, status, cf, tet, visited, triangle, t, tet_back):
    """Pack per-ray outputs (torch tensors on one device) into a uint8 (n, 40) buffer."""
    import torch

    n = idx.numel()
    buf = torch.zeros((n, RECORD_BYTES), dtype=torch.uint8, device=idx.device)
    buf[:, 0:8] = idx.to(torch.int64).contiguous().view(torch.uint8).view(n, 8)
    buf[:, 8:16] = t.to(torch.float64).contiguous().view(torch.uint8).view(n, 8)
    for k, a in enumerate((cf, tet, visited, triangle, tet_back)):
        buf[:, 16 + 4 * k : 20 + 4 * k] = a.to(torch.int32).contiguous().view(torch.uint8).view(n, 4)
    buf[:, 36] = status.to(torch.uint8)
    return buf


def unpack_hits(buf):
    """Inverse of pack_hits: dict of torch tensors."""
    import torch

    n = buf.shape[0]
    b = buf.contiguous()
    out = {
        "idx": b[:, 0:8].contiguous().view(torch.int64).view(n),
        "t": b[:, 8:16].contiguous().view(torch.float64).view(n),
    }
    for k, name in enumerate(("cf", "tet", "visited", "triangle", "tet_back")):
        out[name] = b[:, 16 + 4 * k : 20 + 4 * k].contiguous().view(torch.int32).view(n)
    out["status"] = b[:, 36].contiguous()
    return out


def gather_hits(packed, total: int, root: int = 0, group=None):
    """Gather every rank's packed hits to ``root`` with one collective and
    scatter them into full-job arrays (by global ray index).

    Returns the dict of full arrays on root, None elsewhere.  Shards may
    differ in length: lengths are exchanged first and buffers padded.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if dist.get_backend(group) == "gloo":  # gloo collectives run on host tensors
        packed = packed.cpu()
    dev = packed.device
    n = torch.tensor([packed.shape[0]], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(sizes) if sizes else 0
    pad = torch.zeros((cap, RECORD_BYTES), dtype=torch.uint8, device=dev)
    pad[: packed.shape[0]] = packed
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == root else None
    dist.gather(pad, gather_list=bufs, dst=dist.get_global_rank(group, root) if group is not None else root,
                group=group)
    if rank != root:
        return None
    recs = unpack_hits(torch.cat([b[:s] for b, s in zip(bufs, sizes)]))
    idx = recs.pop("idx")
    full = {}
    for name, a in recs.items():
        fill = {"t": float("inf"), "status": 0, "visited": 0}.get(name, -1)
        dst = torch.full((total,), fill, dtype=a.dtype, device=dev)
        dst[idx] = a
        full[name] = dst
    return full
