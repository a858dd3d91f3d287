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


# Compact per-ray record of the per-frame gather: cf, tet, visited | status << 30,
# t (fp64 as two int32) = 20 bytes.  The root rebuilds the ray index from the
# static shard map and triangle / tet_back from cf with its own mesh copy.
COMPACT_WORDS = 5


def split_chunks(n: int, chunks: int) -> list[tuple[int, int]]:
    """Exactly ``chunks`` contiguous (start, stop) pieces of a rank's ray
    list (some empty when n < chunks), so every rank issues the same
    collectives."""
    chunks = max(1, chunks)
    edges = [n * k // chunks for k in range(chunks + 1)]
    return [(edges[k], edges[k + 1]) for k in range(chunks)]


class FrameGather:
    """Every frame's hits to the root, overlapped with tracing.

    All ranks know every rank's shard (``shard_pixels`` is deterministic, or
    ``index`` -- this rank's global ray indices when the job does not cover
    every slot -- is exchanged once at setup), so chunk sizes need no
    exchange per step; slots no rank traces keep the "no ray" values.  The caller traces chunk k of its shard and
    calls ``send(k, res_k)``: the chunk's compact records go out with an
    async ``dist.gather`` (NCCL runs it on its own stream, ordered after the
    trace), while the caller already traces chunk k+1 on its stream.
    ``finish()`` waits for the collectives and, on the root, scatters the
    records into full-frame arrays -- the same seven arrays a single-GPU
    trace of the whole job returns (the root recomputes triangle and
    tet_back from cf exactly as the trace epilogue does, batch.py:63-71).
    """

    def __init__(self, width, height, world, rank, frames, chunks, device, cf_triangle, cf_tets, root=0,
                 group=None, tile=16, index=None):
        import torch
        import torch.distributed as dist

        self.world, self.rank, self.root, self.group = world, rank, root, group
        self.device = torch.device(device)
        # gloo moves host tensors only: stage through host memory there
        self.comm = torch.device("cpu") if dist.get_backend(group) == "gloo" else self.device
        self.total = width * height * frames
        if index is None:  # the static tile shards: every rank derives every rank's
            shards = [shard_pixels(width, height, r, world, tile, frames) for r in range(world)]
        else:  # data-dependent shards (e.g. secondaries of primary hits): exchanged once at setup
            shards = [None] * world
            dist.all_gather_object(shards, np.ascontiguousarray(index, dtype=np.int64), group=group)
        self.pieces = [split_chunks(len(s), chunks) for s in shards]  # per rank, same count everywhere
        self.n_chunks = len(self.pieces[0])
        self.cap = [max(1, max(p[k][1] - p[k][0] for p in self.pieces)) for k in range(self.n_chunks)]
        self.works = []
        if rank == root:
            self.idx = [[torch.from_numpy(shards[r][a:b]).to(self.device) for (a, b) in self.pieces[r]]
                        for r in range(world)]
            self.recv = [[torch.empty((self.cap[k], COMPACT_WORDS), dtype=torch.int32, device=self.comm)
                          for _ in range(world)] for k in range(self.n_chunks)]
            self.cf_triangle = torch.as_tensor(np.asarray(cf_triangle, np.int32)).to(self.device)
            self.cf_tets = torch.as_tensor(np.asarray(cf_tets, np.int32).reshape(-1, 2)).to(self.device)
        self.send_bufs = [torch.zeros((self.cap[k], COMPACT_WORDS), dtype=torch.int32, device=self.device)
                          for k in range(self.n_chunks)]

    def my_pieces(self):
        return self.pieces[self.rank]

    def send(self, k: int, status, cf, tet, visited, t) -> None:
        """Queue chunk k's hits (visited < 2^30: it shares a word with status)."""
        import torch
        import torch.distributed as dist

        a, b = self.pieces[self.rank][k]
        n = b - a
        buf = self.send_bufs[k]
        if n:
            buf[:n, 0] = cf
            buf[:n, 1] = tet
            buf[:n, 2] = visited.to(torch.int32) | (status.to(torch.int32) << 30)
            buf[:n, 3:5] = t.to(torch.float64).contiguous().view(torch.int32).view(n, 2)
        dst = dist.get_global_rank(self.group, self.root) if self.group is not None else self.root
        gl = self.recv[k] if self.rank == self.root else None
        if self.comm != self.device:
            buf = buf.to(self.comm)
        self.works.append(dist.gather(buf, gather_list=gl, dst=dst, group=self.group, async_op=True))

    def finish(self):
        """Wait for the gathers; on the root return the full-job arrays."""
        import torch

        for w in self.works:
            w.wait()
        self.works = []
        if self.rank != self.root:
            return None
        parts, idxs = [], []
        for k in range(self.n_chunks):
            for r in range(self.world):
                a, b = self.pieces[r][k]
                parts.append(self.recv[k][r][: b - a])
                idxs.append(self.idx[r][k])
        rec = torch.cat(parts).to(self.device)
        idx = torch.cat(idxs)
        cf = rec[:, 0]
        tet = rec[:, 1]
        w2 = rec[:, 2]
        visited = w2 & 0x3FFFFFFF
        status = ((w2 >> 30) & 3).to(torch.uint8)
        t = rec[:, 3:5].contiguous().view(torch.float64).view(-1)
        hit = cf >= 0
        cfc = cf.clamp(min=0).long()
        triangle = torch.where(hit, self.cf_triangle[cfc], torch.full_like(cf, -1))
        ct = self.cf_tets[cfc]
        back = torch.where(ct[:, 0] == tet, ct[:, 1], ct[:, 0])
        tet_back = torch.where(hit, back, torch.full_like(cf, -1))
        out = {}
        for name, vals, fill in (("status", status, 0), ("cf", cf, -1), ("tet", tet, -1), ("visited", visited, 0),
                                 ("triangle", triangle, -1), ("t", t, float("inf")), ("tet_back", tet_back, -1)):
            full = torch.full((self.total,), fill, dtype=vals.dtype, device=self.device)
            full[idx] = vals
            out[name] = full
        return out


class _CudaArray:
    """__cuda_array_interface__ view of raw device memory (no copy)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


# (name, numpy typestr, bytes per ray) of the seven per-ray outputs, in the
# order tb_cast_rays_scatter takes them
_OUTPUTS = (("status", "|u1", 1), ("cf", "<i4", 4), ("tet", "<i4", 4), ("visited", "<i4", 4),
            ("triangle", "<i4", 4), ("t", "<f8", 8), ("tet_back", "<i4", 4))


class PeerFrameGather:
    """Frame assembly fused into the trace: no collective moves the hits.

    The root allocates the job's seven full-frame arrays in one device block
    and shares it with the other ranks by CUDA IPC (the 64-byte handle goes
    out with one broadcast at setup).  Every rank then traces its rays with
    ``tb_cast_rays_scatter_sched`` (or ``tb_sctp_cast_rays_scatter``): the
    kernel's epilogue stores each finished ray's results straight into the
    root's arrays at the ray's global index -- P2P stores over NVLink that
    overlap the walk ray by ray, instead of a trace followed by a gather.
    ``step`` ends with a stream sync and a barrier, after which the root's
    returned frame holds the whole job (the same arrays a single-GPU trace of
    all of it returns).

    ``index``: the global ray indices this rank traces (default: its 16x16
    tile shard, ``shard_pixels``).  Jobs that do not cover every slot (e.g.
    diffuse secondaries, spawned only from primary hits) pass the rank's real
    index array; slots no rank traces keep the "no ray" values (status 0,
    cf / triangle / tet / tet_back -1, t +inf, visited 0) written once at
    setup.

    Two frame buffers alternate between steps (three when pipelined), so a
    rank that runs ahead into step k+1 writes another buffer while the root
    still reads the frame it returned (every rank passes step k's closing
    barrier before any starts k+2).

    ``pipelined`` (lean assembly): the root's whole-job epilogue of step k
    runs on a side stream during step k+1 -- concurrently with the root's own
    trace of step k+1, which writes the other buffer -- and is joined before
    step k+1's closing barrier, so no rank touches buffer k again before it is
    finished.  Without it the epilogue follows the barrier and every rank
    waits for it (at N GPUs it covers N frames, while each rank traces one).
    ``step`` then returns the most recent *completed* frame set (step k's
    after step k+1); ``finish()`` completes the last one.

    ``root_rays``: lean assembly.  Every rank passes it -- the root the job's
    full (origins, dirs) device tensors in global ray order, the others
    ``True`` -- and the ranks then store only status / cf / tet / visited
    (13 B per ray over NVLink instead of 29); after the barrier the root
    derives triangle / t / tet_back for the whole job with
    ``tb_cast_epilogue`` (bit-identical to the fused epilogue).  ``step`` may
    pass this step's rays (``root_rays=``) when they change between steps.
    """

    BUFFERS = 2  # 3 when pipelined (the frame returned by step k+1 is step k's)

    def __init__(self, width, height, world, rank, frames, device, root=0, group=None, tile=16, root_rays=None,
                 index=None, pipelined=False):
        import ctypes

        import torch
        import torch.distributed as dist

        from ._lib import check, lib

        self.world, self.rank, self.root, self.group = world, rank, root, group
        self.lean = root_rays is not None
        self.root_rays = root_rays if (self.lean and rank == root) else None
        self.pipelined = bool(pipelined) and self.lean
        # pipelined, step k+1 returns step k's frame; a rank running ahead into
        # step k+2 must not touch it, hence a third buffer
        self.buffers = self.BUFFERS + (1 if self.pipelined else 0)
        self.pending = None  # (buffer, rays) whose root epilogue has not run yet
        self.epi_stream = None
        self.device = torch.device(device)
        self.total = width * height * frames
        shard = shard_pixels(width, height, rank, world, tile, frames) if index is None else np.asarray(index)
        if shard.size and (shard.min() < 0 or shard.max() >= self.total):
            raise ValueError(f"index out of range [0, {self.total})")
        self.idx = torch.from_numpy(np.ascontiguousarray(shard, dtype=np.int64)).to(self.device)
        self.offsets = []
        off = 0
        for _, _, size in _OUTPUTS:
            self.offsets.append(off)
            off += (size * self.total + 255) // 256 * 256
        self.frame_bytes = off
        self.bytes = off * self.buffers
        self.base = None
        self.remote = None
        self.steps = 0
        dev_idx = self.device.index if self.device.index is not None else torch.cuda.current_device()
        handle = None
        err = None
        if rank == root:
            try:
                p = ctypes.c_void_p()
                check(lib.tb_device_alloc(self.bytes, dev_idx, ctypes.byref(p)), "tb_device_alloc")
                self.base = p.value
                buf = (ctypes.c_char * 64)()
                check(lib.tb_ipc_get_handle(self.base, buf), "tb_ipc_get_handle")
                handle = bytes(buf)
            except Exception as exc:  # every rank must learn of it (below), not hang in the broadcast
                err = repr(exc)
        obj = [handle]
        src = dist.get_global_rank(group, root) if group is not None else root
        dist.broadcast_object_list(obj, src=src, group=group)
        if rank != root and obj[0] is not None:
            try:
                p = ctypes.c_void_p()
                check(lib.tb_ipc_open(obj[0], dev_idx, ctypes.byref(p)), "tb_ipc_open")
                self.remote = p.value
            except Exception as exc:
                err = repr(exc)
        # collective verdict: either every rank has the shared block or all
        # of them give it up together (callers then fall back to FrameGather)
        verdicts = [None] * dist.get_world_size(group)
        dist.all_gather_object(verdicts, err, group=group)
        failed = [v for v in verdicts if v is not None]
        if failed or obj[0] is None:
            if self.remote is not None:
                lib.tb_ipc_close(self.remote)
                self.remote = None
            dist.barrier(group=group)
            if self.base is not None:
                lib.tb_device_free(self.base)
                self.base = None
            raise RuntimeError(f"peer frame assembly unavailable: {failed[0] if failed else 'no IPC handle'}")
        dest = self.base if rank == root else self.remote
        self.ptrs = [[dest + b * self.frame_bytes + o for o in self.offsets] for b in range(self.buffers)]
        self.frames = None
        if rank == root:
            fills = {"status": 0, "cf": -1, "tet": -1, "visited": 0, "triangle": -1, "t": float("inf"),
                     "tet_back": -1}
            self.frames = []
            for b in range(self.buffers):
                fr = {name: torch.as_tensor(_CudaArray(self.base + b * self.frame_bytes + o, self.total, ts),
                                            device=self.device)
                      for (name, ts, _), o in zip(_OUTPUTS, self.offsets)}
                for name, a in fr.items():
                    a.fill_(fills[name])
                self.frames.append(fr)
            torch.cuda.synchronize(self.device)
        dist.barrier(group=group)  # the defaults are in place before any rank stores

    @property
    def frame(self):
        """The root's most recently completed frame (None on other ranks)."""
        if self.frames is None:
            return None
        done = self.steps - (1 if self.pending is not None else 0)
        return self.frames[(done - 1) % self.buffers if done else 0]

    def _epilogue(self, ptrs, rays, stream):
        from ._lib import addr, check, lib

        ro, rd = rays
        if ro.shape[0] != self.total or rd.shape[0] != self.total:
            raise ValueError(f"root_rays must hold the job's {self.total} rays")
        check(lib.tb_cast_epilogue(self._dm.handle, self.total, addr(ro), addr(rd), ptrs[1], ptrs[2], ptrs[4],
                                   ptrs[5], ptrs[6], stream.cuda_stream), "tb_cast_epilogue")

    def finish(self):
        """Complete a pipelined step's pending root epilogue; returns the
        root's latest frame (None on other ranks)."""
        import torch

        if self.pending is not None:
            ptrs, rays, evs = self.pending
            s = torch.cuda.current_stream(self.device)
            for ev in evs:
                s.wait_event(ev)
            self._epilogue(ptrs, rays, s)
            s.synchronize()
            self.pending = None
        return self.frame

    def step(self, dm, origins, dirs, start, stream=None, *, schedule="lane", sctp=False, root_rays=None):
        """Trace this rank's rays into the root's frame; returns the frame on
        the root (torch tensors over the shared block), None elsewhere.
        ``schedule``: "lane" or "binned" (the binned walk's permutation is
        composed with the scatter index); ``sctp`` runs the ScTP walk."""
        import torch
        import torch.distributed as dist

        from ._lib import SCHEDULES, addr, check, lib

        n = self.idx.numel()
        if origins.shape[0] != n or dirs.shape[0] != n or start.numel() != n:
            raise ValueError(f"this rank traces {n} rays (its index), got {origins.shape[0]} origins, "
                             f"{dirs.shape[0]} dirs, {start.numel()} starts")
        s = stream or torch.cuda.current_stream(self.device)
        ptrs = self.ptrs[self.steps % self.buffers]
        self._dm = dm
        epi = None
        if self.pending is not None:  # pipelined: the previous step's root epilogue, beside this trace
            if self.epi_stream is None:
                self.epi_stream = torch.cuda.Stream(self.device)
            epi = self.pending
            for ev in epi[2]:  # the rays were produced in the caller's stream order
                self.epi_stream.wait_event(ev)
            self._epilogue(epi[0], epi[1], self.epi_stream)
        # _OUTPUTS order: status, cf, tet, visited, triangle, t, tet_back
        outs = ptrs[:4] + [None, None, None] if self.lean else ptrs
        if sctp:
            check(lib.tb_sctp_cast_rays_scatter(dm.handle, n, addr(origins), addr(dirs), addr(start), addr(self.idx),
                                                *outs, s.cuda_stream), "tb_sctp_cast_rays_scatter")
        else:
            mode = SCHEDULES[schedule] if isinstance(schedule, str) else int(schedule)
            check(lib.tb_cast_rays_scatter_sched(dm.handle, n, addr(origins), addr(dirs), addr(start),
                                                 addr(self.idx), *outs, mode, s.cuda_stream),
                  "tb_cast_rays_scatter_sched")
        s.synchronize()  # this rank's stores have landed in the root's memory
        if epi is not None:
            self.epi_stream.synchronize()  # buffer k is finished before anyone passes this barrier
            self.pending = None
        dist.barrier(group=self.group)
        self.steps += 1
        if self.rank == self.root and self.lean:
            rays = root_rays if root_rays is not None else self.root_rays
            if rays[0].shape[0] != self.total or rays[1].shape[0] != self.total:
                raise ValueError(f"root_rays must hold the job's {self.total} rays")
            if self.pipelined:
                evs = []
                for st in {s, torch.cuda.current_stream(self.device)}:
                    ev = torch.cuda.Event()
                    ev.record(st)
                    evs.append(ev)
                self.pending = (ptrs, rays, evs)
            else:
                self._epilogue(ptrs, rays, s)
                s.synchronize()
        return self.frame

    def close(self):
        import torch.distributed as dist

        from ._lib import lib

        self.pending = None  # a pipelined step's unfinished epilogue dies with the frames
        if self.remote is not None:
            lib.tb_ipc_close(self.remote)
            self.remote = None
        dist.barrier(group=self.group)  # every mapping is gone before the root frees the block
        if self.base is not None:
            self.frames = None
            lib.tb_device_free(self.base)
            self.base = None


def trace_multi(meshes, width: int, height: int, origins, dirs, start, *, out=None, stream=None, epilogue=True):
    """Single-process multi-GPU trace of one frame (``tb_trace_multi``).

    ``meshes``: DeviceMesh replicas, one per GPU (``device_mesh(mesh, device=k)``);
    ``origins`` / ``dirs`` (W*H, 3) float32 and ``start`` (W*H,) int32 are torch
    tensors on ``meshes[0]``'s device.  The frame's 16x16 tiles go round-robin
    to the replicas; each GPU walks its tiles straight from these arrays and
    stores its results into ``out`` (a TraceResult on the same device) -- the
    same arrays a single-GPU ``trace`` of the frame returns.
    """
    import ctypes

    import torch

    from ._lib import addr, check, lib
    from .trace import empty_result

    n = int(width) * int(height)
    if origins.shape != (n, 3) or dirs.shape != (n, 3) or start.shape != (n,):
        raise ValueError(f"rays must be ({n}, 3) / ({n},) for a {width}x{height} frame")
    dev = origins.device
    for x, dt in ((origins, torch.float32), (dirs, torch.float32), (start, torch.int32)):
        if x.device != dev or x.dtype != dt or not x.is_contiguous():
            raise ValueError("rays must be contiguous float32 / int32 tensors on one device")
    res = out if out is not None else empty_result(n, dev)
    handles = (ctypes.c_void_p * len(meshes))(*[m.handle.value for m in meshes])
    s = (stream or torch.cuda.current_stream(dev)).cuda_stream
    check(lib.tb_trace_multi(len(meshes), ctypes.cast(handles, ctypes.c_void_p), int(width), int(height), addr(origins), addr(dirs), addr(start),
                             addr(res.status), addr(res.cf), addr(res.tet), addr(res.visited),
                             addr(res.triangle) if epilogue else None, addr(res.t) if epilogue else None,
                             addr(res.tet_back) if epilogue else None, s), "tb_trace_multi")
    return res
