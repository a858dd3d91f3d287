"""ctypes binding of libtetb200.so (the C ABI in include/tetb200.h).

The library is built in-tree (``make`` or ``__graft_entry__.build()``) and
loaded from this package directory.  There is deliberately no fallback: if
the library is missing the import fails loudly.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int64, c_size_t, c_uint32, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TETB200_LIB", os.path.join(_HERE, "libtetb200.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libtetb200.so not found at {LIB_PATH}: build it with `make` or "
        "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
    )

lib = ctypes.CDLL(LIB_PATH)

P = c_void_p  # every array argument is passed as a raw address

_SIGS = {
    "tb_abi_version": (c_int, []),
    "tb_last_error": (c_char_p, []),
    "tb_mesh_create": (
        c_int,
        [c_int, c_int, c_int64, P, c_int64, P, P, P, c_int64, P, P, c_int64, P, POINTER(c_void_p)],
    ),
    "tb_mesh_destroy": (c_int, [c_void_p]),
    "tb_mesh_info": (
        c_int,
        [c_void_p, POINTER(c_int), POINTER(c_int), POINTER(c_int64), POINTER(c_int64), POINTER(c_int64),
         POINTER(c_int64), POINTER(c_int64)],
    ),
    "tb_mesh_validated": (c_int, [c_void_p, POINTER(c_int)]),
    "tb_probe_gather": (c_int, [c_void_p, c_int64, c_uint32, P, c_void_p]),
    "tb_cast_epilogue": (c_int, [c_void_p, c_int64, P, P, P, P, P, P, P, c_void_p]),
    "tb_mesh_replicate": (c_int, [c_void_p, c_int, POINTER(c_void_p)]),
    "tb_trace_multi": (c_int, [c_int, P, c_int64, c_int64, P, P, P, P, P, P, P, P, P, P, c_void_p]),
    "tb_cast_rays": (c_int, [c_void_p, c_int64, P, P, P, P, P, P, P, P, P, P, c_void_p]),
    "tb_cast_rays_sched": (c_int, [c_void_p, c_int64, P, P, P, P, P, P, P, P, P, P, c_int, c_void_p]),
    "tb_cast_block_size": (c_int, []),
    "tb_auto_schedule": (c_int, [c_int, c_int64]),
    "tb_sampled_head_blocks": (c_int64, [c_int, c_int64]),
    "tb_binned_pieces": (c_int, [c_int64]),
    "tb_block_order": (c_int, [c_int64, P, P, c_int64, c_void_p]),
    "tb_cast_rays_ordered": (c_int, [c_void_p, c_int64, P, P, P, P, c_int64, P, P, P, P, P, P, P, c_void_p]),
    "tb_cast_rays_scatter": (c_int, [c_void_p, c_int64, P, P, P, P, P, P, P, P, P, P, P, c_void_p]),
    "tb_cast_rays_scatter_sched": (c_int, [c_void_p, c_int64, P, P, P, P, P, P, P, P, P, P, P, c_int, c_void_p]),
    "tb_sctp_cast_rays_scatter": (c_int, [c_void_p, c_int64, P, P, P, P, P, P, P, P, P, P, P, c_void_p]),
    "tb_device_alloc": (c_int, [c_size_t, c_int, POINTER(c_void_p)]),
    "tb_device_free": (c_int, [P]),
    "tb_ipc_get_handle": (c_int, [P, P]),
    "tb_ipc_open": (c_int, [P, c_int, POINTER(c_void_p)]),
    "tb_ipc_close": (c_int, [P]),
    "tb_cast_rays_host": (c_int, [c_void_p, c_int64, P, P, P, P, P, P, P, P, P, P]),
    "tb_sctp_cast_rays": (c_int, [c_void_p, c_int64, P, P, P, P, P, P, P, P, P, P, c_void_p]),
    "tb_sctp_cast_rays_host": (c_int, [c_void_p, c_int64, P, P, P, P, P, P, P, P, P, P]),
    "tb_cast_rays_visits": (c_int, [c_void_p, c_int64, P, P, P, P, P, c_void_p]),
    "tb_locate_points": (c_int, [c_void_p, c_int64, P, P, P, P, c_void_p]),
    "tb_hull_clip": (c_int, [c_void_p, c_int64, P, P, P, c_int64, P, P, P, c_void_p]),
    "tb_camera_rays": (c_int, [c_int64, c_int64, P, P, c_int64, P, P, c_void_p]),
    "tb_trace_camera": (c_int, [c_void_p, c_int64, c_int64, P, c_int, P, P, P, P, P, P, P, c_void_p]),
    "tb_locate_points_host": (c_int, [c_void_p, c_int64, P, P, P, P]),
    "tb_shadow_rays": (c_int, [c_void_p, c_int64, P, P, c_int, P, P, c_int, c_double, P, P, c_void_p]),
    "tb_shadow_rays_host": (c_int, [c_void_p, c_int64, P, P, c_int, P, P, c_int, c_double, P, P]),
    "tb_set_schedule": (c_int, [c_int, c_int]),
    "tb_get_schedule": (c_int, [POINTER(c_int), POINTER(c_int)]),
    "tb_hilbert_keys": (c_int, [P, c_int64, c_int, P]),
    "tb_hilbert_quantize": (c_int, [P, c_int64, P, P, c_int, P]),
    "tb_tet_centroids": (c_int, [P, c_int64, P, c_int64, P]),
    "tb_build_side_tables": (c_int, [c_int64, P, P, P, P, c_int64, P, c_int64, P, P]),
    "tb_pack_records": (c_int, [c_int, c_int64, P, P, P]),
    "tb_host_alloc": (c_int, [c_size_t, POINTER(c_void_p)]),
    "tb_host_free": (c_int, [c_void_p]),
}

EXPORTED = tuple(_SIGS)

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

if lib.tb_abi_version() != 1:
    raise ImportError(f"libtetb200.so ABI {lib.tb_abi_version()} != 1; rebuild")


class TetB200Error(RuntimeError):
    """A C-ABI call failed (bad argument, CUDA error, out of memory)."""


def check(code: int, what: str) -> None:
    if code != 0:
        msg = lib.tb_last_error()
        raise TetB200Error(f"{what} failed ({code}): {msg.decode() if msg else 'unknown error'}")


SCHEDULES = {"auto": 0, "lane": 1, "refill": 2, "compact": 3, "compact512": 4, "dynamic": 5, "binned": 6,
             "sampled": 7}


def set_schedule(mode: str | int | None = None, steps_per_round: int | None = None) -> None:
    """Process-wide ray-to-lane schedule of the cast kernels (tb_set_schedule).
    Results are identical in every mode."""
    m = -1 if mode is None else (SCHEDULES[mode] if isinstance(mode, str) else int(mode))
    check(lib.tb_set_schedule(m, -1 if steps_per_round is None else int(steps_per_round)), "tb_set_schedule")


def get_schedule() -> tuple[int, int]:
    m, k = c_int(), c_int()
    check(lib.tb_get_schedule(ctypes.byref(m), ctypes.byref(k)), "tb_get_schedule")
    return m.value, k.value


_from_buffer = ctypes.c_char.from_buffer
_addressof = ctypes.addressof


def addr(a) -> int | None:
    """Raw address of a numpy array or torch tensor (None stays NULL).
    Writable numpy arrays go through the buffer protocol (~0.4 us; the
    per-tile protocol calls pass 7-10 arrays), read-only ones through
    ``ndarray.ctypes`` (~2.5 us)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    if a.flags.writeable and a.size:
        try:
            return _addressof(_from_buffer(a))
        except (TypeError, ValueError, BufferError):
            pass
    return a.ctypes.data
