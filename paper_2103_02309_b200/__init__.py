"""B200-native tetrahedral-mesh ray traversal (Aman, Demirci, Gudukbay,
"Compact Tetrahedralization-based Acceleration Structure for Ray Tracing",
arXiv 2103.02309).

A drop-in CUDA backend for the reference package's kernel-module protocol
(tetray._kernels: cast_rays / locate_points / shadow_rays) plus a host-side
mirror of the mesh API it consumes.  The traversal runs in hand-written
sm_100a kernels (csrc/) behind a C ABI (include/tetb200.h); there is no CPU
fallback: importing the kernel module without the built library raises.
"""

__version__ = "0.1.0"
