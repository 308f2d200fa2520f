"""B200-native ExaBricks hot path (arXiv 2009.03076), drop-in for `amrvol`.

Python host code mirrors the reference's public API (R/ = /root/reference/
pkg/src/amrvol/): build_bricks, build_regions, build_scene, render_frame, ...
Every compute entry point crosses a C ABI (`include/exabricks.h`,
`libexabricks.so`, ctypes) into hand-written sm_100a CUDA kernels.  There is no
CPU fallback: without the native library the compute API raises.
"""

__version__ = "0.1.0"
