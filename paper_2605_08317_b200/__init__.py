"""B200-native RDKV accelerator path (allocate -> pack -> decode) for sm_100a.

The product is the native library _lib/librdkv_b200.so (C-ABI in
include/rdkv_cuda.h, C++ drop-in API in include/rdkv/). `capi` binds it with
ctypes; `pipeline` is the device-resident Python mirror of the reference's
entry points used by tests and bench.py.
"""
import os as _os

ROOT = _os.path.dirname(_os.path.abspath(__file__))


def build(verbose: bool = False) -> None:
    """Compile every CUDA/C++ source of the package for sm_100a (nvcc, in-tree)."""
    import subprocess

    subprocess.run(["make", "-C", _os.path.join(ROOT, "csrc"), "-j8"], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)
