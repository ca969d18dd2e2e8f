"""Test-side device memory helpers (plain cudart through ctypes; the primary
context is shared with the library's static runtime)."""
import ctypes
import glob
import os

import numpy as np

_RT = None


def rt():
    global _RT
    if _RT is None:
        cands = glob.glob("/usr/local/cuda/lib64/libcudart.so*") + glob.glob(
            "/usr/local/cuda/targets/x86_64-linux/lib/libcudart.so*")
        _RT = ctypes.CDLL(sorted(cands)[0])
        _RT.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
        _RT.cudaMemset.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t]
        _RT.cudaMalloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t]
        _RT.cudaFree.argtypes = [ctypes.c_void_p]
        _RT.cudaSetDevice.argtypes = [ctypes.c_int]
        _RT.cudaDeviceSynchronize.argtypes = []
    return _RT


def _ck(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed with cudaError {rc}")


def set_device(d):
    _ck(rt().cudaSetDevice(d), "cudaSetDevice")


def sync():
    _ck(rt().cudaDeviceSynchronize(), "cudaDeviceSynchronize")


def d2h(ptr, nbytes, dtype=np.uint8):
    out = np.empty(nbytes, np.uint8)
    if nbytes:
        _ck(rt().cudaMemcpy(out.ctypes.data, ptr, nbytes, 2), "cudaMemcpy D2H")
    return out.view(dtype)


def h2d(ptr, arr):
    a = np.ascontiguousarray(arr)
    if a.nbytes:
        _ck(rt().cudaMemcpy(ptr, a.ctypes.data, a.nbytes, 1), "cudaMemcpy H2D")


def memset(ptr, val, nbytes):
    _ck(rt().cudaMemset(ptr, val, nbytes), "cudaMemset")


def malloc(nbytes):
    p = ctypes.c_void_p()
    _ck(rt().cudaMalloc(ctypes.byref(p), max(1, nbytes)), "cudaMalloc")
    return p.value


def free(p):
    rt().cudaFree(p)


def host_mapped_words(n=16):
    """Zeroed pinned host words the device can poll: (host address, device pointer)."""
    L = rt()
    L.cudaHostAlloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_uint]
    L.cudaHostGetDevicePointer.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_void_p, ctypes.c_uint]
    hp, dp = ctypes.c_void_p(), ctypes.c_void_p()
    _ck(L.cudaHostAlloc(ctypes.byref(hp), 4 * n, 2), "cudaHostAlloc")  # cudaHostAllocMapped
    ctypes.memset(hp, 0, 4 * n)
    _ck(L.cudaHostGetDevicePointer(ctypes.byref(dp), hp, 0), "cudaHostGetDevicePointer")
    return hp.value, dp.value
