"""Device plumbing: torch CUDA tensors as buffers, stream handles, caches.

torch is used only to allocate device memory and name the current stream;
every computation goes through libtopofuse_b200.so.
"""

from __future__ import annotations

import weakref

import numpy as np

from . import _lib

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def require_cuda(device=None):
    """Raise (no CPU fallback) unless a CUDA device and the kernel library exist."""
    t = torch()
    if not t.cuda.is_available():
        raise _lib.TfError("paper_2604_18020_b200 needs a CUDA device (B200, sm_100a); "
                           "this product path has no CPU fallback")
    _lib.load()
    dev = t.device("cuda", t.cuda.current_device() if device is None else device)
    return dev


def stream_ptr():
    return torch().cuda.current_stream().cuda_stream


def tdtype(np_dtype):
    t = torch()
    return {np.dtype(np.float32): t.float32, np.dtype(np.float64): t.float64,
            np.dtype(np.int32): t.int32, np.dtype(np.int64): t.int64,
            np.dtype(np.uint8): t.uint8}[np.dtype(np_dtype)]


def to_dev(a, dtype=None, device=None):
    """numpy/torch -> contiguous CUDA tensor of `dtype` (numpy dtype)."""
    t = torch()
    dev = require_cuda(device)
    if isinstance(a, t.Tensor):
        out = a.to(device=dev, dtype=tdtype(dtype) if dtype is not None else a.dtype)
        return out.contiguous()
    arr = np.ascontiguousarray(a, dtype=dtype)
    return t.from_numpy(arr).to(dev, non_blocking=False)


def ptr(x) -> int:
    """Device address of a tensor.  The caller must keep `x` alive until the
    kernel using it has been enqueued -- never pass a temporary (the caching
    allocator may hand its block to the next allocation of the same call)."""
    return 0 if x is None else x.data_ptr()


def is_tensor(x) -> bool:
    if _torch is None:
        try:
            import torch as _t  # noqa: F401
        except ImportError:  # pragma: no cover
            return False
    return isinstance(x, torch().Tensor)


class IdCache:
    """Per-object cache keyed by identity, released when the object dies.

    Cached values must not hold strong references to their key object
    (the finalizer would never fire); DeviceProblem keeps a weakref to its
    edof for that reason.  ``clear()`` drops every entry explicitly."""

    def __init__(self):
        self._d = {}

    def __len__(self):
        return len(self._d)

    def clear(self):
        self._d.clear()

    def get(self, obj, key, make):
        k = (id(obj), key)
        hit = self._d.get(k)
        if hit is not None:
            ref, val = hit
            if ref() is obj:
                return val
        val = make()
        try:
            ref = weakref.ref(obj)
        except TypeError:  # not weak-referenceable: do not cache
            return val
        self._d[k] = (ref, val)
        weakref.finalize(obj, self._d.pop, k, None)
        return val


CACHE = IdCache()


def node_fixed_mask(n_nodes: int, fixed_dofs: np.ndarray, nodes_per_plane: int | None = None) -> np.ndarray:
    """Host restatement of tf_build_node_fixed: one byte per node (bit c set
    when DOF 3*node + c is constrained), optionally followed by the per-column
    OR over node planes."""
    m = np.zeros(n_nodes, dtype=np.uint8)
    f = np.asarray(fixed_dofs, dtype=np.int64)
    if f.size:
        np.bitwise_or.at(m, f // 3, (1 << (f % 3)).astype(np.uint8))
    if nodes_per_plane is None:
        return m
    planes = m.reshape(-1, nodes_per_plane)
    return np.concatenate([m, np.bitwise_or.reduce(planes, axis=0), np.bitwise_and.reduce(planes, axis=0)])


def masked_edof(edof: np.ndarray, fixed_dofs: np.ndarray, n_dof: int) -> np.ndarray:
    """edof with every constrained DOF slot marked by its sign bit (d | 2^31,
    a negative int32): every kernel gathers 0 there and never scatters to it
    (slots < 0), except the neighbour-merged atomic product, which adds the
    slot's row to DOF d itself -- a constrained DOF the pass-through then
    overwrites -- to keep its reductions branch-free (csrc/tf_matvec.cu)."""
    free = np.ones(n_dof, dtype=bool)
    free[np.asarray(fixed_dofs, dtype=np.int64)] = False
    e = np.ascontiguousarray(edof, dtype=np.int32)
    return np.where(free[e], e, e | np.int32(-(2**31))).astype(np.int32)


def bind_gpu_local_cpus(index: int = 0):
    """Bind this process to the CPUs NVML reports as local to GPU `index`
    (its NUMA node), so pinned host buffers allocated afterwards live next to
    the GPU's PCIe root: host<->device copies then run at the link rate
    instead of crossing the socket interconnect.  Returns the CPU list (None
    when NVML is unavailable; nothing is changed then)."""
    import os

    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
    except Exception:
        return None
    cpus = [64 * w + b for w, mask in enumerate(words) for b in range(64) if (mask >> b) & 1]
    cpus = [c for c in cpus if c < (os.cpu_count() or 0)]
    if not cpus:
        return None
    try:
        os.sched_setaffinity(0, cpus)
    except OSError:
        return None
    return cpus


class _HostBlock:
    """Owner of one cudaHostAlloc block (freed when the last tensor view dies)."""

    def __init__(self, nbytes: int):
        import ctypes

        from . import _lib

        self.ptr = ctypes.c_void_p()
        _lib.call("tf_host_alloc", ctypes.byref(self.ptr), int(nbytes))
        self.nbytes = int(nbytes)

    def __del__(self):
        try:
            from . import _lib

            _lib.load().tf_host_free(self.ptr)
        except Exception:  # pragma: no cover - interpreter teardown
            pass


def pinned_empty(n: int, dtype):
    """A CPU torch tensor of `n` elements in page-locked memory from
    cudaHostAlloc -- the host side of the e2e path.  (torch's pin_memory()
    buffers measured 13.9 GB/s host-to-device on the pool's B200 VMs; these
    run at the PCIe link rate, 51.8 GB/s, scripts/h2d_probe.cu.)"""
    import ctypes

    t = torch()
    tdt = dtype if isinstance(dtype, t.dtype) else tdtype(dtype)
    nbytes = int(n) * t.empty(0, dtype=tdt).element_size()
    blk = _HostBlock(max(nbytes, 16))
    buf = (ctypes.c_char * nbytes).from_address(blk.ptr.value)
    out = t.frombuffer(buf, dtype=tdt, count=int(n))
    out._tf_host_block = blk  # keeps the allocation alive with the tensor
    return out


class gc_paused:
    """Pause Python's automatic cyclic GC for a host-driven device loop
    (restored on exit).  A full collection over a torch process's ~10^6
    long-lived objects takes ~0.1 s -- several SIMP iterations' worth at
    c1/c2 -- and the loops create no reference cycles, so nothing
    accumulates while it is paused."""

    def __enter__(self):
        import gc

        self._was = gc.isenabled()
        gc.disable()
        return self

    def __exit__(self, *a):
        import gc

        if self._was:
            gc.enable()
        return False
