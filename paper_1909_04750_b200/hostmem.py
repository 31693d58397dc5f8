"""Pinned host memory for result arrays, and the per-thread context pool.

The reference's bulk API hands the caller a FRESH numpy array per call
(pkg/src/slicerng/kernels.py:194-200).  A fresh pageable array is the slowest
possible D2H destination: the driver stages the copy through small internal
buffers and the pages take their first-touch faults on the way.  `empty()`
returns numpy arrays backed by page-locked memory (mk2_host_alloc, include/mk2.h)
from a cache of released blocks, so large results take the direct asynchronous
D2H path at link speed and cost no cudaHostAlloc in steady state.  The array owns
its block: when the last view dies the block goes back to the cache.

`borrow_context()` keeps a few C-ABI contexts per (thread, device, class) alive
between calls of the reference-shaped entry points (`mickey_sliced_words`,
`MickeySliced.from_key_ivs`, `bulk_*`, `derive_arrays`): a context is two streams,
eight events, a memory pool and four device arrays, which the reference's
64-lane batching loops (cli.py:219-231) would otherwise create and destroy per
batch.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import threading

import numpy as np

from . import _native

PINNED_MIN_BYTES = 1 << 20        # smaller results stay in ordinary numpy memory (a pageable copy of that size is cheap)
CACHE_LIMIT_BYTES = 8 << 30       # released blocks kept for reuse; beyond this they are freed at once
_GRANULE = 2 << 20


class _Block:
    """One page-locked allocation; exposes its bytes through the array interface so numpy keeps it alive."""

    __slots__ = ("ptr", "size", "pool", "__array_interface__", "__weakref__")

    def __init__(self, ptr: int, size: int, nbytes: int, pool: "PinnedPool"):
        self.ptr, self.size, self.pool = ptr, size, pool
        self.__array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}

    def __del__(self):
        pool, self.pool = self.pool, None
        if pool is not None:
            pool._release(self.ptr, self.size)


class PinnedPool:
    def __init__(self, limit: int = CACHE_LIMIT_BYTES):
        self.limit = limit
        self._lock = threading.Lock()
        self._free: list[tuple[int, int]] = []   # (size, ptr), sorted by size
        self._cached = 0
        self.allocs = 0                           # cudaHostAlloc calls so far (diagnostics / tests)

    def empty(self, shape, dtype) -> np.ndarray:
        dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape, dtype=np.int64)) * dtype.itemsize
        if nbytes < PINNED_MIN_BYTES:
            return np.empty(shape, dtype)
        ptr, size = self._take(nbytes)
        return np.asarray(_Block(ptr, size, nbytes, self)).view(dtype).reshape(shape)

    def _take(self, nbytes: int):
        with self._lock:
            for i, (size, ptr) in enumerate(self._free):
                if size >= nbytes:
                    if size <= nbytes + nbytes // 4 + _GRANULE:   # close enough: reuse
                        del self._free[i]
                        self._cached -= size
                        return ptr, size
                    break
        size = (nbytes + _GRANULE - 1) // _GRANULE * _GRANULE
        out = C.c_void_p()
        rc = _native.lib().mk2_host_alloc(size, C.byref(out))
        if rc == _native.MK2_E_NOMEM:
            self.trim()
            rc = _native.lib().mk2_host_alloc(size, C.byref(out))
        _native.check(rc, None, "mk2_host_alloc")
        self.allocs += 1
        return int(out.value), size

    def _release(self, ptr: int, size: int):
        # may run from a garbage collection at any point, also while this thread is inside _take: never block
        try:
            if self._lock.acquire(blocking=False):
                try:
                    if self._cached + size <= self.limit:
                        self._free.append((size, ptr))
                        self._free.sort()
                        self._cached += size
                        return
                finally:
                    self._lock.release()
            _native.lib().mk2_host_free(C.c_void_p(ptr))
        except Exception:  # interpreter shutdown
            pass

    def trim(self):
        """Give every cached block back to the system."""
        with self._lock:
            blocks, self._free, self._cached = self._free, [], 0
        for _size, ptr in blocks:
            _native.lib().mk2_host_free(C.c_void_p(ptr))

    @property
    def cached_bytes(self) -> int:
        return self._cached


pool = PinnedPool()


def empty(shape, dtype) -> np.ndarray:
    """A fresh, caller-owned result array: page-locked when it is large enough to matter."""
    return pool.empty(shape, dtype)


# ---------------------------------------------------------------------------- context pool

_MAX_IDLE = 4              # idle contexts kept per (thread, device, class)
_MAX_IDLE_GROUPS = 1 << 16  # contexts that grew beyond 2^21 instances (52 MB of state) are not kept
_tls = threading.local()


def _idle(key):
    d = getattr(_tls, "idle", None)
    if d is None:
        d = _tls.idle = {}
    return d.setdefault(key, [])


def acquire_context(cls, device: int):
    """A context of class `cls` (MickeyGenerator or a subclass) on `device`: an idle one of this thread, else new."""
    idle = _idle((cls, int(device)))
    while idle:
        gen = idle.pop()
        if gen._ctx:
            return gen
    return cls(device)


def release_context(gen) -> None:
    """Hand a context back; it is destroyed instead when the thread already holds enough idle ones, when it grew
    large, or when tuning knobs may have been changed on it."""
    if gen is None or not getattr(gen, "_ctx", None):
        return
    try:
        idle = _idle((type(gen), gen.device))
        if len(idle) < _MAX_IDLE and not gen._knobs_touched and gen._peak_groups <= _MAX_IDLE_GROUPS:
            idle.append(gen)
            return
    except Exception:
        pass
    gen.close()


@contextlib.contextmanager
def borrow_context(cls, device: int):
    gen = acquire_context(cls, device)
    try:
        yield gen
    except BaseException:
        gen.close()   # an error may have left it in any state
        raise
    else:
        release_context(gen)


def drop_idle_contexts() -> None:
    """Destroy this thread's idle contexts (tests; before a fork)."""
    for lst in getattr(_tls, "idle", {}).values():
        while lst:
            lst.pop().close()
