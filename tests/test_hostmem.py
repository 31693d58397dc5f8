"""CPU-only checks of the host-side memory and context pools (paper_1909_04750_b200/hostmem.py).

The page-locked allocator behind the package's result arrays needs a GPU; here `mk2_host_alloc` / `mk2_host_free`
are replaced by malloc / free so that the pool's logic -- ownership through the array's base object, reuse of
released blocks, the cache limit, never blocking inside a finaliser -- is tested without one.  The context pool is
exercised with a stand-in generator class.
"""
import ctypes as C
import gc
import threading

import numpy as np
import pytest

from paper_1909_04750_b200 import _native, hostmem


class _FakeLib:
    def __init__(self):
        self.libc = C.CDLL(None)
        self.libc.malloc.restype = C.c_void_p
        self.libc.malloc.argtypes = [C.c_size_t]
        self.libc.free.argtypes = [C.c_void_p]
        self.live = {}
        self.fail_next = False

    def mk2_host_alloc(self, size, out):
        if self.fail_next:
            self.fail_next = False
            return _native.MK2_E_NOMEM
        p = self.libc.malloc(size)
        self.live[p] = size
        out._obj.value = p
        return 0

    def mk2_host_free(self, p):
        assert p.value in self.live, "double free or foreign pointer"
        del self.live[p.value]
        self.libc.free(p)
        return 0

    def mk2_last_error(self, ctx):
        return b"fake"


@pytest.fixture
def fake(monkeypatch):
    lib = _FakeLib()
    monkeypatch.setattr(_native, "lib", lambda: lib)
    return lib


def test_small_arrays_stay_in_ordinary_memory(fake):
    pool = hostmem.PinnedPool()
    a = pool.empty((100, 8), np.uint32)
    assert a.shape == (100, 8) and a.dtype == np.uint32 and pool.allocs == 0 and not fake.live


def test_blocks_are_owned_by_the_array_and_reused(fake):
    pool = hostmem.PinnedPool()
    n = hostmem.PINNED_MIN_BYTES
    a = pool.empty((n // 4,), np.uint32)
    assert pool.allocs == 1 and a.flags.writeable and a.nbytes == n
    a[:] = 7
    view = a[10:20]                       # a view keeps the block alive
    del a
    gc.collect()
    assert pool.cached_bytes == 0 and int(view.sum()) == 70
    del view
    gc.collect()
    assert pool.cached_bytes >= n and len(fake.live) == 1
    b = pool.empty((n,), np.uint8)        # same size class: the released block comes back, no new allocation
    assert pool.allocs == 1 and pool.cached_bytes == 0
    c = pool.empty((3 * n,), np.uint8)    # larger: a new block
    assert pool.allocs == 2
    del b, c
    gc.collect()
    d = pool.empty((n,), np.uint8)        # the small block again, not the 3x one (close-fit rule)
    assert pool.allocs == 2 and pool.cached_bytes >= 3 * n
    del d
    pool.trim()
    gc.collect()
    assert pool.cached_bytes == 0 and not fake.live


def test_cache_limit_and_allocation_failure(fake):
    n = hostmem.PINNED_MIN_BYTES
    pool = hostmem.PinnedPool(limit=2 * hostmem._GRANULE + 1)             # blocks are multiples of the 2 MiB granule
    arrs = [pool.empty((n,), np.uint8) for _ in range(3)]
    del arrs
    gc.collect()
    assert pool.cached_bytes <= pool.limit and len(fake.live) == 2      # the third block was freed at once
    fake.fail_next = True                                               # NOMEM: the pool trims itself and retries
    big = pool.empty((8 * n,), np.uint8)
    assert big.nbytes == 8 * n and pool.cached_bytes == 0
    del big
    pool.trim()
    assert not fake.live


def test_release_never_blocks_while_the_pool_lock_is_held(fake):
    pool = hostmem.PinnedPool()
    a = pool.empty((hostmem.PINNED_MIN_BYTES,), np.uint8)
    with pool._lock:                      # a finaliser that fires inside _take must not deadlock: it frees instead
        del a
        gc.collect()
    assert pool.cached_bytes == 0 and not fake.live


class _FakeGen:
    made = 0

    def __init__(self, device=0):
        type(self).made += 1
        self.device = device
        self._ctx = object()
        self._knobs_touched = False
        self._peak_groups = 0
        self.closed = False

    def close(self):
        self.closed = True
        self._ctx = None


def test_context_pool_reuses_per_thread_and_drops_modified_contexts():
    hostmem.drop_idle_contexts()
    _FakeGen.made = 0
    with hostmem.borrow_context(_FakeGen, 0) as g1:
        pass
    with hostmem.borrow_context(_FakeGen, 0) as g2:
        assert g2 is g1                                   # idle context reused
        with hostmem.borrow_context(_FakeGen, 0) as g3:   # nested borrow: a second context
            assert g3 is not g1
    assert _FakeGen.made == 2 and len(hostmem._idle((_FakeGen, 0))) == 2
    with hostmem.borrow_context(_FakeGen, 1) as other:    # keyed by device
        assert other is not g1 and other.device == 1
    g = hostmem.acquire_context(_FakeGen, 0)
    g._knobs_touched = True                               # tuning knobs changed: not kept
    hostmem.release_context(g)
    assert g.closed
    g = hostmem.acquire_context(_FakeGen, 0)
    g._peak_groups = hostmem._MAX_IDLE_GROUPS + 1         # grew large: not kept
    hostmem.release_context(g)
    assert g.closed
    with pytest.raises(RuntimeError):
        with hostmem.borrow_context(_FakeGen, 0) as g4:
            raise RuntimeError("boom")
    assert g4.closed                                      # an error may have left it in any state
    seen = []
    t = threading.Thread(target=lambda: seen.append(hostmem.acquire_context(_FakeGen, 0)))
    t.start()
    t.join()
    assert all(seen[0] is not x for x in hostmem._idle((_FakeGen, 0)))   # pools are per thread
    hostmem.drop_idle_contexts()
    assert not hostmem._idle((_FakeGen, 0))
