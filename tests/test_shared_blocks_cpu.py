"""distributed.SharedBlocks on CPU (the page-locking call stubbed): the
node-shared result blocks of render(distributed=True) are /dev/shm files every
rank maps; rank 0 hands a block out again only once no array it returned
views it, and removes the files at the end."""

import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


class _FakeLib:
    """tr_host_register / tr_host_unregister without a GPU: the device
    address is the host address (UVA)."""

    def __init__(self):
        self.registered = set()

    def tr_host_register(self, host, nbytes, dptr):
        addr = host.value
        self.registered.add(addr)
        C.cast(dptr, C.POINTER(C.c_void_p))[0] = addr
        return 0

    def tr_host_unregister(self, host):
        self.registered.discard(host.value)
        return 0


@pytest.fixture
def fake_lib(monkeypatch):
    from paper_1908_01906_b200 import _lib
    fake = _FakeLib()
    monkeypatch.setattr(_lib, "lib", lambda: fake)
    return fake


@pytest.mark.skipif(not os.path.isdir("/dev/shm"), reason="no /dev/shm")
def test_blocks_are_shared_recycled_and_removed(fake_lib):
    from paper_1908_01906_b200.distributed import SharedBlocks
    token = f"test_{os.getpid()}"
    try:
        _check(SharedBlocks, token, fake_lib)
    finally:   # a failed run leaves no files behind
        for i in range(8):
            try:
                os.unlink(f"/dev/shm/tetray_b200_{token}_4096_{i}")
            except OSError:
                pass


def _check(SharedBlocks, token, fake_lib):
    r0 = SharedBlocks(token, 4096, 0)   # creates block 0
    r1 = SharedBlocks(token, 4096, 1)   # another rank: maps what rank 0 created
    b0, d0 = r0.block(0)
    assert d0 == b0.ctypes.data and d0 in fake_lib.registered
    o0, _ = r1.block(0)
    o0[:8] = np.arange(8, dtype=np.uint8)          # rank 1 writes its tiles ...
    assert np.array_equal(b0[:8], np.arange(8))    # ... rank 0 sees them: one file
    # frame 0 returned (a view of block 0 is alive): the next frame gets a new block
    frame0 = b0[:16].view(np.float64)
    del b0, o0
    assert r0.pick_next() == 1 and os.path.exists(r0._path(1))
    r0.cur = 1
    # frame 1 returned too; frame 0 still held -> a third block
    frame1 = r0.block(1)[0][:16]
    assert r0.pick_next() == 2
    r0.cur = 2
    del frame0                                      # the caller dropped frame 0
    assert r0.pick_next() == 0                      # block 0 is handed out again
    del frame1
    r1.close()
    paths = [r0._path(i) for i in range(len(r0.blocks))]
    r0.close()
    assert not any(os.path.exists(p) for p in paths)
    assert not fake_lib.registered
