"""Fake engine for the one-process-per-GPU runtime (TEST DOUBLE, never shipped).

``FakeEngine`` with node-shared arenas: each rank's arena is a /dev/shm file, so a peer's
"IPC-opened" arena is the same bytes mapped into another process; flags are plain shared
memory; a remote copy is not runnable until the holder's flag is raised (the GPU's
cuStreamWaitValue32), exactly the cross-process ordering the runtime relies on."""

from __future__ import annotations

import mmap
import os

import numpy as np

from fake_engine import FakeEngine


def _shm_array(path, nbytes, create):
    if create:
        fd = os.open(path, os.O_RDWR | os.O_CREAT | os.O_TRUNC, 0o600)
        os.ftruncate(fd, nbytes)
    else:
        fd = os.open(path, os.O_RDWR)
    try:
        mm = mmap.mmap(fd, nbytes)
    finally:
        os.close(fd)
    return np.frombuffer(mm, dtype=np.float64)


class SpmdFakeEngine(FakeEngine):
    """A real GPU keeps executing its streams while the host sleeps; the base fake only
    advances inside engine calls.  Across processes that matters: a holder that has retired
    its last task may still have the arrival-flag write behind its final H2D queued, and a
    peer waits on that flag.  A daemon thread therefore keeps stepping the queues."""

    def __init__(self, rank, job, seed=0):
        super().__init__(1, seed=seed)
        import threading
        import time
        self._stop = False

        def progress():
            while not self._stop:
                with self._lock:
                    stepped = self._step()
                if not stepped:
                    time.sleep(2e-4)
        self._progress = threading.Thread(target=progress, daemon=True)
        self._progress.start()
        self.cuda_ids = [rank]
        self.rank = rank
        self.job = job
        self._gen = 0
        self._files = []
        self._remote = {}        # token base -> float64 array of a peer arena
        self._mapped = {}        # token base -> uint32 array (flags)
        self._next_tok = 1

    def ensure_arenas(self, caps):
        for slot, c in caps.items():
            if c > self._arena_cap[slot]:
                self._gen += 1
                path = f"/dev/shm/bxfake_{self.job}_r{self.rank}_g{self._gen}"
                nbytes = (c + 7) // 8 * 8
                self.arenas[slot] = _shm_array(path, nbytes, True)
                self._files.append(path)
                self._arena_cap[slot] = c

    def ipc_export(self, slot):
        path = self._files[-1].encode()
        return path.ljust(64, b"\0"), self._arena_cap[slot]

    def ipc_open(self, slot, handle):
        path = handle.rstrip(b"\0").decode()
        arr = _shm_array(path, os.path.getsize(path), False)
        base = self._next_tok << 40
        self._next_tok += 1
        self._remote[base] = arr
        return base

    def ipc_close(self, slot, base):
        self._remote.pop(base, None)

    def register_mapped(self, array):
        # any page-locked host range (the runtime maps a whole call file); flags are the
        # uint32 words at dptr offsets from its base
        base = (1 << 56) + (self._next_tok << 40)
        self._next_tok += 1
        self._mapped[base] = array.view(np.uint8).reshape(-1)
        return base

    def unregister_host(self, array):
        for b, a in list(self._mapped.items()):
            if a.ctypes.data == array.ctypes.data:
                del self._mapped[b]
                return
        super().unregister_host(array)

    def _flag(self, dptr):
        for b, a in self._mapped.items():
            if b <= dptr < b + a.nbytes:
                assert (dptr - b) % 4 == 0, "misaligned flag"
                return a[:a.nbytes // 4 * 4].view(np.uint32), (dptr - b) // 4
        raise AssertionError(f"unmapped flag address {dptr:#x}")

    def copy_remote(self, slot, dst_off, src_ptr, nbytes, flag_dptr=0, flag_min=0, waits=()):
        with self._lock:
            base = src_ptr & ~((1 << 40) - 1)
            src = self._remote[base]
            soff = src_ptr - base
            cond = None
            if flag_dptr:
                arr, i = self._flag(flag_dptr)
                cond = lambda: int(arr[i]) >= flag_min   # noqa: E731

            def fn():
                assert soff % 8 == 0 and dst_off % 8 == 0
                self.arenas[slot][dst_off // 8:(dst_off + nbytes) // 8] = src[soff // 8:(soff + nbytes) // 8]
            return self._enqueue(slot, -3, fn, waits, cond=cond)

    def write_flag(self, slot, lane, flag_dptr, value, waits=()):
        with self._lock:
            arr, i = self._flag(flag_dptr)

            def fn():
                arr[i] = value
            self._enqueue(slot, lane, fn, waits)

    def cleanup(self):
        self._stop = True
        for p in self._files:
            try:
                os.unlink(p)
            except OSError:
                pass
