"""First-fit arena allocator over one device-memory reservation.

Same policy as the reference arena (/root/reference/pkg/src/tileblas/memory.py:32-153):
address-ordered first fit, the remainder of a split stays free, frees coalesce with free
neighbours, sizes are rounded up to the alignment, and an allocation that does not fit
raises the recoverable ``ArenaOutOfMemoryError`` (the tile cache then evicts).

On B200 the backing store is one ``cudaMalloc`` per device made by the engine
(``bx_init``); this class only hands out byte offsets into it.  The default alignment is
256 bytes (TMA / 16-byte vector staging of tile columns) instead of the reference's 64.
"""

from __future__ import annotations

import bisect

from .errors import ArenaOutOfMemoryError, InvalidArgumentError, InvalidFreeError

ALIGNMENT = 256


class Arena:
    def __init__(self, capacity: int, alignment: int = ALIGNMENT):
        if alignment < 1:
            raise InvalidArgumentError(f"alignment must be >= 1, got {alignment}")
        if capacity < alignment:
            raise InvalidArgumentError(
                f"arena capacity must be >= alignment ({alignment}), got {capacity}")
        self.capacity = capacity
        self.alignment = alignment
        self.reservations = 1
        self._free_off = [0]          # sorted offsets of free segments
        self._free_len = {0: capacity}
        self._used = {}               # offset -> length

    def aligned(self, nbytes: int) -> int:
        a = self.alignment
        return -(-nbytes // a) * a

    def alloc(self, nbytes: int) -> int:
        if nbytes < 1:
            raise InvalidArgumentError(f"alloc size must be >= 1, got {nbytes}")
        size = self.aligned(nbytes)
        for pos, off in enumerate(self._free_off):
            length = self._free_len[off]
            if length < size:
                continue
            del self._free_len[off]
            if length > size:
                self._free_off[pos] = off + size
                self._free_len[off + size] = length - size
            else:
                del self._free_off[pos]
            self._used[off] = size
            return off
        raise ArenaOutOfMemoryError(
            f"no free segment of {size} bytes (capacity {self.capacity})")

    def free(self, offset: int) -> None:
        size = self._used.pop(offset, None)
        if size is None:
            raise InvalidFreeError(f"offset {offset} is not an allocation start")
        pos = bisect.bisect_left(self._free_off, offset)
        start, length = offset, size
        # merge with the following free segment
        if pos < len(self._free_off) and self._free_off[pos] == offset + size:
            nxt = self._free_off.pop(pos)
            length += self._free_len.pop(nxt)
        # merge with the preceding free segment
        if pos > 0:
            prv = self._free_off[pos - 1]
            if prv + self._free_len[prv] == offset:
                self._free_len[prv] += length
                return
        self._free_off.insert(pos, start)
        self._free_len[start] = length

    # ---- introspection -------------------------------------------------------------

    def segments(self) -> list:
        """All segments in address order as (offset, length, occupied)."""
        segs = [(o, self._free_len[o], False) for o in self._free_off]
        segs += [(o, n, True) for o, n in self._used.items()]
        return sorted(segs)

    def free_segments(self) -> list:
        return [(o, self._free_len[o]) for o in self._free_off]

    def occupied_bytes(self) -> int:
        return sum(self._used.values())

    def largest_free(self) -> int:
        return max(self._free_len.values(), default=0)

    def check_invariants(self) -> None:
        pos, prev_free = 0, False
        for off, length, occ in self.segments():
            assert off == pos, f"gap/overlap at {off} (expected {pos})"
            assert length > 0
            if occ:
                assert length % self.alignment == 0
            assert not (prev_free and not occ), f"adjacent free segments at {off}"
            prev_free = not occ
            pos += length
        assert pos == self.capacity
