"""Arena allocator, ALRU cache and coherence directory: unit + property tests
(the reference's invariants: memory.py:132-153, cache.py SPEC invariants — directory equals
the union of the ALRUs after every operation, pinned blocks are never evicted)."""

import random
import threading

import pytest

from paper_1510_05041_b200.cache import (HOST_FETCH, L1_HIT, L2_HIT, CoherenceDirectory,
                                         DeviceTileCache, LruBlock)
from paper_1510_05041_b200.errors import (ArenaOutOfMemoryError, CapacityDeadlockError,
                                          InvalidArgumentError, InvalidFreeError,
                                          NotEvictableError)
from paper_1510_05041_b200.memory import Arena
from paper_1510_05041_b200.scheduler import TaskQueue
from paper_1510_05041_b200.tiling import TileRef


# ------------------------------------------------------------------------- arena

def test_arena_first_fit_split_and_coalesce():
    a = Arena(1024, alignment=64)
    x = a.alloc(100)            # 128
    y = a.alloc(64)
    z = a.alloc(200)            # 256
    assert (x, y, z) == (0, 128, 192)
    a.free(y)
    assert a.alloc(10) == 128   # first fit reuses the hole
    a.free(128)
    a.free(x)
    assert a.free_segments()[0] == (0, 192)   # coalesced with the freed neighbour
    a.check_invariants()


def test_arena_errors():
    a = Arena(256, alignment=64)
    with pytest.raises(InvalidArgumentError):
        a.alloc(0)
    a.alloc(256)
    with pytest.raises(ArenaOutOfMemoryError):
        a.alloc(1)
    with pytest.raises(InvalidFreeError):
        a.free(64)
    with pytest.raises(InvalidArgumentError):
        Arena(16, alignment=64)


def test_arena_random_ops_keep_invariants():
    rng = random.Random(7)
    a = Arena(1 << 16, alignment=256)
    live = []
    for _ in range(20000):
        if live and (rng.random() < 0.45 or len(live) > 40):
            a.free(live.pop(rng.randrange(len(live))))
        else:
            try:
                live.append(a.alloc(rng.randint(1, 6000)))
            except ArenaOutOfMemoryError:
                pass
        if _ % 97 == 0:
            a.check_invariants()
    for off in live:
        a.free(off)
    a.check_invariants()
    assert a.free_segments() == [(0, 1 << 16)]


# ------------------------------------------------------------------------- cache

class Fetch:
    """Fetch-protocol double: records traffic; copy_from_peer keeps no source pin."""

    def __init__(self):
        self.host = 0
        self.peer = 0
        self.syncs = 0
        self.pinned = []

    def copy_from_host(self, ref, blk):
        self.host += 1

    def copy_from_peer(self, src_cache, src_blk, ref, blk):
        self.peer += 1
        return False

    def pressure_sync(self):
        self.syncs += 1
        for cache, blk in self.pinned:
            cache.unpin(blk)
        self.pinned = []


def ref(i, j=0, mid="A"):
    return TileRef(mid, i, j, 4, 4, False)


def make(ndev=2, cap=8 * 256, group="g"):
    d = CoherenceDirectory()
    caches = [DeviceTileCache(i, Arena(cap, alignment=256), d, peer_group=group) for i in range(ndev)]
    return d, caches


def test_translate_l1_l2_host_and_recency():
    d, (c0, c1) = make()
    f = Fetch()
    b, o = c0.translate(ref(1), f, nbytes=256)
    assert o == HOST_FETCH and f.host == 1
    b2, o = c0.translate(ref(1), f, nbytes=256)
    assert o == L1_HIT and b2 is b
    b3, o = c1.translate(ref(1), f, nbytes=256)
    assert o == L2_HIT and f.peer == 1
    assert d.state(ref(1).key()) == "S"
    c0.translate(ref(2), f, nbytes=256)
    c0.translate(ref(1), f, nbytes=256)
    assert c0.recency_order()[0] == ref(1).key()


def test_peer_source_respects_groups_and_lowest_id():
    d = CoherenceDirectory()
    cs = [DeviceTileCache(i, Arena(4096, alignment=256), d, peer_group=g)
          for i, g in enumerate(["x", "x", "y", "x"])]
    for c in (cs[3], cs[2], cs[1]):
        blk = LruBlock(ref(5).key(), c.allocate(256), 256)
        c.insert_front(blk)
    assert d.peer_source(ref(5).key(), 0) == 1
    assert d.peer_source(ref(5).key(), 1) == 3
    assert d.peer_source(ref(5).key(), 2) is None     # other group only


def test_eviction_skips_pinned_and_deadlock_after_one_sync():
    d, (c0,) = make(1, cap=3 * 256)
    f = Fetch()
    blks = [c0.translate(ref(i), f, nbytes=256)[0] for i in range(3)]
    for b in blks:
        c0.pin(b)
    with pytest.raises(CapacityDeadlockError):
        c0.translate(ref(9), f, nbytes=256)
    assert f.syncs == 1
    c0.unpin(blks[1])
    b, o = c0.translate(ref(9), f, nbytes=256)
    assert ref(1).key() not in c0.keys()              # only the unpinned block left
    assert all(x.key in c0.keys() for x in (blks[0], blks[2]))


def test_write_back_asserts_no_holder():
    d, (c0,) = make(1)
    c0.translate(ref(3, mid="C"), Fetch(), nbytes=256)
    with pytest.raises(AssertionError):
        d.note_write_back(ref(3, mid="C").key())


@pytest.mark.parametrize("seed", range(6))
def test_cache_directory_fuzz(seed):
    """Random translate / pin / release over 3 devices with tiny arenas: the directory always
    equals the union of the ALRU contents and pinned blocks are never evicted."""
    rng = random.Random(seed)
    d, caches = make(3, cap=5 * 256)
    f = Fetch()
    pinned = {i: [] for i in range(3)}
    for step in range(3000):
        i = rng.randrange(3)
        c = caches[i]
        r = rng.random()
        if r < 0.6:
            try:
                blk, _ = c.translate(ref(rng.randrange(12)), f, nbytes=256)
            except CapacityDeadlockError:
                continue
            if rng.random() < 0.3 and len(pinned[i]) < 3:
                c.pin(blk)
                pinned[i].append(blk)
        elif pinned[i]:
            c.unpin(pinned[i].pop(rng.randrange(len(pinned[i]))))
        # invariants
        snap = d.snapshot()
        union = {}
        for cc in caches:
            for k in cc.keys():
                union.setdefault(k, set()).add(cc.device_id)
        assert snap == {k: frozenset(v) for k, v in union.items()}
        for j, lst in pinned.items():
            for blk in lst:
                assert blk.key in caches[j].keys()
        for cc in caches:
            cc.check_invariants()
            cc.arena.check_invariants()


# ------------------------------------------------------------------------- queue

def test_task_queue_exactly_once_under_threads():
    q = TaskQueue()
    n_prod, per = 4, 20000
    got = []
    lock = threading.Lock()

    def prod(p):
        for i in range(per):
            q.put((p * per + i, 0.0))

    def cons():
        mine = []
        while True:
            item = q.get()
            if item is None:
                if done.is_set() and len(q) == 0:
                    break
                continue
            mine.append(item[0])
        with lock:
            got.extend(mine)
    done = threading.Event()
    cs = [threading.Thread(target=cons) for _ in range(4)]
    ps = [threading.Thread(target=prod, args=(p,)) for p in range(n_prod)]
    for t in cs + ps:
        t.start()
    for t in ps:
        t.join()
    done.set()
    for t in cs:
        t.join()
    assert sorted(got) == list(range(n_prod * per))
