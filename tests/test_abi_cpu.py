"""CPU-side checks of the C ABI (no GPU): the library loads, exports every declared symbol,
and its host pieces (FCFS scheduler H1, a6 token table) agree with the oracle.
"""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="session")
def lib():
    from paper_2406_18200_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2406_18200_b200 import build
        build.build()
    return _lib.load()


def _declared():
    names = set()
    for h in ("seed.h", "seed_ops.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names |= set(re.findall(r"SEED_API\s+[\w\s\*]+?\b(seed_\w+)\s*\(", src))
    return names


def test_exports_every_declared_symbol(lib):
    from paper_2406_18200_b200 import _lib
    declared = _declared()
    assert len(declared) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (seed_\w+)", out))
    assert declared <= exported, declared - exported
    assert set(_lib._SIGS) <= declared
    for name in declared:
        getattr(lib, name)


def test_no_torch_in_abi():
    for h in ("seed.h", "seed_ops.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        assert "torch" not in src.lower().replace("torch types", "")
        assert "at::" not in src and "Tensor" not in src


def test_init_without_gpu_fails_loudly(lib):
    import ctypes as C
    from paper_2406_18200_b200 import _lib
    cfg = _lib.Config()
    ctx = C.c_void_p()
    st = lib.seed_init(C.byref(cfg), C.byref(ctx))
    assert st != 0  # EINVAL for the empty config, ECUDA without a device: never a silent fallback


def test_scheduler_matches_oracle(lib):
    from oracle.scheduler import RoundScheduler
    from paper_2406_18200_b200 import Scheduler
    rng = np.random.default_rng(0)
    for trial in range(20):
        ids = rng.choice(1000, size=int(rng.integers(1, 12)), replace=False).tolist()
        a, b = Scheduler(ids), RoundScheduler(ids)
        for _ in range(40):
            if b.all_done():
                assert a.all_done()
                break
            cap = int(rng.integers(1, 6))
            x, y = a.pop(cap), b.schedule(cap)
            assert x == y
            done = [bool(rng.random() < 0.3) for _ in x]
            a.complete(x, done)
            b.complete(y, done)


def test_scheduler_liveness_and_errors(lib):
    from paper_2406_18200_b200 import Scheduler, SeedError
    s = Scheduler([3, 1, 2])
    assert s.pop(2) == [1, 2]
    assert s.pop(2) == [3]
    with pytest.raises(SeedError):
        s.pop(2)                       # nothing ready, work remains: liveness violation surfaced
    s.complete([1, 2, 3], [True, True, True])
    assert s.all_done() and s.pop(2) == []


def test_token_table_merge(lib):
    from paper_2406_18200_b200 import TokenTable
    g = 4
    t = TokenTable(g)
    recs = np.full((3, g + 3), -1, dtype=np.int32)
    recs[0, :4] = [7, 2, 11, 12]
    recs[1, :3] = [9, 1, 5]
    t.merge(recs)
    t.merge(np.array([[7, 3, 1, 2, 3, -1, -1]], dtype=np.int32))
    assert t.get(7) == [11, 12, 1, 2, 3] and t.get(9) == [5]


def test_scheduler_remove_then_readd(lib):
    """removing an undone stream and adding the same id again must leave one queue entry."""
    from paper_2406_18200_b200 import Scheduler
    s = Scheduler([1, 2])
    assert s.pop(1) == [1]
    s.complete([1], [False])               # 2, 1 queued
    assert lib.seed_sched_remove(s.h, 1) == 0
    s.add(1)                               # 2, 1 (fresh)
    assert s.pop(4) == [2, 1]
    s.complete([2, 1], [False, False])
    assert s.pop(4) == [2, 1]              # no stale duplicate of 1


def test_round_book_pack_complete(lib):
    """The exchange block: records [gid, c, tokens] with c truncated to l (R7), padding gid -1, and the
    rank's undone count after the round; completion commits, requeues and sums the pending counts."""
    from paper_2406_18200_b200 import RoundBook, SeedError
    g, l, cap = 2, 5, 3
    b = RoundBook(g, l, cap, world=2, rank=1)
    b.add(10, [3, 4])
    b.add(12, [3, 4, 5])
    b.add(14, [9, 9])
    with pytest.raises(SeedError):
        b.add(12, [1, 2])                 # duplicate id
    batch = b.schedule(2)
    assert batch == [10, 12]
    tok = np.array([[7, 8, 9], [6, -1, -1]], dtype=np.int32)
    blk = b.pack(batch, tok, [3, 1])
    stride = g + 3
    assert blk.size == cap * stride + 1
    assert blk[:stride].tolist() == [10, 3, 7, 8, 9]
    assert blk[stride:2 * stride].tolist() == [12, 1, 6, -1, -1]
    assert (blk[2 * stride:3 * stride] == -1).all()
    assert blk[-1] == 3                   # 14 not in the batch + 10, 12 still undone
    other = np.full(cap * stride + 1, -1, dtype=np.int32)
    other[:stride] = [11, 2, 1, 2, -1]
    other[-1] = 1
    b.complete(np.stack([other, blk]))
    assert b.global_pending() == 4
    assert b.tokens(10) == [7, 8, 9] and b.tokens(11) == [1, 2]
    assert b.info(10)["L"] == 3 and b.info(10)["r"] == 1
    # truncation to l: 10 has room 2
    batch = b.schedule(3)
    assert batch == [14, 10, 12]
    blk = b.pack(batch, np.array([[1, 1, 1], [5, 5, 5], [2, 2, 2]], dtype=np.int32), [1, 3, 3])
    assert blk[stride:stride + 2].tolist() == [10, 2]
    assert blk[-1] == 2                   # 10 done (3 + 2 = l); 14 (1 of 5), 12 (4 of 5) undone
    other[-1] = 0
    other[:stride] = -1
    b.complete(np.stack([other, blk]))
    assert b.global_pending() == 2 and b.info(10)["done"] == 1
    assert b.schedule(3) == [14, 12]
    # remove and re-add an undone id: no stale queue entry, fresh tokens
    b.remove(14)
    b.add(14, [8, 8])
    assert b.tokens(14) == []
    with pytest.raises(SeedError):
        b.complete(np.stack([other, other]))   # the own tail cannot be below the own undone count
