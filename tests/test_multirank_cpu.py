"""N > 1 host path on CPU (gloo, world size 2): replicas own the streams g with g mod N = rank,
run their rounds, exchange fixed-size per-round record blocks with an all-gather (the a6 step,
NCCL on GPU) and merge them with libseed's token table.  Every rank must end with every
stream's tokens, identical to a world-size-1 run (world-size invariance): the RNG is
keyed by global ids and stream-local rounds.  The per-rank rounds are the oracle's (no GPU here).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import seedgen
from oracle import llama as ll
from oracle.seed_round import SeedOracle

GAMMA, MAX_NEW, N_STREAMS, C = 4, 12, 4, 4


def _oracle(prompts, ids):
    cfg = seedgen.CONFIGS["toy"]
    ds, ts = seedgen.SHAPES[cfg["draft"]], seedgen.SHAPES[cfg["target"]]
    o = SeedOracle(ll.LlamaShape(**ts), seedgen.model_weights(ts, seedgen.TARGET_SEED), ll.LlamaShape(**ds),
                   seedgen.model_weights(ds, seedgen.DRAFT_SEED), gamma=GAMMA, temperature=1.0,
                   seed=seedgen.PHILOX_SEED, max_new=MAX_NEW)
    for g in ids:
        o.add_stream(g, prompts[g])
    return o


def _prompts():
    return seedgen.prompts("toy", n_streams=N_STREAMS - 1) + [[7, 8, 9, 10, 11, 12]]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.scheduler import RoundScheduler
    from paper_2406_18200_b200 import TokenTable
    prompts = _prompts()
    mine = [g for g in range(N_STREAMS) if g % world == rank]
    orc = _oracle(prompts, mine)
    sched = RoundScheduler(mine)
    table = TokenTable(GAMMA)
    stride = GAMMA + 3
    while True:
        busy = torch.tensor([0 if sched.all_done() else 1])
        dist.all_reduce(busy)
        if busy.item() == 0:
            break
        block = np.full((C, stride), -1, dtype=np.int32)      # fixed-size per-rank record block
        if not sched.all_done():
            batch = sched.schedule(C)
            before = {g: len(orc.streams[g].T) for g in batch}
            orc.round(batch)
            for b, g in enumerate(batch):
                st = orc.streams[g]
                new = st.T[before[g]:]
                block[b, 0], block[b, 1] = g, len(new)
                block[b, 2:2 + len(new)] = new
            sched.complete(batch, [orc.streams[g].done for g in batch])
        out = [torch.empty((C, stride), dtype=torch.int32) for _ in range(world)]
        dist.all_gather(out, torch.from_numpy(block))
        table.merge(torch.stack(out).numpy())
    q.put((rank, {g: table.get(g) for g in range(N_STREAMS)}))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def lib():
    from paper_2406_18200_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2406_18200_b200 import build
        build.build()
    return _lib.load()


def test_world_size_invariance_gloo(lib):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # world size 1 reference
    prompts = _prompts()
    orc = _oracle(prompts, range(N_STREAMS))
    ref, _, _ = orc.run(C)
    for rank in (0, 1):
        for g in range(N_STREAMS):
            assert res[rank][g] == ref[g], (rank, g)
            assert len(ref[g]) == MAX_NEW
