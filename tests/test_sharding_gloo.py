"""Multi-process (gloo, world size 2, CPU) check of the utterance sharding:
sharded decode + host gather equals the unsharded decode.  The per-shard
decoder here is the CPU oracle (this runs without a GPU); on the B200 the same
host logic wraps the CUDA decoder (bench.py --gpus N)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2406_03791_b200.sharding import shard_range, sort_by_length


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2406_03791_b200.sharding import decode_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = O.random_case(17, False)
    x = np.concatenate([c.x] * 3)
    lens = np.concatenate([c.out_len] * 3)

    def dec(xs, ls):
        return [(h.tokens, h.frames) for h in O.decode_batch(c.dims, c.params, xs, ls, c.max_symbols, False)]

    out = decode_sharded(dec, x, lens, rank, world)
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_covers_batch():
    for B in (1, 7, 32, 256):
        for W in (1, 2, 3, 8):
            rs = [shard_range(B, r, W) for r in range(W)]
            assert rs[0][0] == 0 and rs[-1][1] == B
            assert all(rs[i][1] == rs[i + 1][0] for i in range(W - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_sort_by_length():
    assert sort_by_length([3, 9, 1, 9]) == [1, 3, 0, 2]


def test_gloo_two_ranks_match_unsharded():
    from oracle import oracle as O
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = O.random_case(17, False)
    x = np.concatenate([c.x] * 3)
    lens = np.concatenate([c.out_len] * 3)
    ref = [(h.tokens, h.frames) for h in O.decode_batch(c.dims, c.params, x, lens, c.max_symbols, False)]
    assert out == ref
