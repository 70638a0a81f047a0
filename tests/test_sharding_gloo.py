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


def _cuda_worker(rank, world, port, q):
    """decode_sharded over the CUDA decoder: both ranks share GPU 0."""
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2406_03791_b200 import DecodeAlgo, Model, ModelDims
    from paper_2406_03791_b200 import decoders as D
    from paper_2406_03791_b200.sharding import decode_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = O.Dims(150, 64, 64, 96, 24, (), O.CELL_LSTM, 2)
    p = O.init_params(41, d)
    B, T = 45, 12
    x = O.fill_uniform(42, -1.0, 1.0, (B, T, d.feature))
    lens = np.array([T - (5 * i) % 9 for i in range(B)], np.int32)
    m = Model(ModelDims(150, 64, 64, 96, 24, (), "lstm", 2), p, device=0)

    def dec(xs, ls):
        got = D.label_looping_decode(m, np.ascontiguousarray(xs), np.ascontiguousarray(ls), 3, D.Exec.Tensor)
        return [(list(h.tokens), list(h.frames), np.asarray(h.scores, np.float32).tobytes()) for h in got]

    out = decode_sharded(dec, x, lens, rank, world)
    if rank == 0:
        whole = dec(x, lens)
        q.put((out, whole))
    dist.barrier()
    m.close()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_cuda_sharded_decode_matches_unsharded():
    """SPEC.md:567 / SURVEY §8e: two ranks (gloo, sharing one B200) each decode
    their utterance range on the tensor-core executor; the host gather equals
    the unsharded decode bit for bit (rows are independent, model.hpp:89-91)."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_cuda_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out, whole = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert out == whole


@pytest.mark.gpu
def test_bench_spawns_ranks():
    """`python bench.py --gpus 2` launches 2 ranks itself (torch.distributed.run,
    gloo barriers, no NCCL); on a 1-GPU box they share the GPU."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RNNTG_BENCH_SHARE_GPU="1")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--config", "c5",
                        "--steps", "2", "--warmup", "1", "--no-compare", "--no-e2e", "--no-cpu-baseline"],
                       capture_output=True, text=True, env=env, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["parity"]["checked"] and line["parity"]["ranks_checked"] == 2
    assert line["parity"]["failures"] == 0
