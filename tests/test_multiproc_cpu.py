"""World-size-2 `gloo` tests of the N>1 host path, on CPU (no GPU needed).

One process per rank, as torchrun launches bench.py on the box.  What runs
without a GPU is exactly the host logic in front of the device: the
bootstrap allgather adapter (Comm.create's callback), the collective config
check (runtime.cpp:86-105 -> CONFIG_MISMATCH), and the per-rank sharding of
the MoE workload (each rank owns E/n experts, harness_moe.cpp:109, 147-148):
per-rank routing gathered over gloo equals the global count table."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def _allgather_fn(dist, world):
    def ag(blob):
        out = [None] * world
        dist.all_gather_object(out, blob)
        return out
    return ag


def _worker_config(rank, world, port, q, mismatch):
    sys.path.insert(0, ROOT)
    dist = _init(rank, world, port)
    import paper_2511_15076_b200 as G
    cfg = G.Config(queue_depth=512 if (mismatch and rank == 1) else 1024)
    try:
        G.Comm.create(rank, world, 0, _allgather_fn(dist, world), cfg)
        q.put((rank, "created"))
    except G.ConfigMismatch as e:
        q.put((rank, "ConfigMismatch:" + str(e)))
    except G.Error as e:  # past the config check, the first device call fails on a CPU box
        q.put((rank, type(e).__name__))
    dist.destroy_process_group()


def _worker_shard(rank, world, port, q):
    sys.path.insert(0, ROOT)
    dist = _init(rank, world, port)
    from oracle import oracle as O
    seed, E, K, T = 1, 256, 8, 128
    idx = O.route_table(seed, E, K, rank, T)          # this rank's routing only
    mine = np.bincount(idx.reshape(-1), minlength=E).astype(np.uint32)
    parts = [None] * world
    dist.all_gather_object(parts, mine.tobytes())
    table = np.stack([np.frombuffer(p, np.uint32) for p in parts], axis=1)   # [E, src]
    e_local = E // world
    owned = table[rank * e_local:(rank + 1) * e_local]                       # what this rank receives
    q.put((rank, table.tobytes(), int(owned.sum()), int(mine.sum())))
    dist.destroy_process_group()


def _run(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


@pytest.mark.parametrize("mismatch", [True, False])
def test_bootstrap_config_check_over_gloo(mismatch):
    """comm_init's collective config equality over a real 2-process bootstrap:
    differing configs raise ConfigMismatch on every rank before any device
    call; equal configs pass the check and reach the device allocation (which
    fails loudly on this GPU-less box -- no CPU fallback)."""
    res = _run(_worker_config, 2, mismatch)
    for rank, what in res:
        if mismatch:
            assert what.startswith("ConfigMismatch"), (rank, what)
        else:
            assert what in ("CudaError", "created"), (rank, what)
            assert not what.startswith("ConfigMismatch")


def test_expert_sharding_gathered_counts_match_oracle():
    """Each rank routes only its own tokens; the gathered per-(expert, source)
    table equals the oracle's global counts, every rank sends T*K messages and
    the experts' owners receive all of them (the dispatch all-to-all's totals)."""
    from oracle import oracle as O
    world = 2
    res = _run(_worker_shard, world)
    full = O.counts(1, world, 256, 8, 128)
    for rank, table, owned, sent in res:
        assert (np.frombuffer(table, np.uint32).reshape(256, world) == full).all()
        assert sent == 128 * 8
    assert sum(r[2] for r in res) == world * 128 * 8
