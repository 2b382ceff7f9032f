"""world_size-2 gloo coverage of the multi-process plumbing bench.py uses for
N > 1 (max-over-ranks timing, summed token counts, barrier).  CPU only."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms = 10.0 + 5 * rank          # per-rank elapsed time
    toks = 100 + rank             # per-rank emitted tokens
    bench.barrier(world)
    q.put((rank, bench.reduce_max(ms, world), bench.reduce_sum(toks, world)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_bench_reductions_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for _, mx, sm in res:
        assert mx == 15.0            # max over ranks, not the rank's own time
        assert sm == 201.0           # value = tokens of all ranks / max time
