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


def _tp_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import synth
    from paper_2506_01986_b200 import tp_shard
    # handle exchange (bench.peer_syms' plumbing) with stand-in 64-byte handles
    hs = bench.exchange_handles(bytes([rank]) * 64, world)
    sh = tp_shard(synth.model_cfg("llama70b"), rank, world)
    shards = [None] * world
    dist.all_gather_object(shards, sh)
    q.put((rank, hs, shards))
    dist.destroy_process_group()


def test_tp_plumbing_gloo():
    """world 2: every rank gets every rank's handle in rank order, and the ranks'
    shards of the 70B shape tile heads, FFN features and vocabulary exactly."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for _, hs, shards in res:
        assert hs == [bytes([r]) * 64 for r in range(world)]
        for key, full in (("q_rows", 64 * 128), ("k_rows", 8 * 128), ("o_cols", 64 * 128), ("ffn", 28672),
                          ("vocab", 32000)):
            ranges = [s[key] for s in shards]
            assert ranges[0][0] == 0 and ranges[-1][1] == full
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))


def test_tp_shard_rejects_bad_sizes():
    import synth
    from paper_2506_01986_b200 import tp_shard
    with pytest.raises(ValueError):
        tp_shard(synth.model_cfg("llama70b"), 0, 3)
    with pytest.raises(ValueError):
        tp_shard(synth.model_cfg("tiny"), 0, 8)  # F = 256: 8 ranks x 64-row blocks do not fit


def _pp_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2506_01986_b200 as sm
    mine = list(sm.pp_layers(80, rank, world))       # the 70B shape's 80 layers
    got = [None] * world
    dist.all_gather_object(got, mine)
    q.put((rank, got))
    dist.destroy_process_group()


def test_pipeline_layer_partition_gloo():
    """f4 layer split ("equal-sized chunks"): the ranks' layer ranges, gathered over a
    world-size-2 gloo group, tile [0, L) in rank order with equal sizes; bad splits are refused."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for _, got in res:
        assert sum(got, []) == list(range(80)) and len({len(g) for g in got}) == 1
    import paper_2506_01986_b200 as sm
    for L, pp in [(80, 3), (2, 4)]:
        with pytest.raises(ValueError):
            sm.pp_layers(L, 0, pp)


def test_dist_struct_matches_header():
    """sm_dist in include/specmemo.h: pp_rank / pp_size follow peer_sym[SM_MAX_TP], then emu_group."""
    import ctypes

    import paper_2506_01986_b200 as sm
    assert sm.Dist.pp_rank.offset == 8 + 8 * sm.MAX_TP
    assert sm.Dist.emu_group.offset == 16 + 8 * sm.MAX_TP and ctypes.sizeof(sm.Dist) == 16 + 8 * sm.MAX_TP + 8
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                            "specmemo.h")).read()
    body = hdr[hdr.index("typedef struct {\n  int tp_rank, tp_size;"):hdr.index("} sm_dist;")]
    assert [ln.split()[1].rstrip(";").split("[")[0].lstrip("*") for ln in body.splitlines()[1:] if ln.strip()] == \
        ["tp_rank,", "peer_sym", "pp_rank,", "emu_group"]
