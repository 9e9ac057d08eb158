"""Vocabulary-sharded decoding across real ranks (world_size 2, gloo, CPU).

Each rank owns half the clusters; per-rank device work is stood in for by the
oracle (tests/shard_oracle.py) so the distributed merge, certification and
fallback chain of paper_2511_21702_b200.distributed run for real across two
processes.  Contract (tests/test_acceptance.py:142-161 of the reference): the
sharded outcome equals decode_step_batchselect for every placement strategy.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import TRANS_RTOL, assert_outcome


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fields(o):
    st = o.stats
    return dict(ids=o.token_ids, logits=o.logits, kind=o.status.kind, fallback=o.fallback_used,
                sub_size=st["sub_size"], clusters_opened=st["clusters_opened"], heap_pops=st["heap_pops"],
                flops_sparse=st["flops_sparse"], flops_bounds=st["flops_bounds"], eps=o.status.epsilon_achieved,
                u_max=o.status.u_max, topk_min=o.status.topk_min, rho=st["rho"], xi=st["xi"], ratio=st["ratio"])


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import csvd_oracle as O
        import paper_2511_21702_b200 as P
        from paper_2511_21702_b200 import distributed as Dm, shard, workload as wl
        from shard_oracle import OracleShard

        T = wl.synth_vocab(3000, 64, 12, 0.3, 1)
        ix = wl.fast_index(T, 12, 3)
        qs = np.vstack([wl.generate_queries(3, 64, "contextual", 7, centroids=ix.centroids),
                        wl.generate_queries(1, 64, "random", 9)])
        cfgs = [P.DecodeConfig(k=10), P.DecodeConfig(k=5, k_max=400),
                P.DecodeConfig(k=4, epsilon=0.2, targets=("softmax_eps",), k_max=250),
                P.DecodeConfig(k=3, epsilon=0.1, targets=("topp",), k_max=300),
                P.DecodeConfig(k=8, k_max=60)]
        n = 0
        seen = set()
        for strategy in ("contiguous", "round_robin"):
            plan = shard.contiguous_plan(ix, world) if strategy == "contiguous" else shard.make_plan(ix, world)
            comm = Dm.TorchComm()
            dec = Dm.ShardedDecoder(T, ix, plan, comm=comm,
                                    backend=OracleShard(T, ix, np.asarray(plan.assignment) == rank))
            for ci, cfg in enumerate(cfgs):
                for i, h in enumerate(qs):
                    got = dec.step(h, cfg)
                    exp = O.decode_step_batchselect(T, ix, h, cfg)
                    assert_outcome(got, _fields(exp), rtol=TRANS_RTOL, where=f"{strategy}[{ci},{i}] rank {rank}")
                    seen.add((got.status.kind, got.fallback_used))
                    n += 1
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok", (n, sorted(seen, key=str))))
    except Exception as e:  # report to the parent
        import traceback
        q.put((rank, "fail", traceback.format_exc()))


def test_sharded_step_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, info in res:
        assert status == "ok", f"rank {rank}:\n{info}"
    n, seen = res[0][2]
    assert n > 0
    fbs = {fb for _, fb in seen}
    # the query/config mix exercises the merge and every fallback level
    assert {None, "partial_expand", "full_vocab"} <= fbs, seen


def _worker_api(rank, world, port, q):
    """shard.sharded_decode_step(..., group=pg): the opt-in distributed path
    of the reference call site, with the rank's device work stood in for by
    the oracle shard; the inputs digest check rejects mismatched queries."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import csvd_oracle as O
        import paper_2511_21702_b200 as P
        from paper_2511_21702_b200 import distributed as Dm, shard, workload as wl
        from shard_oracle import OracleShard

        T = wl.synth_vocab(2000, 64, 10, 0.3, 1)
        ix = wl.fast_index(T, 10, 2)
        plan = shard.contiguous_plan(ix, world)
        Dm.DeviceShard = lambda table, index, owned, dev: OracleShard(table, index, owned)  # no GPU here
        h = wl.generate_queries(2, 64, "contextual", 7, centroids=ix.centroids)
        cfg = P.DecodeConfig(k=10)
        out, ledger = shard.sharded_decode_step(T, ix, plan, h[0], cfg, group=dist.group.WORLD)
        exp = O.decode_step_batchselect(T, ix, h[0], cfg)
        assert_outcome(out, _fields(exp), rtol=TRANS_RTOL, where=f"api rank {rank}")
        assert ledger.bytes_bounds_phase > 0
        try:  # ranks disagree on the query: refused on every rank
            shard.sharded_decode_step(T, ix, plan, h[rank], cfg, group=dist.group.WORLD)
            q.put((rank, "fail", "mismatched queries were accepted"))
        except ValueError:
            q.put((rank, "ok", None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, "fail", traceback.format_exc()))


def test_sharded_decode_step_api_group_opt_in():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_api, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, info in res:
        assert status == "ok", f"rank {rank}:\n{info}"
