"""GPU: the vocabulary-shard device path (csvd_shard_open / csvd_shard_dense)
against the oracle's per-rank merge record, and the full sharded step with two
real processes sharing the B200 (gloo carries the tiny merge records)."""

import os
import socket

import numpy as np
import pytest

from conftest import TRANS_RTOL, assert_outcome, close, has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a GPU")]


def _setup(V=20000, d=512, n_modes=40, g=3, dtype="f32"):
    from paper_2511_21702_b200 import workload as wl
    T = wl.synth_vocab(V, d, n_modes, 0.3, 1, dtype=dtype)
    ix = wl.fast_index(T, n_modes, g)
    qs = np.vstack([wl.generate_queries(3, d, "contextual", 7, centroids=ix.centroids),
                    wl.generate_queries(1, d, "random", 9)])
    return T, ix, qs


EXACT = ("MIN", "MAX", "NTOK", "NLIST", "P_LO", "P_HI", "P_SEL", "CUM_LO", "CUM_HI", "U_NEXT", "QNORM", "SLACK")


def _cmp_record(got, exp, k, where):
    from paper_2511_21702_b200 import distributed as Dm
    for name in EXACT:
        i = getattr(Dm, "SH_" + name)
        assert got[i] == exp[i], f"{where}: {name} {got[i]!r} != {exp[i]!r}"
    for name in ("LSE", "LRH_NEXT"):
        i = getattr(Dm, "SH_" + name)
        assert close(float(got[i]), float(exp[i]), TRANS_RTOL), f"{where}: {name} {got[i]!r} vs {exp[i]!r}"
    nl = int(exp[Dm.SH_NLIST])
    assert np.array_equal(np.sort(got[Dm.SH_TOPK:Dm.SH_TOPK + nl]), np.sort(exp[Dm.SH_TOPK:Dm.SH_TOPK + nl])), \
        f"{where}: top-k lists differ"


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_shard_records_match_oracle(dtype):
    import paper_2511_21702_b200 as P
    from paper_2511_21702_b200 import distributed as Dm, engine, shard
    from shard_oracle import OracleShard
    T, ix, qs = _setup(dtype=dtype)
    for strategy in ("contiguous", "round_robin"):
        plan = shard.contiguous_plan(ix, 2) if strategy == "contiguous" else shard.make_plan(ix, 2)
        for r in range(2):
            owned = np.asarray(plan.assignment) == r
            dev, ora = Dm.DeviceShard(T, ix, owned, 0), OracleShard(T, ix, owned)
            for cfg in (P.DecodeConfig(k=10), P.DecodeConfig(k=40, k_max=900)):
                cs = engine.config_struct(cfg, ix.vocab_size, None, P._lib.VARIANT_BATCHSELECT)
                for i, h in enumerate(qs):
                    for lo, hi in ((0, 0), (3, 9)):
                        g = dev.open(h, cs, lo, hi)
                        e = ora.open(h, cs, lo, hi)
                        where = f"{dtype}/{strategy}/r{r}/k{cfg.k}/q{i}/[{lo},{hi})"
                        _cmp_record(g[0], e[0], cfg.k, where)
                        for a, b, nm in zip(g[1:], e[1:], ("positions", "ids", "logits")):
                            assert np.array_equal(a, b), f"{where}: {nm} differ"
                    gd, ed = dev.dense(h, cfg.k), ora.dense(h, cfg.k)
                    nl = int(ed[0][Dm.SH_NLIST])
                    assert gd[0][Dm.SH_NTOK] == ed[0][Dm.SH_NTOK] and gd[0][Dm.SH_NLIST] == nl
                    assert np.array_equal(np.sort(gd[0][Dm.SH_TOPK:Dm.SH_TOPK + nl]),
                                          np.sort(ed[0][Dm.SH_TOPK:Dm.SH_TOPK + nl]))
                    assert np.array_equal(gd[1], ed[1]) and np.array_equal(gd[2], ed[2])
            dev.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        import torch
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import csvd_oracle as O
        import paper_2511_21702_b200 as P
        from paper_2511_21702_b200 import shard
        from test_distributed import _fields
        T, ix, qs = _setup()
        plan = shard.contiguous_plan(ix, world)
        n = 0
        for cfg in (P.DecodeConfig(k=10), P.DecodeConfig(k=5, k_max=400), P.DecodeConfig(k=8, k_max=60)):
            for i, h in enumerate(qs):
                got, ledger = P.sharded_decode_step(T, ix, plan, h, cfg)  # the public API
                exp = O.decode_step_batchselect(T, ix, h, cfg)
                assert_outcome(got, _fields(exp), rtol=TRANS_RTOL, where=f"[{cfg.k},{i}] rank {rank}")
                assert ledger.bytes_bounds_phase == ix.n_clusters * 4
                n += 1
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok", n))
    except Exception:
        import traceback
        q.put((rank, "fail", traceback.format_exc()))


def test_sharded_step_two_processes_one_gpu():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, info in res:
        assert status == "ok", f"rank {rank}:\n{info}"
