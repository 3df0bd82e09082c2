"""N > 1 host-side path on CPU: world_size-2 (and 3) gloo process groups.

Each rank takes its DP partition of the lex order (the same fs_plan partition the kernels
use), computes its partial with the host model of the kernels' lane code (no GPU here), and
the partials are combined with the SAME combine functions the NCCL path uses
(paper_2405_07989_b200.dist): all_reduce(SUM) for count/histogram, all_reduce(MAX) for the
any flag, all_gather of row counts -> exclusive offsets checked against the DP."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_07989_b200 import _lib as L


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2405_07989_b200 import dist as fsdist
        from tests.fsdbg import host_model

        res = []
        for n, g in cases:
            r = host_model(n, g, L.FS_CONSUMER_COUNT, rank=rank, world=world, want_hist=True)
            t = torch.tensor([r["count"]], dtype=torch.int64)
            fsdist.combine_sum(t)
            h = torch.tensor(r["hist"], dtype=torch.int64)
            fsdist.combine_sum(h)
            rr = host_model(n, g, L.FS_CONSUMER_ROWS, rank=rank, world=world, want_rows=True, B=16)
            counts = fsdist.gather_counts(rr["count"], torch.device("cpu"))
            offs = fsdist.exclusive_offsets(counts)
            assert offs[rank] == rr["info"]["row_begin"]
            # gather the row blocks to rank 0 and compare with the oracle there
            blocks = [None] * world
            dist.all_gather_object(blocks, rr["rows"])
            # any: a length predicate satisfied only by the lex-last row
            last = oracle.rows_as_tuples(oracle.rows(n, g, B=32), len(g), 32)
            f = torch.tensor([0], dtype=torch.int32)
            if last:
                tgt = last[-1]
                mine = oracle.rows_as_tuples(rr["rows"], len(g), 16)
                f[0] = int(tuple(tgt) in set(mine))
            fsdist.combine_max(f)
            res.append((int(t.item()), [int(x) for x in h], b"".join(blocks), int(f.item()), bool(last)))
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


CASES = [(1000, (6, 9, 20)), (600, (11, 13, 17, 19, 23)), (300, (3, 5, 7, 11)), (0, (4, 6)), (7, (4, 6)),
         (200, (20, 6, 9)), (12, (4,))]


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_combine(oracle_mod, world):
    import oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for (n, g), (cnt, hist, rows, found, nonempty) in zip(CASES, res):
        want = oracle.run(n, g, hist_len=oracle.hist_len_for(n, g))
        assert cnt == want["count"]
        assert hist == want["hist"]
        assert rows == oracle.rows(n, g, B=16)
        assert found == int(nonempty)
