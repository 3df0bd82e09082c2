"""GPU: the multi-rank execution path (paper_2405_07989_b200.dist) end to end.

Two (and three) processes, one rank each, share the one GPU of the test box with the gloo
backend (FS_DIST_BACKEND=gloo; device partials are staged through the host).  Every rank
runs its contiguous lex range of the instance in the CUDA kernels (PAPER.md:196-200 bounds,
P:230-231 distributed workers) and the partials are combined by the same dist.* functions
the NCCL path uses.  Results are checked at rank 0 against the oracle (C1, C2) and the
oracle-written golden fixtures (C4 = C3 histogram, C5).  A torchrun launch of bench.py with
2 ranks checks the bench's multi-rank line."""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


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
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2405_07989_b200 import _lib as L
        from paper_2405_07989_b200 import dist as fsdist
        from paper_2405_07989_b200 import workloads as W

        out = {}
        for inst in (W.C1, W.C2, W.C4, W.C5):
            out[inst.name] = {"count": fsdist.count(inst.n, inst.gens),
                              "hist": [int(x) for x in fsdist.length_set(inst.n, inst.gens).cpu().tolist()]}
        # forced small slices: many slices per rank, ragged rank ends
        out["C2_T3"] = {"count": fsdist.count(W.C2.n, W.C2.gens, slice_units=3),
                        "hist": [int(x) for x in fsdist.length_set(W.C2.n, W.C2.gens, slice_units=3).cpu().tolist()]}
        # any: C5 predicates (P_late: only the lex-last row; P_none; P_first)
        out["any"] = [fsdist.any_pred(W.C5.n, W.C5.gens, L.FS_PRED_LEN_LE, 20),
                      fsdist.any_pred(W.C5.n, W.C5.gens, L.FS_PRED_LEN_LE, 19),
                      fsdist.any_pred(W.C5.n, W.C5.gens, L.FS_PRED_LEN_GE, 19995),
                      fsdist.any_pred(W.C1.n, W.C1.gens, L.FS_PRED_COORD_GE, (2 << 32) | 50),
                      fsdist.any_pred(W.C1.n, W.C1.gens, L.FS_PRED_COORD_GE, (2 << 32) | 51)]
        # rows: each rank's canonical block, gathered to rank 0 in rank order
        blocks = {}
        for inst, B, T in ((W.C1, 16, 0), (W.C2, 16, 0), (W.C2, 32, 64)):
            off, rows, t = fsdist.enumerate_rows(inst.n, inst.gens, B=B, slice_units=T)
            mine = (off, rows, t.contiguous().cpu().numpy().tobytes())
            allb = [None] * world
            dist.all_gather_object(allb, mine)
            blocks["%s_%d_%d" % (inst.name, B, T)] = allb
        out["rows"] = blocks
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def _gold(name):
    with open(os.path.join(GOLD, name + ".json")) as f:
        return json.load(f)


@pytest.mark.parametrize("world", [2, 3])
def test_dist_paths_on_one_gpu(oracle_mod, world):
    import torch.multiprocessing as mp

    import oracle
    from paper_2405_07989_b200 import workloads as W

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=900)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for inst in (W.C1, W.C2):
        want = oracle.run(inst.n, inst.gens, hist_len=oracle.hist_len_for(inst.n, inst.gens))
        assert res[inst.name]["count"] == want["count"]
        assert res[inst.name]["hist"] == want["hist"]
    want = oracle.run(W.C2.n, W.C2.gens, hist_len=oracle.hist_len_for(W.C2.n, W.C2.gens))
    assert res["C2_T3"] == {"count": want["count"], "hist": want["hist"]}
    for name, gname in (("C4", "C3"), ("C5", "C5")):
        g = _gold(gname)
        assert res[name]["count"] == g["count"]
        assert res[name]["hist"] == [int(x) for x in g["hist"]]
    assert res["any"] == [True, False, True, True, False]  # C1: max a_3 = 50
    for key, blocks in res["rows"].items():
        name, B, T = key.split("_")
        inst = {"C1": W.C1, "C2": W.C2}[name]
        offs = [b[0] for b in blocks]
        counts = [b[1] for b in blocks]
        assert offs == [sum(counts[:r]) for r in range(world)]
        assert b"".join(b[2] for b in blocks) == oracle.rows(inst.n, inst.gens, B=int(B))


def test_torchrun_bench_two_ranks_gloo():
    """`torchrun --nproc-per-node 2 bench.py --gpus 2` on a one-GPU box (gloo, ranks share the
    device): a valid JSON line from rank 0 with n_gpus = 2 and the exact total."""
    env = dict(os.environ, FS_DIST_BACKEND="gloo", FS_BENCH_QUICK="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-extra"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["steps"] == 3
    assert line["value"] > 0 and line["config"]["instance"] == "C3"
    assert line["plan"]["dist_backend"] == "gloo"
    assert line["plan"]["rank_units"] and len(line["plan"]["rank_units"]) == 2
