"""Run one hot-path kernel a few times for ncu captures (never a bench number).

  python profiles/workload.py <name> [reps]
  names: c3count c3closed c3auto c3autoclosed c4hist c5count c5any_none c2xl_m1 c2xl_m2 c2xl_m2auto
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("FS_PKG_ROOT", ROOT))

import torch  # noqa: E402

from paper_2405_07989_b200 import _lib as L  # noqa: E402
from paper_2405_07989_b200 import api  # noqa: E402
from paper_2405_07989_b200 import workloads as W  # noqa: E402


def build(name):
    """A callable launching the workload once."""
    if name.startswith("c3autoclosed_w"):  # rank r of a W-way partition: c3autoclosed_w8r0
        world, rank = (int(x) for x in name[len("c3autoclosed_w"):].split("r"))
        p = api.Plan(W.C3.n, W.C3.gens, L.FS_CONSUMER_COUNT, tail=1, gen_order=1, rank=rank, world=world)
        out = torch.zeros(1, dtype=torch.int64, device="cuda")
        fn = lambda: p.count_async(out)
    elif name in ("c3count", "c3closed", "c5count", "c3auto", "c3autoclosed"):
        inst = W.C5 if name == "c5count" else W.C3
        p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_COUNT, tail=1 if "closed" in name else 0,
                     gen_order=1 if "auto" in name else 0)
        out = torch.zeros(1, dtype=torch.int64, device="cuda")
        fn = lambda: p.count_async(out)
    elif name in ("c4hist", "c4histclosed"):
        inst = W.C4
        p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_HIST, tail=1 if "closed" in name else 0,
                     gen_order=1 if "closed" in name else 0)
        out = torch.zeros(api.hist_len(inst.n, inst.gens), dtype=torch.int64, device="cuda")
        fn = lambda: p.hist_async(out)
    elif name == "c5any_none":
        inst = W.C5
        p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ANY)
        f = torch.zeros(1, dtype=torch.int32, device="cuda")
        fn = lambda: p.any_async(L.FS_PRED_LEN_LE, 19, f)
    elif name in ("c2xl_m1", "c2xl_m2", "c2xl_m2auto"):
        inst = W.C2XL
        p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS, order=0 if name == "c2xl_m1" else 1,
                     gen_order=1 if name == "c2xl_m2auto" else 0)
        rows = p.info["total_rows"]
        out = torch.empty((rows, inst.d), dtype=torch.uint16, device="cuda")
        fn = lambda: p.enumerate_async(16, out, rows)
    else:
        raise SystemExit("unknown workload " + name)
    return fn


def main():
    name = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    fn = build(name)
    if os.environ.get("FS_TIME"):  # diagnostic timing (CUDA events), never under ncu
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(round(a.elapsed_time(b), 3))
        print(name, "ms", ts)
        return
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print(name, "ok")


if __name__ == "__main__":
    main()
