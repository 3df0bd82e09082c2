"""Diagnostic: time the materialise kernels repeatedly (CUDA events), M1/M2, several orders,
on two separate allocations of the 26 GB output."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_07989_b200 import _lib as L  # noqa: E402
from paper_2405_07989_b200 import api  # noqa: E402
from paper_2405_07989_b200 import workloads as W  # noqa: E402

inst = W.C2XL
stream = torch.cuda.current_stream()
plans = {(o, g): api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS, order=o, gen_order=g, stream=stream.cuda_stream)
         for o, g in ((0, 0), (1, 0), (1, 1))}
rows = plans[(0, 0)].info["total_rows"]
for alloc in range(3):
    out = torch.empty((rows, inst.d), dtype=torch.uint16, device="cuda")
    print("alloc", alloc, "ptr", hex(out.data_ptr()), flush=True)
    for key in ((0, 0), (1, 0), (1, 1), (1, 0)):
        p = plans[key]
        ts = []
        for r in range(4):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            p.enumerate_async(16, out, rows)
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(round(a.elapsed_time(b), 3))
        print("  order", key[0], "gen_order", key[1], "ms", ts, flush=True)
    del out
    torch.cuda.empty_cache()
