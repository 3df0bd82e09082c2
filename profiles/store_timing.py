"""Diagnostic: time the materialise kernels repeatedly (CUDA events), M1/M2, several orders."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_07989_b200 import _lib as L  # noqa: E402
from paper_2405_07989_b200 import api  # noqa: E402
from paper_2405_07989_b200 import workloads as W  # noqa: E402

inst = W.C2XL
stream = torch.cuda.current_stream()
for order, go in ((0, 0), (1, 0), (1, 1), (1, 0), (0, 0)):
    p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS, order=order, gen_order=go, stream=stream.cuda_stream)
    rows = p.info["total_rows"]
    out = torch.empty((rows, inst.d), dtype=torch.uint16, device="cuda")
    ts = []
    for r in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        p.enumerate_async(16, out, rows)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(round(a.elapsed_time(b), 3))
    print("order", order, "gen_order", go, "grid", p.info["grid"], "ms", ts, flush=True)
    del out, p
    torch.cuda.empty_cache()
