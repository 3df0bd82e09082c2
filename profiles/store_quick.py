"""Diagnostic: C2-XL materialise (26 GB of u16 rows), canonical and increasing order, CUDA-event
time of 5 launches after 2 warm-ups (never a bench number)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("FS_PKG_ROOT", ROOT))
import torch  # noqa: E402

from paper_2405_07989_b200 import _lib as L  # noqa: E402
from paper_2405_07989_b200 import api  # noqa: E402
from paper_2405_07989_b200 import workloads as W  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else ""
inst = W.C2XL
stream = torch.cuda.current_stream()
rows = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS).info["total_rows"]
out = torch.empty((rows, inst.d), dtype=torch.uint16, device="cuda")
res = []
for order in (L.FS_ORDER_CANONICAL, L.FS_ORDER_INCREASING, L.FS_ORDER_ANY):
    p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS, order=order, stream=stream.cuda_stream)
    ts = []
    for r in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        p.enumerate_async(16, out, rows)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts[2:])[2]
    res.append("order%d %.3f ms %.0f GB/s" % (order, ms, rows * 10 / ms / 1e6))
print(tag, " | ".join(res), flush=True)
