"""Diagnostic: the bench's store sequence (M1, M2 given, M2 auto), each with its own fresh
26 GB allocation (mode 'fresh') or one shared allocation (mode 'shared')."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("FS_PKG_ROOT", ROOT))
import torch  # noqa: E402

from paper_2405_07989_b200 import _lib as L  # noqa: E402
from paper_2405_07989_b200 import api  # noqa: E402
from paper_2405_07989_b200 import workloads as W  # noqa: E402

mode = sys.argv[1]
inst = W.C2XL
stream = torch.cuda.current_stream()
shared = None
line = []
for order, go in ((0, 0), (1, 0), (1, 1)):
    p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS, order=order, gen_order=go, stream=stream.cuda_stream)
    rows = p.info["total_rows"]
    if mode == "shared":
        if shared is None:
            shared = torch.empty((rows, inst.d), dtype=torch.uint16, device="cuda")
        out = shared
    else:
        out = torch.empty((rows, inst.d), dtype=torch.uint16, device="cuda")
    ts = []
    for r in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        p.enumerate_async(16, out, rows)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(round(a.elapsed_time(b), 2))
    line.append("o%dg%d %s" % (order, go, ts))
    if mode != "shared":
        del out
        torch.cuda.empty_cache()
print(mode, " | ".join(line), flush=True)
