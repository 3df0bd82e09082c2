"""Diagnostic: M2 (order any) time, given and auto generator order, 4 runs each."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("FS_PKG_ROOT", ROOT))
import torch  # noqa: E402

from paper_2405_07989_b200 import _lib as L  # noqa: E402
from paper_2405_07989_b200 import api  # noqa: E402
from paper_2405_07989_b200 import workloads as W  # noqa: E402

inst = W.C2XL
stream = torch.cuda.current_stream()
tag = sys.argv[1] if len(sys.argv) > 1 else ""
out = None
res = []
for go in (0, 1):
    p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS, order=1, gen_order=go, stream=stream.cuda_stream,
                 ctas_per_sm=int(os.environ.get("FS_CTAS", "0")))
    rows = p.info["total_rows"]
    if out is None:
        out = torch.empty((rows, inst.d), dtype=torch.uint16, device="cuda")
    ts = []
    for r in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        p.enumerate_async(16, out, rows)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(round(a.elapsed_time(b), 2))
    res.append("go%d %s" % (go, ts[1:]))
print(tag, " | ".join(res), flush=True)
