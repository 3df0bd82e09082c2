"""Diagnostic: M2 (order any) time per plan instance.  Each Plan owns its own scratch
(front/back cursors); if the time is bimodal across plans in one process, the cursor's
placement (L2 slice / die) decides the speed."""
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
go = int(sys.argv[1]) if len(sys.argv) > 1 else 0
nplans = int(sys.argv[2]) if len(sys.argv) > 2 else 12
plans = [api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS, order=1, gen_order=go, stream=stream.cuda_stream)
         for _ in range(nplans)]
rows = plans[0].info["total_rows"]
out = torch.empty((rows, inst.d), dtype=torch.uint16, device="cuda")
for i, p in enumerate(plans):
    ts = []
    for r in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        p.enumerate_async(16, out, rows)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(round(a.elapsed_time(b), 3))
    print("gen_order", go, "plan", i, "ms", ts, flush=True)
