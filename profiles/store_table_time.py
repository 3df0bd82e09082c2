"""Diagnostic: the one-shot cost of a canonical-order materialise plan (C2-XL): plan creation,
the first enumerate (slice-start table build + kernel) and a repeated enumerate, CUDA events
and host wall clock (never a bench number)."""
import os
import sys
import time

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
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.time()
    p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS, stream=stream.cuda_stream)
    t1 = time.time()
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    a.record(stream)
    p.enumerate_async(16, out, rows)
    b.record(stream)
    p.enumerate_async(16, out, rows)
    c.record(stream)
    torch.cuda.synchronize()
    t2 = time.time()
    res.append("plan %.2f ms, first %.3f ms, second %.3f ms, wall %.2f ms" % (
        (t1 - t0) * 1e3, a.elapsed_time(b), b.elapsed_time(c), (t2 - t0) * 1e3))
    del p
print(tag, " | ".join(res), flush=True)
