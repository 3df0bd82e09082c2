"""Diagnostic: C3 count (fs_count's configuration: largest-first order, closed tail), CUDA-event
time of 5 launches after 2 warm-ups (never a bench number), checked against |Z| from the DP."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("FS_PKG_ROOT", ROOT))
import torch  # noqa: E402

from paper_2405_07989_b200 import _lib as L  # noqa: E402
from paper_2405_07989_b200 import api  # noqa: E402
from paper_2405_07989_b200 import workloads as W  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else ""
stream = torch.cuda.current_stream()
res = []
for inst in (W.C3, W.C3CD) if hasattr(W, "C3CD") else (W.C3,):
    p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_COUNT, tail=L.FS_TAIL_CLOSED, gen_order=L.FS_GENORDER_AUTO,
                 stream=stream.cuda_stream)
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    import time
    t0 = time.time()
    while time.time() - t0 < 1.0:  # warm the clocks up (about 1 s of launches)
        p.count_async(out) if hasattr(p, "count_async") and p.consumer == L.FS_CONSUMER_COUNT else p.hist_async(out)
        torch.cuda.synchronize()
    ts = []
    for r in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        p.count_async(out)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ok = int(out.item()) == p.info["total_rows"]
    res.append("%s sb=%d %.3f ms %s" % (inst.name, p.info["state_block"], sorted(ts[2:])[2], "ok" if ok else "MISMATCH"))
print(tag, " | ".join(res), flush=True)
