"""Diagnostic: C3 count (fs_count configuration: generator order auto + closed tail), CUDA-event
time of 5 launches after 2 warm-ups."""
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
for inst in (W.C3, W.C5):
    T = int(os.environ.get("FS_T", "0"))
    if T and inst.name != "C3":
        T = 0
    p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_COUNT, tail=L.FS_TAIL_CLOSED, gen_order=L.FS_GENORDER_AUTO,
                 stream=stream.cuda_stream, slice_units=T)
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    ts = []
    for r in range(7):
        out.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        p.count_async(out)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(round(a.elapsed_time(b), 3))
    ok = int(out.item()) == {"C3": 100032405189, "C5": 4055053706}[inst.name]
    res.append("%s %s %s" % (inst.name, ts[2:], "ok" if ok else "WRONG"))
print(tag, " | ".join(res), flush=True)
