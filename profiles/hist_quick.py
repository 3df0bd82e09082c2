"""Diagnostic: C4 length histogram (fs_length_set's configuration: largest-first order, closed
tail), state-form walk vs residue-form walk, CUDA-event time of 5 launches after 2 warm-ups
(never a bench number), checked against the SURVEY golden SHA-256 of the histogram."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("FS_PKG_ROOT", ROOT))
import torch  # noqa: E402

from paper_2405_07989_b200 import _lib as L  # noqa: E402
from paper_2405_07989_b200 import api  # noqa: E402
from paper_2405_07989_b200 import workloads as W  # noqa: E402

GOLD = "732d09b032db36b6c536250ec753ddae1612ccfae0e19df8ccd8c028897bcdbd"
tag = sys.argv[1] if len(sys.argv) > 1 else ""
inst = W.C4
stream = torch.cuda.current_stream()
res = []
for walk in (L.FS_WALK_AUTO, L.FS_WALK_RESIDUE):
    p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_HIST, tail=L.FS_TAIL_CLOSED, gen_order=L.FS_GENORDER_AUTO,
                 walk=walk, stream=stream.cuda_stream)
    out = torch.zeros(api.hist_len(inst.n, inst.gens), dtype=torch.int64, device="cuda")
    import time
    t0 = time.time()
    while time.time() - t0 < 1.0:  # warm the clocks up (about 1 s of launches)
        p.count_async(out) if hasattr(p, "count_async") and p.consumer == L.FS_CONSUMER_COUNT else p.hist_async(out)
        torch.cuda.synchronize()
    ts = []
    for r in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        p.hist_async(out)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ok = hashlib.sha256(out.cpu().numpy().astype("<u8").tobytes()).hexdigest() == GOLD
    res.append("walk%d sb=%d %.3f ms %s" % (walk, p.info["state_block"], sorted(ts[2:])[2], "ok" if ok else "MISMATCH"))
print(tag, " | ".join(res), flush=True)
