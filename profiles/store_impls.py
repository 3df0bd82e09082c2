"""Diagnostic: CUDA-event timing of the materialise kernels, batch (FS_ROWS_BATCH) vs staged
(FS_ROWS_STAGED), M1 (canonical) / M2 (order any), on C2-XL (26 GB of u16 rows).  Checks the
batch M1 output against the staged M1 output by a device-side hash of sampled windows."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("FS_PKG_ROOT", ROOT))
import torch  # noqa: E402

from paper_2405_07989_b200 import _lib as L  # noqa: E402
from paper_2405_07989_b200 import api  # noqa: E402
from paper_2405_07989_b200 import workloads as W  # noqa: E402

inst = W.C2XL if len(sys.argv) < 2 else getattr(W, sys.argv[1])
stream = torch.cuda.current_stream()
keys = [(o, g, impl) for impl in (0, 1) for (o, g) in ((0, 0), (1, 0), (1, 1))]
plans = {k: api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS, order=k[0], gen_order=k[1], rows_impl=k[2],
                     stream=stream.cuda_stream) for k in keys}
rows = plans[keys[0]].info["total_rows"]
out = torch.empty((rows, inst.d), dtype=torch.uint16, device="cuda")
gb = rows * inst.d * 2 / 1e9
sums = {}
for key in keys:
    p = plans[key]
    ts = []
    for r in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        p.enumerate_async(16, out, rows)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    best = min(ts[1:])
    x = out.view(torch.int16)
    idx = torch.arange(0, rows, 9973, device="cuda")
    if key[0] == 0:
        sig = int((x[idx].to(torch.int64) * torch.arange(1, inst.d + 1, device="cuda")).sum())
    else:
        sig = int(x.to(torch.int64).sum(0).sum()) if rows < (1 << 31) else None
    sums[key] = sig
    print("order %d gen_order %d impl %d launches %d: ms %s  best %.3f ms = %.0f GB/s  sig %s"
          % (key[0], key[1], key[2], p.last_launches(), [round(t, 3) for t in ts], best, gb / best * 1e3, sig),
          flush=True)
print("M1 batch == staged sampled:", sums[(0, 0, 0)] == sums[(0, 0, 1)])
