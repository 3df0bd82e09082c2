"""Diagnostic: canonical materialise (M1) time vs rows per slice (the write window of the
grid is lanes x slice rows x row bytes; small windows keep the TLB warm)."""
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
p0 = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS)
rows = p0.info["total_rows"]
out = torch.empty((rows, inst.d), dtype=torch.uint16, device="cuda")
for T in (0, 64, 128, 256, 512, 2048):
    p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS, slice_units=T, stream=stream.cuda_stream)
    ts = []
    for r in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        p.enumerate_async(16, out, rows)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(round(a.elapsed_time(b), 3))
    print("T", p.info["slice_units"], "slices", p.info["num_slices"], "ms", ts, flush=True)
