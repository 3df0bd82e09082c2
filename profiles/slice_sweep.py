"""Diagnostic: C3 count (fs_count configuration) kernel time vs slice size, at W = 1 and for
rank 0 / rank 7 of W = 8 (CUDA events, median of 5 after 2 warm-ups; never a bench number)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("FS_PKG_ROOT", ROOT))
import torch  # noqa: E402

from paper_2405_07989_b200 import _lib as L  # noqa: E402
from paper_2405_07989_b200 import api  # noqa: E402
from paper_2405_07989_b200 import workloads as W  # noqa: E402

inst = W.C3
stream = torch.cuda.current_stream()
out = torch.zeros(1, dtype=torch.int64, device="cuda")
for world, rank in ((1, 0), (8, 0), (8, 7)):
    line = []
    for T in [int(x) for x in sys.argv[1:]] or (0, 400, 1500, 4000, 12000):
        p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_COUNT, tail=L.FS_TAIL_CLOSED, gen_order=L.FS_GENORDER_AUTO,
                     stream=stream.cuda_stream, rank=rank, world=world, slice_units=T)
        xs = []
        for k in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            p.count_async(out)
            b.record(stream)
            torch.cuda.synchronize()
            xs.append(a.elapsed_time(b))
        line.append("T=%d(%d):%.3f" % (T, p.info["slice_units"], statistics.median(xs[2:])))
    print("W=%d r=%d " % (world, rank) + " ".join(line), flush=True)
