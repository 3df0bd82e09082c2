"""Diagnostic: time of tiny shards of the C3 count (rank 0 of W = 64 .. 4096), i.e. the fixed
cost of one persistent launch (CUDA events, median of 5; never a bench number)."""
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
line = []
for world in (8, 64, 512, 4096, 32768):
    for rank in (0, world - 1):
        p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_COUNT, tail=L.FS_TAIL_CLOSED, gen_order=L.FS_GENORDER_AUTO,
                     stream=stream.cuda_stream, rank=rank, world=world)
        xs = []
        for k in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            p.count_async(out)
            b.record(stream)
            torch.cuda.synchronize()
            xs.append(a.elapsed_time(b))
        i = p.info
        line.append("W=%d r=%d T=%d slices=%d grid=%d: %.4f ms" % (world, rank, i["slice_units"], i["num_slices"],
                                                                  i["grid"], statistics.median(xs[2:])))
print("\n".join(line), flush=True)
