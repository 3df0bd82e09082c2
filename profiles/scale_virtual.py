"""Virtual-rank scaling estimate on ONE GPU (never a bench number): for W in (1, 2, 4, 8) run
each rank's share of the C3 count (fs_count configuration) alone, CUDA-event timed (median of
5 after 2 warm-ups), and report max over ranks -- the per-rank kernel time an 8-GPU run would
see before its all_reduce.  predicted scaling = t(1) / max_r t_r(W)."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.environ.get("FS_PKG_ROOT", ROOT))
import torch  # noqa: E402

from paper_2405_07989_b200 import _lib as L  # noqa: E402
from paper_2405_07989_b200 import api  # noqa: E402
from paper_2405_07989_b200 import workloads as W  # noqa: E402

inst = W.CONFIGS[sys.argv[1]] if len(sys.argv) > 1 else W.C3
cons = L.FS_CONSUMER_HIST if inst.name == "C4" else L.FS_CONSUMER_COUNT
stream = torch.cuda.current_stream()
out = torch.zeros(max(1, api.hist_len(inst.n, inst.gens)), dtype=torch.int64, device="cuda")
res = {}
import time  # noqa: E402

_p0 = api.Plan(inst.n, inst.gens, cons, tail=L.FS_TAIL_CLOSED, gen_order=L.FS_GENORDER_AUTO, stream=stream.cuda_stream)
_t0 = time.time()
while time.time() - _t0 < 1.0:  # warm the clocks up
    (_p0.hist_async(out) if cons == L.FS_CONSUMER_HIST else _p0.count_async(out))
    torch.cuda.synchronize()
WORLDS = [int(x) for x in os.environ.get("FS_WORLDS", "1,2,4,8").split(",")]
for world in WORLDS:
    ts = []
    tot = 0
    for r in range(world):
        p = api.Plan(inst.n, inst.gens, cons, tail=L.FS_TAIL_CLOSED, gen_order=L.FS_GENORDER_AUTO,
                     stream=stream.cuda_stream, rank=r, world=world)
        fn = (lambda: p.hist_async(out)) if cons == L.FS_CONSUMER_HIST else (lambda: p.count_async(out))
        xs = []
        for k in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            xs.append(a.elapsed_time(b))
        tot += int(out.sum().item()) if cons == L.FS_CONSUMER_HIST else int(out[0].item())
        ts.append(statistics.median(xs[2:]))
    assert tot == p.info["total_rows"], (world, tot)
    res[world] = {"per_rank_ms": [round(x, 4) for x in ts], "max_ms": round(max(ts), 4)}
for world in WORLDS[1:]:
    res[world]["predicted_scaling"] = round(res[1]["max_ms"] / res[world]["max_ms"], 3)
print(json.dumps({"instance": inst.name, **{str(k): v for k, v in res.items()}}), flush=True)
