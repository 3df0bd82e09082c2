"""Diagnostic: which state makes the M2 (order any, generator order auto) kernel fast or slow:
back-to-back runs, host sleep between runs, output zeroed between runs, fresh plan per run."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_07989_b200 import _lib as L  # noqa: E402
from paper_2405_07989_b200 import api  # noqa: E402
from paper_2405_07989_b200 import workloads as W  # noqa: E402

inst = W.C2XL
stream = torch.cuda.current_stream()
go = int(sys.argv[1]) if len(sys.argv) > 1 else 1


def mk():
    return api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS, order=1, gen_order=go, stream=stream.cuda_stream)


p = mk()
rows = p.info["total_rows"]
out = torch.empty((rows, inst.d), dtype=torch.uint16, device="cuda")


def run(pl):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    pl.enumerate_async(16, out, rows)
    b.record(stream)
    torch.cuda.synchronize()
    return round(a.elapsed_time(b), 3)


run(p)
print("back-to-back", [run(p) for _ in range(6)], flush=True)
ts = []
for _ in range(6):
    time.sleep(0.2)
    ts.append(run(p))
print("sleep 200ms", ts, flush=True)
ts = []
for _ in range(6):
    out.zero_()
    torch.cuda.synchronize()
    ts.append(run(p))
print("zeroed", ts, flush=True)
ts = []
for _ in range(6):
    q = mk()
    ts.append(run(q))
    del q
print("fresh plan", ts, flush=True)
ts = []
for _ in range(6):
    q = mk()
    q.enumerate_async(16, out, 0) if False else None
    torch.cuda.synchronize()
    ts.append(run(q))
    del q
print("fresh plan, synced", ts, flush=True)
ts = []
for _ in range(6):
    out.fill_(0x1234)
    torch.cuda.synchronize()
    ts.append(run(p))
print("filled", ts, flush=True)
