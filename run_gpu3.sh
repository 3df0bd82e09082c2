set -x
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,driver_version --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -3 gpurun_out/bench3.err
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest3.log 2>&1; tail -15 gpurun_out/pytest3.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fs_enum_kernel -s 3 -c 1 -o gpurun_out/prof_count3 python bench.py --steps 1 --warmup 3 --no-extra --cpu-seconds 1 > gpurun_out/ncu_full3.log 2>&1; tail -3 gpurun_out/ncu_full3.log
cat > /tmp/store.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_2405_07989_b200 import api, _lib as L, workloads as W
i = W.C2XL
for order in (0, 1):
    p = api.Plan(i.n, i.gens, L.FS_CONSUMER_ROWS, order=order)
    rows = p.info['total_rows']
    out = torch.empty((rows, i.d), dtype=torch.uint16, device='cuda')
    for _ in range(2):
        p.enumerate_async(16, out, rows)
    torch.cuda.synchronize()
    del out
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fs_enum_kernel -s 1 -c 1 -o gpurun_out/prof_store3 python /tmp/store.py > gpurun_out/ncu_store3.log 2>&1; tail -3 gpurun_out/ncu_store3.log
ls -la gpurun_out
