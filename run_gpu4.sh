set -x
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; tail -3 gpurun_out/bench4.err
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest4.log 2>&1; tail -5 gpurun_out/pytest4.log
for w in c3count c3closed c2xl_m1 c2xl_m2 c4hist c5any_none; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fs_enum_kernel -s 1 -c 1 -o gpurun_out/prof4_$w python profiles/workload.py $w 2 > gpurun_out/ncu4_$w.log 2>&1; tail -1 gpurun_out/ncu4_$w.log
done
ls gpurun_out
