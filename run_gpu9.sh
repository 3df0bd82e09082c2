set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest9.log 2>&1; tail -3 gpurun_out/pytest9.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench9.json 2> gpurun_out/bench9.err; tail -3 gpurun_out/bench9.err
for w in c3autoclosed c2xl_m1 c2xl_m2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fs_enum_kernel -s 1 -c 1 -o gpurun_out/prof9_$w python profiles/workload.py $w 2 > gpurun_out/ncu9_$w.log 2>&1; tail -1 gpurun_out/ncu9_$w.log
done
