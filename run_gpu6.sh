set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest6.log 2>&1; tail -3 gpurun_out/pytest6.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench6.json 2> gpurun_out/bench6.err; tail -3 gpurun_out/bench6.err
for w in c2xl_m1 c2xl_m2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fs_enum_kernel -s 1 -c 1 -o gpurun_out/prof6_$w python profiles/workload.py $w 2 > gpurun_out/ncu6_$w.log 2>&1; tail -1 gpurun_out/ncu6_$w.log
done
