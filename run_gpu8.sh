set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest8.log 2>&1; tail -3 gpurun_out/pytest8.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench8.json 2> gpurun_out/bench8.err; tail -3 gpurun_out/bench8.err
for w in c2xl_m1 c4histclosed; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fs_enum_kernel -s 1 -c 1 -o gpurun_out/prof8_$w python profiles/workload.py $w 2 > gpurun_out/ncu8_$w.log 2>&1; tail -1 gpurun_out/ncu8_$w.log
done
