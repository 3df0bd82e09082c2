set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest7.log 2>&1; tail -3 gpurun_out/pytest7.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench7.json 2> gpurun_out/bench7.err; tail -3 gpurun_out/bench7.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches7.csv python bench.py --steps 2 --warmup 3 --no-extra --cpu-seconds 1 > /dev/null 2>&1
for w in c3autoclosed c3count c2xl_m1 c2xl_m2auto; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fs_enum_kernel -s 1 -c 1 -o gpurun_out/prof7_$w python profiles/workload.py $w 2 > gpurun_out/ncu7_$w.log 2>&1; tail -1 gpurun_out/ncu7_$w.log
done
