set -x
timeout 600 python profiles/store_timing.py 2>&1 | tail -20
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest11.log 2>&1; tail -3 gpurun_out/pytest11.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench11.json 2> gpurun_out/bench11.err; tail -3 gpurun_out/bench11.err
for w in c3autoclosed c2xl_m1 c2xl_m2auto; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fs_enum_kernel -s 1 -c 1 -o gpurun_out/prof11_$w python profiles/workload.py $w 2 > gpurun_out/ncu11_$w.log 2>&1; tail -1 gpurun_out/ncu11_$w.log
done
