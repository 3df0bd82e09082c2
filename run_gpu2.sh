set -x
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,driver_version --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -3 gpurun_out/bench2.err
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest2.log 2>&1; tail -30 gpurun_out/pytest2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2.csv python bench.py --steps 2 --warmup 3 --no-extra --cpu-seconds 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fs_enum_kernel -s 3 -c 1 -o gpurun_out/prof_count2 python bench.py --steps 1 --warmup 3 --no-extra --cpu-seconds 1 > gpurun_out/ncu_full2.log 2>&1; tail -3 gpurun_out/ncu_full2.log
ls -la gpurun_out
