set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; tail -3 gpurun_out/bench5.err
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest5.log 2>&1; tail -3 gpurun_out/pytest5.log
FS_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --no-extra > gpurun_out/bench5_gloo2.json 2> gpurun_out/bench5_gloo2.err; tail -3 gpurun_out/bench5_gloo2.err
for w in c3count c3closed c2xl_m1 c4hist; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fs_enum_kernel -s 1 -c 1 -o gpurun_out/prof5_$w python profiles/workload.py $w 2 > gpurun_out/ncu5_$w.log 2>&1; tail -1 gpurun_out/ncu5_$w.log
done
