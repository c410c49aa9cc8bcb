set -x
cd $GRAFT_REPO_ROOT
/usr/bin/time -v python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
tail -3 gpurun_out/r02d_bench.err
VISLOC_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --no-configs --steps 3 --no-cpu > gpurun_out/r02d_gloo2.json 2> gpurun_out/r02d_gloo2.err
tail -3 gpurun_out/r02d_gloo2.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_lift -c 3 -o gpurun_out/r02d_lift python bench.py --workload c5 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r02d_ncu_lift.log 2>&1
tail -3 gpurun_out/r02d_ncu_lift.log
