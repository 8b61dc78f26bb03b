# state of the tree: GPU tests, smoke, default bench, launch list of the bench command
mkdir -p gpurun_out
nproc > gpurun_out/host.log; lscpu | grep -i "model name" >> gpurun_out/host.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit $? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit $? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
CMD="python bench.py --steps 5 --warmup 3 --skip-cpu --skip-c4 --skip-vortex --skip-configs"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo done >> gpurun_out/plain.log
