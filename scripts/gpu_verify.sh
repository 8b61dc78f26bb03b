# re-entry check: GPU tests, smoke, default bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit $? >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit $? >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2>&1; echo bench_exit $? >> gpurun_out/bench.log
