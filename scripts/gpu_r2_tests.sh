mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage_strict.py tests/test_gpu_partition.py -x -q > gpurun_out/pytest_strict.log 2>&1; echo exit $? >> gpurun_out/pytest_strict.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo exit $? >> gpurun_out/smoke.log
