mkdir -p gpurun_out
export DG_LIB=paper_2404_16648_b200/lib/libdg_debug.so
timeout 600 python scripts/sanitize_run.py > gpurun_out/debug_run.log 2>&1; echo exit $? >> gpurun_out/debug_run.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nonconforming.py tests/test_gpu_partition.py tests/test_gpu_regrid.py -x -q > gpurun_out/debug_tests.log 2>&1; echo exit $? >> gpurun_out/debug_tests.log
