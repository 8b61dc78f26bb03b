mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "projection_orders or copy_elements" > gpurun_out/pytest_new.log 2>&1; echo exit $? >> gpurun_out/pytest_new.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_rhs or c2_rhs or rest_state or random_amr_orders or projection_orders or copy_elements or argument" > gpurun_out/memcheck.log 2>&1; echo exit $? >> gpurun_out/memcheck.log
