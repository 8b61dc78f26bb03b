timeout 60 python scripts/ab_c5.py c3 3 > gpurun_out/smoke_c3.log 2>&1; echo exit $? >> gpurun_out/smoke_c3.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit $? >> gpurun_out/pytest_gpu.log
