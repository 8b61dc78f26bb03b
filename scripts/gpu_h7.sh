mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stage_strict.py tests/test_gpu_partition.py -x -q -k "c5 or 7 or single" > gpurun_out/h7_tests.log 2>&1; echo exit $? >> gpurun_out/h7_tests.log
timeout 300 python bench.py --skip-cpu --skip-vortex --skip-c4 --steps 20 > gpurun_out/h7_bench.log 2>&1
DG_PHASE_PROF=1 python scripts/phase_prof.py c5 6 > gpurun_out/phase.log 2>&1
