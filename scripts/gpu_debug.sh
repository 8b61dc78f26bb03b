# DG_DEBUG build (shared-memory / index bounds checks, bounded mbarrier waits; a failed check traps):
# the sanitize driver and the GPU tests of every stage kernel, the transfers, the tracers and partitions
mkdir -p gpurun_out
export DG_LIB=paper_2404_16648_b200/lib/libdg_debug.so
timeout 600 python scripts/sanitize_run.py > gpurun_out/debug_run.log 2>&1; echo exit $? >> gpurun_out/debug_run.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nonconforming.py tests/test_gpu_partition.py tests/test_gpu_regrid.py tests/test_gpu_h4.py tests/test_gpu_passive.py tests/test_gpu_stage_strict.py -x -q > gpurun_out/debug_tests.log 2>&1; echo exit $? >> gpurun_out/debug_tests.log
