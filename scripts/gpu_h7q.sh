mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stage_strict.py tests/test_gpu_partition.py tests/test_gpu_regrid.py -x -q -k "c5 or 7 or single or regrid" > gpurun_out/h7_tests.log 2>&1; echo exit $? >> gpurun_out/h7_tests.log
: > gpurun_out/ab.log
for rep in 1 2; do for lib in "$@"; do DG_LIB=paper_2404_16648_b200/lib/$lib python scripts/ab_c5.py c5 10 >> gpurun_out/ab.log 2>&1; done; done
