mkdir -p gpurun_out; : > gpurun_out/ab.log
DG_LIB=paper_2404_16648_b200/lib/libdg_both.so timeout 600 python -m pytest tests/test_gpu_stage_strict.py tests/test_gpu_parity.py -x -q -k "c5 or 7 or c1 or c2 or c3" > gpurun_out/ab_tests.log 2>&1; echo exit $? >> gpurun_out/ab_tests.log
for rep in 1 2; do
for lib in "$@"; do
  DG_LIB=paper_2404_16648_b200/lib/$lib python scripts/ab_c5.py c5 10 >> gpurun_out/ab.log 2>&1
done; done
