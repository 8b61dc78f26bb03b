# A/B timing of library variants on c5 and c4 (stage-1 launches)
mkdir -p gpurun_out
for lib in paper_2404_16648_b200/lib/libdg*.so; do
  echo "== $lib" >> gpurun_out/ab.log
  DG_LIB=$lib python scripts/run_stage.py c5 10 >> gpurun_out/ab.log 2>&1
  DG_LIB=$lib python scripts/run_stage.py c4 20 >> gpurun_out/ab.log 2>&1
done
DG_LIB=paper_2404_16648_b200/lib/libdg_ll.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c5 or c3 or random_amr_orders" > gpurun_out/ab_tests.log 2>&1
