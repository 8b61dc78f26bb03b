# same-box A/B of every lib/libdg*.so on c4 / c5n4, with parity of each variant on c4/c3
mkdir -p gpurun_out
for lib in paper_2404_16648_b200/lib/libdg*.so; do
  echo "== $lib" >> gpurun_out/ab_tests.log
  DG_LIB=$lib python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "c3 or c4 or random_amr" >> gpurun_out/ab_tests.log 2>&1
done
for rep in 1 2; do
for lib in paper_2404_16648_b200/lib/libdg*.so; do
  echo "== $lib" >> gpurun_out/ab.log
  DG_LIB=$lib python scripts/run_stage.py c4 20 >> gpurun_out/ab.log 2>&1
  DG_LIB=$lib python scripts/run_stage.py c5n4 10 >> gpurun_out/ab.log 2>&1
done
done
