# z-pass field split (DG_ZFIELD) vs the row split: N = 7 parity on the variant, then same-box A/B on c5 (3 reps)
mkdir -p gpurun_out
DG_LIB=paper_2404_16648_b200/lib/libdg_zf.so python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "c5 or h7 or 7" > gpurun_out/ab_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/ab_tests.log
for rep in 1 2 3; do
for lib in paper_2404_16648_b200/lib/libdg.so paper_2404_16648_b200/lib/libdg_zf.so; do
  echo "== $lib" >> gpurun_out/ab.log
  DG_LIB=$lib python scripts/run_stage.py c5 20 >> gpurun_out/ab.log 2>&1
done
done
