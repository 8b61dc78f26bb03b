# generic kernel evict-first hints (DG_CSQ: q_n loads only) A/B on c4 / c5n4 (h7 already streams by default); full GPU tests on the default lib
mkdir -p gpurun_out
DG_LIB=paper_2404_16648_b200/lib/libdg_cs.so python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/ab_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/ab_tests.log
for rep in 1 2 3; do
for lib in paper_2404_16648_b200/lib/libdg.so paper_2404_16648_b200/lib/libdg_cs.so; do
  echo "== $lib" >> gpurun_out/ab.log
  DG_LIB=$lib python scripts/run_stage.py c4 20 >> gpurun_out/ab.log 2>&1
  DG_LIB=$lib python scripts/run_stage.py c5n4 10 >> gpurun_out/ab.log 2>&1
done
done
