mkdir -p gpurun_out
for lib in paper_2404_16648_b200/lib/libdg*.so; do
  echo "== $lib" >> gpurun_out/ab.log
  DG_LIB=$lib python scripts/run_stage.py c5 10 >> gpurun_out/ab.log 2>&1
done
DG_LIB=paper_2404_16648_b200/lib/libdg_ze.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c5 or single_element or random_amr_orders" > gpurun_out/pytest_new.log 2>&1
