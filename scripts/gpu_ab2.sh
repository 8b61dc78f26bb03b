mkdir -p gpurun_out
for lib in paper_2404_16648_b200/lib/libdg*.so; do
  echo "== $lib" >> gpurun_out/ab.log
  DG_LIB=$lib python scripts/run_stage.py c5 10 >> gpurun_out/ab.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "single_element or zero_size" > gpurun_out/pytest_new.log 2>&1
