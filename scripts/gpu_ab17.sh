# q_n L2 prefetch one tile ahead (DG_QNX) vs this tile (default)
mkdir -p gpurun_out
DG_LIB=paper_2404_16648_b200/lib/libdg_qnx.so python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "c5 or 7" > gpurun_out/ab_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/ab_tests.log
for rep in 1 2 3; do
for lib in paper_2404_16648_b200/lib/libdg.so paper_2404_16648_b200/lib/libdg_qnx.so; do
  echo "== $lib" >> gpurun_out/ab.log
  DG_LIB=$lib python scripts/run_stage.py c5 20 >> gpurun_out/ab.log 2>&1
done
done
for lib in paper_2404_16648_b200/lib/libdg.so paper_2404_16648_b200/lib/libdg_qnx.so; do
  echo "== $lib" >> gpurun_out/ab_dram.log
  DG_LIB=$lib ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_stage -s 2 -c 2 python scripts/run_stage.py c5 3 >> gpurun_out/ab_dram.log 2>&1
done
