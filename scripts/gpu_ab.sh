# A/B timing of library variants on c5 and c4 (stage-1 launches)
mkdir -p gpurun_out
for lib in paper_2404_16648_b200/lib/libdg*.so; do
  echo "== $lib" >> gpurun_out/ab.log
  DG_LIB=$lib python scripts/run_stage.py c5 10 >> gpurun_out/ab.log 2>&1
  DG_LIB=$lib python scripts/run_stage.py c4 20 >> gpurun_out/ab.log 2>&1
done
