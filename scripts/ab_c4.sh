mkdir -p gpurun_out; : > gpurun_out/ab_c4.log
for rep in 1 2; do
for lib in "$@"; do
  echo "== $lib" >> gpurun_out/ab_c4.log
  DG_LIB=paper_2404_16648_b200/lib/$lib python scripts/ab_c5.py c4 10 >> gpurun_out/ab_c4.log 2>&1
done; done
