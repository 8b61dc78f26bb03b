# A/B of stage-kernel variants: bash scripts/gpu_ab.sh "<configs>" lib1.so lib2.so ...
#   (each lib under paper_2404_16648_b200/lib/; two alternating repetitions; results in gpurun_out/ab.log)
mkdir -p gpurun_out; : > gpurun_out/ab.log
cfgs=$1; shift
for rep in 1 2; do
for cfg in $cfgs; do
for lib in "$@"; do
  DG_LIB=paper_2404_16648_b200/lib/$lib timeout 300 python scripts/ab_c5.py $cfg 10 >> gpurun_out/ab.log 2>&1
done; done; done
