# ncu --set full capture of the stage kernel on one config:  bash scripts/gpu_prof.sh <config> <kernel-regex> [tag]
#   e.g. bash scripts/gpu_prof.sh c4 k_stage h4 [launches]  -> gpurun_out/prof_h4.ncu-rep
# (runs the command once without ncu first; the capture only if that exits 0)
mkdir -p gpurun_out
cfg=${1:-c4}; kre=${2:-k_stage}; tag=${3:-$cfg}; cnt=${4:-1}
CMD="python scripts/run_stage.py $cfg 3"
$CMD > gpurun_out/prof_$tag.plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:$kre -s 2 -c $cnt -o gpurun_out/prof_$tag -f $CMD > gpurun_out/prof_$tag.ncu.log 2>&1
echo done $? >> gpurun_out/prof_$tag.ncu.log
