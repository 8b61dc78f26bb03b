mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --skip-cpu --skip-c4 --skip-vortex --skip-configs"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_stage_h7 -s 12 -c 4 -o gpurun_out/prof_h7r2b -f $CMD > gpurun_out/ncu_h7r2b.log 2>&1
echo done $? >> gpurun_out/ncu_h7r2b.log
