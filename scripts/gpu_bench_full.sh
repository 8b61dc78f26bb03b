mkdir -p gpurun_out
nproc > gpurun_out/host.log; lscpu | grep -i "model name" >> gpurun_out/host.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err
CMD="python bench.py --steps 2 --warmup 3 --skip-cpu --skip-c4 --skip-vortex --skip-configs"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_stage_h7 -s 12 -c 4 -o gpurun_out/prof_h7r2 -f $CMD > gpurun_out/ncu_h7r2.log 2>&1
echo done $? >> gpurun_out/ncu_h7r2.log
