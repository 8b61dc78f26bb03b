# round-end refresh: GPU tests, smoke, default bench, reference arm, launch list of the bench
# command, ncu --set full of k_stage_h7 (stage 0 + stage 1 of c5) and k_stage_h4 (c5n4)
mkdir -p gpurun_out
nproc > gpurun_out/host.log; lscpu | grep -i "model name" >> gpurun_out/host.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit $? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit $? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err
CMD="python bench.py --steps 5 --warmup 3 --skip-cpu --skip-c4 --skip-vortex --skip-configs"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
CMD2="python bench.py --steps 2 --warmup 3 --skip-cpu --skip-c4 --skip-vortex --skip-configs"
ncu --set full --clock-control none --import-source on -k regex:k_stage_h7 -s 12 -c 2 -o gpurun_out/prof_h7 -f $CMD2 > gpurun_out/ncu_h7.log 2>&1
bash scripts/gpu_prof.sh c5n4 k_stage_h4 h4_c5n4
bash scripts/gpu_prof.sh c4 "k_stage_h4|k_mortar_h4" h4_c4 2
bash scripts/gpu_debug.sh
echo done >> gpurun_out/plain.log
