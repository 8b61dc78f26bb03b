mkdir -p gpurun_out
./scripts/fp64_mix > gpurun_out/fp64_mix.log 2>&1
./scripts/fp64_peak > gpurun_out/fp64_peak.log 2>&1
./scripts/dmma_peak > gpurun_out/dmma_peak.log 2>&1
nproc > gpurun_out/host.log; lscpu | grep -i "model name" >> gpurun_out/host.log
timeout 300 python bench.py --skip-cpu --skip-vortex --steps 20 > gpurun_out/bench_r2_base.log 2>&1
python scripts/run_stage.py c4 20 > gpurun_out/stages_base.log 2>&1; python scripts/run_stage.py c5n4 10 >> gpurun_out/stages_base.log 2>&1
