mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit $? >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --skip-cpu > gpurun_out/bench.log 2>&1
python scripts/run_stage.py c4 10 > gpurun_out/stages.log 2>&1; python scripts/run_stage.py c3 20 >> gpurun_out/stages.log 2>&1; python scripts/run_stage.py c5n4 10 >> gpurun_out/stages.log 2>&1
python bench.py --steps 5 --warmup 3 --skip-cpu --skip-c4 --skip-vortex > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_stage -s 3 -c 3 -o gpurun_out/prof python bench.py --steps 5 --warmup 3 --skip-cpu --skip-c4 --skip-vortex > gpurun_out/ncu_full.log 2>&1
python scripts/run_stage.py c4 3 > gpurun_out/c4_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_stage -s 2 -c 1 -o gpurun_out/prof_c4 python scripts/run_stage.py c4 3 > gpurun_out/ncu_c4.log 2>&1
ls gpurun_out
